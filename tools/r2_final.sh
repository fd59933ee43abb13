#!/bin/bash
# round-2 evidence: bench lines of every config, bf16 config 5, and a full-size config-3 ncu capture
TAG=${1:-fin}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1200 python bench.py > $OUT/default.json 2> $OUT/default.err; echo "default $?" >> $OUT/status
for c in tiny c2; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $OUT/$c.json 2> $OUT/$c.err; echo "$c $?" >> $OUT/status; done
timeout 1500 python bench.py --config c4 > $OUT/c4.json 2> $OUT/c4.err; echo "c4 $?" >> $OUT/status
timeout 900 python bench.py --config c5 --also none --bf16 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/c5_bf16.json 2> $OUT/c5_bf16.err; echo "c5bf16 $?" >> $OUT/status
ARGS="--config c3 --also none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 python bench.py $ARGS > $OUT/c3_plain.json 2> $OUT/c3_plain.err && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_doc_score -s 5 -c 1 \
   -o $OUT/prof_c3 python bench.py $ARGS > $OUT/ncu_c3.log 2>&1; echo "ncu_c3 $?" >> $OUT/status
cat $OUT/status
