#!/bin/bash
# round-2 (final) evidence: bench lines of every config (+ containers, bf16), launch list, full-size ncu
TAG=${1:-ev}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1500 python bench.py > $OUT/default.json 2> $OUT/default.err; echo "default $?" >> $OUT/status
for c in tiny c2; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $OUT/$c.json 2> $OUT/$c.err; echo "$c $?" >> $OUT/status; done
timeout 1500 python bench.py --config c4 > $OUT/c4.json 2> $OUT/c4.err; echo "c4 $?" >> $OUT/status
B="--also none --steps 5 --warmup 3 --no-cpu-baseline"
timeout 900 python bench.py --config c5 $B --bf16 > $OUT/c5_bf16.json 2> $OUT/c5_bf16.err; echo "c5bf16 $?" >> $OUT/status
timeout 900 python bench.py --config c3 $B --containers > $OUT/c3_containers.json 2> $OUT/c3_containers.err; echo "c3cont $?" >> $OUT/status
timeout 900 python bench.py --config c5 $B --containers > $OUT/c5_containers.json 2> $OUT/c5_containers.err; echo "c5cont $?" >> $OUT/status
A5="--config c5 --also none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv \
   python bench.py $A5 > $OUT/ncu_launch.log 2>&1; echo "launches $?" >> $OUT/status
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_doc_score -s 5 -c 1 \
   -o $OUT/prof_c5 python bench.py $A5 > $OUT/ncu_c5.log 2>&1; echo "ncu_c5 $?" >> $OUT/status
cat $OUT/status
