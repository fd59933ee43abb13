#!/bin/bash
# full-size config-5 evidence: the launch list of one bench run, then a --set full capture of the EMIT pass
# of k_doc_score (the dominant kernel of the default line); plus the new per-query-mask tests and config 4
TAG=${1:-c5p}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu -k "per_query" > $OUT/masked.log 2>&1; echo "masked $?" >> $OUT/status
timeout 1200 python bench.py --config c4 > $OUT/c4.json 2> $OUT/c4.err; echo "c4 $?" >> $OUT/status
ARGS="--config c5 --also none --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 python bench.py $ARGS > $OUT/plain.json 2> $OUT/plain.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
   --log-file $OUT/launches.csv python bench.py $ARGS > $OUT/ncu_launch.log 2>&1; echo "launch $?" >> $OUT/status
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_doc_score -s 5 -c 1 \
   -o $OUT/prof python bench.py $ARGS > $OUT/ncu_full.log 2>&1; echo "full $?" >> $OUT/status
cat $OUT/status
