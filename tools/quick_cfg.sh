#!/bin/bash
# quick per-config bench at reduced size (profiling iterations): bash tools/quick_cfg.sh <tag>
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python bench.py --config c3 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c3_1M.json 2> $OUT/c3.err; echo "c3 $?" >> $OUT/status
timeout 600 python bench.py --config c5 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c5_1M.json 2> $OUT/c5.err; echo "c5 $?" >> $OUT/status
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c2.json 2> $OUT/c2.err; echo "c2 $?" >> $OUT/status
cat $OUT/status
