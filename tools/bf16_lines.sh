#!/bin/bash
# bfloat16-sketch (F3) bench lines next to the fp32 ones: bash tools/bf16_lines.sh <tag>
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 python bench.py --bf16 --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_bf16.json 2> $OUT/c2.err; echo "c2 $?" >> $OUT/status
timeout 1500 python bench.py --bf16 --config c5 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c5_bf16.json 2> $OUT/c5.err; echo "c5 $?" >> $OUT/status
timeout 1500 python bench.py --bf16 --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_bf16.json 2> $OUT/c3.err; echo "c3 $?" >> $OUT/status
cat $OUT/status
