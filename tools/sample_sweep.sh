#!/bin/bash
OUT=gpurun_out/ss; mkdir -p $OUT
for x in 64 128 256; do
  SINN_SAMPLE_X=$x timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $OUT/c2_x$x.json 2>/dev/null
  SINN_SAMPLE_X=$x timeout 600 python bench.py --config c3 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c3_x$x.json 2>/dev/null
  SINN_SAMPLE_X=$x timeout 600 python bench.py --config c5 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c5_x$x.json 2>/dev/null
done
