#!/bin/bash
OUT=gpurun_out/ps; mkdir -p $OUT
for x in 0 1 2 4; do
  SINN_PARTS_X=$x timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $OUT/c2_x$x.json 2>/dev/null
  SINN_PARTS_X=$x timeout 600 python bench.py --config c3 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c3_x$x.json 2>/dev/null
done
