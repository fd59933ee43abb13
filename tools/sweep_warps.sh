#!/bin/bash
OUT=gpurun_out/sw; mkdir -p $OUT
for c in c3 c5; do for w in 32 24 16 12 8; do
  SINN_DOC_WARPS=$w timeout 600 python bench.py --config $c --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/${c}_w$w.json 2>/dev/null
done; done
for w in 32 24 16; do SINN_DOC_WARPS=$w timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $OUT/c2_w$w.json 2>/dev/null; done
