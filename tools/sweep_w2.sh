#!/bin/bash
OUT=gpurun_out/sw2; mkdir -p $OUT
for w in 28 29 30 31 32; do SINN_DOC_WARPS=$w timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > $OUT/c2_w$w.json 2>/dev/null; done
