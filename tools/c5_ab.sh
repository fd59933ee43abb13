#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
A="--config c5 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2"
timeout 600 python bench.py $A > $OUT/f32.json 2>/dev/null
timeout 600 python bench.py $A --bf16 > $OUT/bf16.json 2>/dev/null
SINN_SINGLE_BUF=0 timeout 600 python bench.py $A --bf16 > $OUT/bf16_sb0.json 2>/dev/null
SINN_SINGLE_BUF=0 timeout 600 python bench.py $A > $OUT/f32_sb0.json 2>/dev/null
for f in f32 bf16 bf16_sb0 f32_sb0; do python -c "
import json; d=json.load(open('$OUT/$f.json')); print('$f', round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
