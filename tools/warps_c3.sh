#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
for w in 20 24 28 32; do
SINN_DOC_WARPS=$w timeout 600 python bench.py --config c3 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c3_w$w.json 2>/dev/null
SINN_DOC_WARPS=$w timeout 600 python bench.py --config c5 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c5_w$w.json 2>/dev/null
done
for f in $OUT/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('/')[-1], round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
