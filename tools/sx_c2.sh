#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
for x in 80 96 128 160; do
SINN_SAMPLE_X=$x timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $OUT/c2_$x.json 2>/dev/null
done
for f in $OUT/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('/')[-1], round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
