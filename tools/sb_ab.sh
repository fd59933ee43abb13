#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
for sb in 0 1; do
SINN_SINGLE_BUF=$sb timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c2_sb$sb.json 2>/dev/null
SINN_SINGLE_BUF=$sb timeout 600 python bench.py --config c3 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c3_sb$sb.json 2>/dev/null
done
for f in c2_sb0 c2_sb1 c3_sb0 c3_sb1; do python -c "
import json; d=json.load(open('$OUT/$f.json')); print('$f', round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
