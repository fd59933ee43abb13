#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
for cap in ${CAPS:-65536 131072}; do
for c in c3 c5; do
SINN_CAND_CAP=$cap timeout 900 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 2 > $OUT/${c}_$cap.json 2>/dev/null
done; done
for f in $OUT/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('/')[-1], round(d['value']), round(d['ms_per_step'],3), d.get('recall@10', d.get('recall@100')), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
