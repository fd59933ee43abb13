#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest $?" > $OUT/status
for cs in 0 1; do for c in c3 c5; do
SINN_CASCADE=$cs timeout 900 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 2 > $OUT/${c}_cas$cs.json 2>/dev/null
done; done
SINN_CASCADE=1 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $OUT/c2_cas1.json 2>/dev/null
SINN_CASCADE=0 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $OUT/c2_cas0.json 2>/dev/null
cat $OUT/status; tail -1 $OUT/pytest.log
for f in $OUT/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('/')[-1], round(d['value']), round(d['ms_per_step'],3), d.get('recall@10', d.get('recall@100')), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
