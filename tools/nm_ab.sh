#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
cp paper_2301_10622_b200/libsinn.so /tmp/libsinn_base.so
for v in 5 12 base; do
  if [ "$v" = base ]; then cp /tmp/libsinn_base.so paper_2301_10622_b200/libsinn.so; else cp nmtest/libsinn_$v.so paper_2301_10622_b200/libsinn.so; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $OUT/c2_$v.json 2>/dev/null
  timeout 600 python bench.py --config c3 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c3_$v.json 2>/dev/null
  timeout 600 python bench.py --config c5 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c5_$v.json 2>/dev/null
done
for f in $OUT/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('/')[-1], round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
