#!/bin/bash
# quick per-config bench, c2 twice (noise check): bash tools/quick2.sh <tag>
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c2a.json 2>/dev/null
timeout 600 python bench.py --config c3 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c3_1M.json 2>/dev/null
timeout 600 python bench.py --config c5 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/c5_1M.json 2>/dev/null
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c2b.json 2>/dev/null
for f in c3_1M c5_1M c2a c2b; do python -c "
import json; d=json.load(open('$OUT/$f.json')); print('$f', round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
