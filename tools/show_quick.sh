#!/bin/bash
# summarise tools/gpu_quick.sh output: bash tools/show_quick.sh <tag>
cat gpurun_out/$1/status; tail -1 gpurun_out/$1/pytest.log
for f in c3_1M c5_1M c2; do python -c "
import json; d=json.load(open('gpurun_out/$1/$f.json')); print('$f', round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
