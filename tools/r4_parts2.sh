#!/bin/bash
TAG=${1:-parts2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -x -q -m "gpu and not slow" -k "head_heavy or sample_rows or config_parity" > $OUT/t.log 2>&1; echo "tests $?" >> $OUT/status
B="--also none --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1"
for c in c5 c3 c2; do
  timeout 600 python bench.py --config $c $B > $OUT/$c.json 2> $OUT/$c.err
  python - <<PY
import json
try:
    d=json.loads(open("$OUT/$c.json").read().strip().splitlines()[-1])
    print("$c", round(d["value"]), round(d["ms_per_step"],2), {k:round(v["ms_per_step"],2) for k,v in d["kernels"].items()}, d["recall"]["vs_gpu_exact"])
except Exception as e: print("$c", "ERR", e)
PY
done
tail -2 $OUT/t.log; cat $OUT/status
