#!/bin/bash
# round-2 (session 4): sampled rows reused by the full pass — forced-path parity, head tests, full-size sampled
# parity of configs 3/5, then the c5 / c3 lines with the rows on and off
TAG=${1:-rows}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu -k "sample_rows or head_heavy or shortfall" > $OUT/edges.log 2>&1; echo "edges $?" >> $OUT/status
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full" > $OUT/full.log 2>&1; echo "full $?" >> $OUT/status
B="--also none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
for c in c5 c3; do
  timeout 600 python bench.py --config $c $B > $OUT/${c}.json 2> $OUT/${c}.err; echo "$c $?" >> $OUT/status
  SINN_ROWS=0 timeout 600 python bench.py --config $c $B > $OUT/${c}_off.json 2> $OUT/${c}_off.err; echo "${c}_off $?" >> $OUT/status
done
python - <<PY
import json
for f in ("c5","c5_off","c3","c3_off"):
    try:
        d=json.loads(open("$OUT/%s.json"%f).read().strip().splitlines()[-1])
        print(f, round(d["value"]), round(d["ms_per_step"],2), {k:round(v["ms_per_step"],2) for k,v in d["kernels"].items()}, d["recall"]["vs_gpu_exact"])
    except Exception as e: print(f, "ERR", e)
PY
tail -3 $OUT/edges.log $OUT/full.log
cat $OUT/status
