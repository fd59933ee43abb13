#!/bin/bash
# round-2 (session 4): insert-path change check — sketch parity tests + insert docs/s of configs 5, 2, 3
TAG=${1:-ins}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q -m "gpu and not slow" -k "config_parity or bf16 or map_count or stream or host_entry or edge" > $OUT/t.log 2>&1; echo "tests $?" >> $OUT/status
B="--also none --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
for c in ${CONFIGS:-c5 c2 c3}; do
  timeout 600 python bench.py --config $c $B > $OUT/${c}.json 2> $OUT/${c}.err; echo "$c $?" >> $OUT/status
  python - <<PY
import json
d=json.loads(open("$OUT/${c}.json").read().strip().splitlines()[-1])
print("$c insert", round(d["insert"]["value"]/1e6,1), "M docs/s frac", round(d["insert"]["roofline"]["frac"],4), d["insert"]["phases_ms"])
PY
done
tail -3 $OUT/t.log
cat $OUT/status
