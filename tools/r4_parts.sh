#!/bin/bash
# round-2 (session 4): work-unit granularity of the full pass (tail of the dynamic schedule)
TAG=${1:-parts}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="--also none --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1"
run() { n=$1; c=$2; shift 2
  env "$@" timeout 600 python bench.py --config $c $B > $OUT/$n.json 2> $OUT/$n.err
  python - <<PY
import json
try:
    d=json.loads(open("$OUT/$n.json").read().strip().splitlines()[-1])
    print("$n", round(d["value"]), round(d["ms_per_step"],2), {k:round(v["ms_per_step"],2) for k,v in d["kernels"].items()}, d["recall"]["vs_gpu_exact"])
except Exception as e: print("$n", "ERR", e)
PY
}
run c5_p4 c5 SINN_PARTS_X=4
run c5_p40 c5 SINN_PARTS_X=40
run c5_p80 c5 SINN_PARTS_X=80
run c5_p160 c5 SINN_PARTS_X=160
run c3_p4 c3 SINN_PARTS_X=4
run c3_p100 c3 SINN_PARTS_X=100
