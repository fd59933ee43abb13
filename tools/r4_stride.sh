#!/bin/bash
# round-2 (session 4): sample-stride sweep with the sampled rows reused by the full pass
TAG=${1:-stride}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="--also none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
run() { # name config env...
  n=$1; c=$2; shift 2
  env "$@" timeout 600 python bench.py --config $c $B > $OUT/$n.json 2> $OUT/$n.err
  python - <<PY
import json
try:
    d=json.loads(open("$OUT/$n.json").read().strip().splitlines()[-1])
    print("$n", round(d["value"]), round(d["ms_per_step"],2), {k:round(v["ms_per_step"],2) for k,v in d["kernels"].items()}, d["recall"]["vs_gpu_exact"])
except Exception as e: print("$n", "ERR", e)
PY
}
run c5_x64 c5 SINN_SAMPLE_X=64
run c5_x128 c5 SINN_SAMPLE_X=128
run c5_x256 c5 SINN_SAMPLE_X=256
run c3_cap57k c3 SINN_CAND_CAP=57344
run c3_cap28k c3 SINN_CAND_CAP=28672
