#!/bin/bash
# round-3: bulk-copy (TMA) column staging — parity (edges + parity suites, not slow) and A/B vs cp.async
TAG=${1:-tma}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" > $OUT/gpu.log 2>&1; echo "gpu $?" >> $OUT/status
B="--also none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
for c in c5 c2 c3; do
  for t in 1 0; do
    SINN_TMA=$t timeout 600 python bench.py --config $c $B > $OUT/${c}_tma$t.json 2> $OUT/${c}_tma$t.err; echo "$c tma$t $?" >> $OUT/status
  done
done
cat $OUT/status
