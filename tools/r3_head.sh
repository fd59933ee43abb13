#!/bin/bash
# round-3 A/B: TMEM head rows, head width 8 vs 16, head coverage threshold; plus the head parity tests
TAG=${1:-h}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu -k "head_heavy or map_count or enomem or poisons" > $OUT/edges.log 2>&1; echo "edges $?" >> $OUT/status
B="--also none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
for c in c5 c3; do
  for hw in 8 16; do
    SINN_HEAD_W=$hw timeout 600 python bench.py --config $c $B > $OUT/${c}_w$hw.json 2> $OUT/${c}_w$hw.err; echo "$c w$hw $?" >> $OUT/status
  done
done
for tau in 0.08 0.04; do
  SINN_HEAD_TAU=$tau timeout 600 python bench.py --config c5 $B > $OUT/c5_tau$tau.json 2> $OUT/c5_tau$tau.err; echo "c5 tau$tau $?" >> $OUT/status
done
cat $OUT/status
