#!/bin/bash
# round-3 quick check: head/edge parity tests + c5 and c3 score pass (5 steps), optional env per run
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu -k "head_heavy or map_count" > $OUT/edges.log 2>&1; echo "edges $?" >> $OUT/status
B="--also none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
for c in ${CONFIGS:-c5 c3}; do
  timeout 600 python bench.py --config $c $B > $OUT/${c}.json 2> $OUT/${c}.err; echo "$c $?" >> $OUT/status
done
cat $OUT/status
