#!/bin/bash
# round-3 A/B: c5 and c3 score pass under environment variants.  usage: bash tools/r3_ab.sh TAG "ENV1" "ENV2" ...
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu -k "head_heavy or map_count" > $OUT/edges.log 2>&1; echo "edges $?" >> $OUT/status
B="--also none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
i=0
for E in "$@"; do
  for c in ${CONFIGS:-c5 c3}; do
    env $E timeout 600 python bench.py --config $c $B > $OUT/${c}_v$i.json 2> $OUT/${c}_v$i.err; echo "$c v$i [$E] $?" >> $OUT/status
  done
  i=$((i+1))
done
cat $OUT/status
