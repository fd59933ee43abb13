#!/bin/bash
# round-3: c2-path change check — the -m gpu suite (not slow), then c2 / tiny / c4 / c5 lines
TAG=${1:-c2x}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" > $OUT/gpu.log 2>&1; echo "gpu $?" >> $OUT/status
B="--also none --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1"
for c in c2 tiny c5; do timeout 600 python bench.py --config $c $B > $OUT/$c.json 2> $OUT/$c.err; echo "$c $?" >> $OUT/status; done
timeout 900 python bench.py --config c4 --no-cpu-baseline > $OUT/c4.json 2> $OUT/c4.err; echo "c4 $?" >> $OUT/status
cat $OUT/status
