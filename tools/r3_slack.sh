#!/bin/bash
# round-3: tile slack (in-place merges) — the whole -m gpu suite (not slow), then configs 4 and 5
TAG=${1:-sl}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" > $OUT/gpu.log 2>&1; echo "gpu $?" >> $OUT/status
timeout 900 python bench.py --config c4 --no-cpu-baseline > $OUT/c4.json 2> $OUT/c4.err; echo "c4 $?" >> $OUT/status
timeout 600 python bench.py --config c5 --also none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/c5.json 2> $OUT/c5.err; echo "c5 $?" >> $OUT/status
cat $OUT/status
