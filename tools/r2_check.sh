#!/bin/bash
# round-2 GPU check: build, edge tests first, then the whole -m gpu suite (minus slow), then a short
# default bench line.  Usage: bash tools/r2_check.sh <tag>
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu > $OUT/edges.log 2>&1; echo "edges $?" >> $OUT/status
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" > $OUT/gpu.log 2>&1; echo "gpu $?" >> $OUT/status
timeout 900 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench $?" >> $OUT/status
cat $OUT/status
