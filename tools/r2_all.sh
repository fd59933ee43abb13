#!/bin/bash
# the driver's round-end GPU checks: smoke, the whole -m gpu suite (slow full-size tests included), the default bench
TAG=${1:-all}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke $?" >> $OUT/status
timeout 3600 python -m pytest tests -q -m gpu > $OUT/gpu.log 2>&1; echo "gpu $?" >> $OUT/status
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench $?" >> $OUT/status
cat $OUT/status
