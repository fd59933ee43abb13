#!/bin/bash
# the whole -m gpu suite (slow full-size sampled parity included) + smoke
TAG=${1:-ft}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 3000 python -m pytest tests -q -m gpu > $OUT/gpu_all.log 2>&1; echo "gpu_all $?" >> $OUT/status
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke $?" >> $OUT/status
cat $OUT/status
