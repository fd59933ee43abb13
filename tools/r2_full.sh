#!/bin/bash
# full GPU check: -m gpu (not slow), then bench lines: default (c5 + c3), c2 with/without the L2 window, c4
TAG=${1:-full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke $?" >> $OUT/status
timeout 1800 python -m pytest tests -x -q -m "gpu and not slow" > $OUT/gpu.log 2>&1; echo "gpu $?" >> $OUT/status
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench $?" >> $OUT/status
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/c2.json 2>> $OUT/bench.err; echo "c2 $?" >> $OUT/status
SINN_L2_PERSIST=0 timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/c2_nol2.json 2>> $OUT/bench.err; echo "c2nol2 $?" >> $OUT/status
timeout 1200 python bench.py --config c4 > $OUT/c4.json 2>> $OUT/bench.err; echo "c4 $?" >> $OUT/status
cat $OUT/status
