#!/bin/bash
# k_ts_score check: its parity tests, then short config-5 and config-3 bench lines
TAG=${1:-ts}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu -k "head_heavy" > $OUT/ts_tests.log 2>&1; echo "ts_tests $?" >> $OUT/status
timeout 900 python bench.py --config c5 --also c3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/bench.json 2> $OUT/bench.err; echo "bench $?" >> $OUT/status
cat $OUT/status
