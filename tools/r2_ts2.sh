#!/bin/bash
# k_ts_score variants: parity (head-heavy tests) and short c5 / c3 bench lines per variant
TAG=${1:-ts2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SINN_TS_WMIN=100000 timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu -k "head_heavy and (ts-c or ts_spill)" > $OUT/ts_tests.log 2>&1; echo "ts_tests $?" >> $OUT/status
for v in "SINN_TS_WMIN=100000" "SINN_TS=0" "SINN_TS_WMIN=100000 SINN_TS_TAU=0.15"; do
  env $v timeout 900 python bench.py --config c5 --also c3 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_$(echo $v | tr ' =' '__').json 2>> $OUT/bench.err; echo "bench $v $?" >> $OUT/status
done
cat $OUT/status
