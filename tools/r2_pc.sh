#!/bin/bash
# pair-cache A/B: parity on the head-heavy laws, then config 5 and 3 lines per cache size
TAG=${1:-pc}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" -k "config_parity or head_heavy or constrained or per_query or exact" > $OUT/tests.log 2>&1; echo "tests $?" >> $OUT/status
for pc in 0 2048 4096 8192; do
  SINN_PCACHE=$pc timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/b_$pc.json 2>> $OUT/bench.err; echo "pc $pc $?" >> $OUT/status
done
cat $OUT/status
