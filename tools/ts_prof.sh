#!/bin/bash
# k_ts_score phase clocks (SINN_TS_PROF=1): bash tools/ts_prof.sh <tag>
TAG=${1:-tsp}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for CFG in c5 c3; do
  SINN_TS_PROF=1 timeout 600 python bench.py --config $CFG --also none --docs 1000000 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/b_$CFG.json 2> $OUT/prof_$CFG.txt
  echo "$CFG $?" >> $OUT/status
done
cat $OUT/status
