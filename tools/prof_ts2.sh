#!/bin/bash
# ncu captures of k_ts_score (the EMIT pass) for configs 5 and 3 at 500K documents
TAG=${1:-pts}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for CFG in c5 c3; do
  ARGS="--config $CFG --also none --docs 500000 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
  timeout 600 python bench.py $ARGS > $OUT/plain_$CFG.json 2> $OUT/plain_$CFG.err && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ts_score -s 3 -c 1 \
     -o $OUT/prof_$CFG python bench.py $ARGS > $OUT/ncu_$CFG.log 2>&1; echo "ncu $CFG $?" >> $OUT/status
done
cat $OUT/status
