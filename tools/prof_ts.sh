#!/bin/bash
# ncu capture of k_ts_score (EMIT) on a config at reduced size: bash tools/prof_ts.sh <tag> <config> <docs>
TAG=${1:-pts}; CFG=${2:-c5}; DOCS=${3:-500000}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
ARGS="--config $CFG --also none --docs $DOCS --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 600 python bench.py $ARGS > $OUT/plain.json 2> $OUT/plain.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ts_score -s 4 -c 1 \
   -o $OUT/prof python bench.py $ARGS > $OUT/ncu.log 2>&1; echo "ncu $?" >> $OUT/status
cat $OUT/status
