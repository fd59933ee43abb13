#!/bin/bash
# round-3: bitmap containers — their parity tests, the edge suite, c5/c3 with and without containers
TAG=${1:-cont}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_containers.py -x -q -m gpu > $OUT/cont.log 2>&1; echo "cont $?" >> $OUT/status
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu > $OUT/edges.log 2>&1; echo "edges $?" >> $OUT/status
B="--also none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
for c in c5 c3; do
  timeout 600 python bench.py --config $c $B > $OUT/${c}.json 2> $OUT/${c}.err; echo "$c $?" >> $OUT/status
  timeout 600 python bench.py --config $c $B --containers > $OUT/${c}_cont.json 2> $OUT/${c}_cont.err; echo "$c cont $?" >> $OUT/status
done
cat $OUT/status
