#!/bin/bash
# round-2 (session 4): ncu capture of the fused validate + sketch-build kernel (config 5 rows)
TAG=${1:-skp}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
A="--config c5 --docs 1000000 --also none --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sketch_build -s 4 -c 1 \
   -o $OUT/prof_sk python bench.py $A > $OUT/ncu.log 2>&1; echo "ncu $?" >> $OUT/status
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raw_append -s 4 -c 1 \
   -o $OUT/prof_raw python bench.py $A > $OUT/ncu2.log 2>&1; echo "ncu2 $?" >> $OUT/status
cat $OUT/status
