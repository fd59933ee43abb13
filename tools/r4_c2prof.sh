#!/bin/bash
# round-2 (session 4): full ncu capture of the config-2 EMIT pass + per-line L1 wavefront summary
TAG=${1:-c2p}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
A="--config c2 --also none --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 python bench.py $A > $OUT/c2.json 2> $OUT/c2.err; echo "c2 $?" >> $OUT/status
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_doc_score -s 5 -c 1 \
   -o $OUT/prof_c2 python bench.py $A > $OUT/ncu_c2.log 2>&1; echo "ncu_c2 $?" >> $OUT/status
python tools/ncu_smem.py $OUT/prof_c2.ncu-rep 40 > $OUT/c2_smem_lines.txt 2>&1
python tools/ncu_top.py $OUT/prof_c2.ncu-rep > $OUT/c2_top.txt 2>&1
cat $OUT/status
