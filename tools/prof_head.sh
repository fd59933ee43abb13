#!/bin/bash
# c3 law at 1M documents: head split on/off, then one ncu capture of the main head-scoring pass.
OUT=gpurun_out/ph; mkdir -p $OUT
A="--config c3 --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2"
SINN_DEBUG=1 SINN_HEAD=1 timeout 600 python bench.py $A > $OUT/h1.json 2> $OUT/h1.err; echo "h1 $?" >> $OUT/status
SINN_HEAD=0 timeout 600 python bench.py $A > $OUT/h0.json 2> $OUT/h0.err; echo "h0 $?" >> $OUT/status
SINN_HEAD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_head_score -s 5 -c 1 \
   -o $OUT/prof python bench.py $A > $OUT/ncu.log 2>&1; echo "ncu $?" >> $OUT/status
cat $OUT/status
