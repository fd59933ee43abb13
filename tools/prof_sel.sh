#!/bin/bash
OUT=gpurun_out/psel; mkdir -p $OUT
A="--steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2"
timeout 600 python bench.py $A > $OUT/plain.json 2> $OUT/plain.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cand_select|k_rerank|k_theta|k_final" -s 8 -c 4 \
   -o $OUT/prof python bench.py $A > $OUT/ncu.log 2>&1; echo "ncu $?" >> $OUT/status
cat $OUT/status
