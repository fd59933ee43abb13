#!/bin/bash
OUT=gpurun_out/pc2; mkdir -p $OUT
A="--config c2 --also none --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 2"
timeout 600 python bench.py $A > $OUT/plain.json 2> $OUT/plain.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_doc_score -s 5 -c 1 \
   -o $OUT/prof python bench.py $A > $OUT/ncu.log 2>&1; echo "ncu $?" >> $OUT/status
cat $OUT/status
