#!/bin/bash
# Bench lines for every BASELINE.json config on one GPU (evidence for profiles/).
#   bash tools/gpu_configs.sh <tag> [configs...]
set -u
TAG=${1:-cfg}; shift || true
CFGS=${*:-"tiny c3 c5 c4"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
free -g > $OUT/host.txt; nproc >> $OUT/host.txt
for c in $CFGS; do
  extra=""
  case $c in c3|c5) extra="--no-cpu-baseline --steps 20 --warmup 3";; c4) extra="";; tiny) extra="--steps 50 --warmup 5";; esac
  timeout 1500 python bench.py --config $c $extra > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "$c exit $?" >> $OUT/status
done
cat $OUT/status
