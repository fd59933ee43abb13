#!/bin/bash
# One gpurun session: GPU parity tests, the default bench line, the ncu launch list and one
# full ncu capture of the top kernel.  Usage (from the repo root, on the GPU box):
#   bash tools/gpu_check.sh <tag> [bench args...]
set -u
TAG=${1:-run}; shift || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/status
timeout 900 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/status
NCUARGS="--steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 $*"
timeout 600 python bench.py $NCUARGS > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
   --log-file $OUT/launches.csv python bench.py $NCUARGS > $OUT/ncu_launch.log 2>&1; echo "ncu-launch exit $?" >> $OUT/status
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_tile_score} -s ${KSKIP:-4} -c ${KCOUNT:-2} \
   -o $OUT/prof python bench.py $NCUARGS > $OUT/ncu_full.log 2>&1; echo "ncu-full exit $?" >> $OUT/status
cat $OUT/status
