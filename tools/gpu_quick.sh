#!/bin/bash
# GPU parity tests + quick per-config bench: bash tools/gpu_quick.sh <tag>
TAG=${1:-q}
mkdir -p gpurun_out/$TAG
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest $?" > gpurun_out/$TAG/status
bash tools/quick_cfg.sh $TAG
