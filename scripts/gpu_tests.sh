#!/bin/bash
# Run GPU test groups with hard timeouts; logs to gpurun_out/
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
for grp in "$@"; do
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$grp" --timeout 150 -x -p no:cacheprovider > gpurun_out/test_${grp// /_}.log 2>&1
  echo "group '$grp' exit $?" >> gpurun_out/summary.txt
done
tail -3 gpurun_out/test_*.log
