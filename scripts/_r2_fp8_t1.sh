#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fp8_build.log 2>&1 || { tail -30 gpurun_out/fp8_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fp8.py -q -x -m gpu > gpurun_out/fp8_t1.log 2>&1
echo "fp8 tests rc $?"
tail -30 gpurun_out/fp8_t1.log
