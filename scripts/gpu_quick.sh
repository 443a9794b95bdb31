#!/bin/bash
# quick dev loop on the box: prefill parity subset + isolated prefill curve points
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" 2>&1 | tail -3
timeout 300 python scripts/microbench.py --kernel prefill --bs 64 --iters 15 --budgets 40,59,74,100,148 2>&1 | tail -5
