#!/bin/bash
# FP8 decode with guided split pieces: parity, then isolated timing over SM budgets
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fp8.py -q -x -m gpu -k decode 2>&1 | tail -2
timeout 600 python scripts/microbench.py --kernel decode --bs 64 --budgets 44,59,67,74,81,89,96,104,148 --iters 20 --layers 8 --fp8 2>&1 | grep '^{'
timeout 600 python scripts/microbench.py --kernel decode --bs 64 --budgets 89,148 --iters 20 --layers 8 --fp8 --ctx-uniform 64,512 2>&1 | grep '^{'
timeout 600 python scripts/microbench.py --kernel decode --bs 64 --budgets 89,148 --iters 20 --layers 8 --ctx-uniform 64,512 2>&1 | grep '^{'
