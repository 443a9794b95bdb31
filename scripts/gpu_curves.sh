#!/bin/bash
# isolated per-budget curves (every budget 8..148 step 4), cfg2 bench
# shapes (bs 64), plus the load-balance decode shape (ctx ~ U[1024, 3072], item 7)
cd "$(dirname "$0")/.."
timeout 900 python scripts/microbench.py --kernel both --bs 64 --iters 15 --budgets 8,12,16,20,24,28,32,36,40,44,48,52,56,60,64,68,72,76,80,84,88,92,96,100,104,108,112,116,120,124,128,132,136,140,144,148 > gpurun_out/curves.jsonl 2>&1
timeout 300 python scripts/microbench.py --kernel decode --bs 64 --ctx-uniform 1024,3072 --budgets 59,74,89,148 > gpurun_out/curves_uniform.jsonl 2>&1
