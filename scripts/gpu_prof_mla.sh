#!/bin/bash
# ncu capture of the MLA decode kernel + isolated curves.  Usage: gpu_prof_mla.sh [ctx] [batch]
cd "$(dirname "$0")/.."
CTX=${1:-1000}
B=${2:-256}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mla -s 2 -c 1 -o gpurun_out/prof_mla python scripts/microbench.py --mla --budgets 148 --batch $B --ctx $CTX --iters 3 --layers 2 > gpurun_out/ncu_mla.log 2>&1
timeout 300 python scripts/microbench.py --mla --budgets 37,74,148 --batch $B --ctx $CTX --layers 4 > gpurun_out/mla.jsonl 2>&1
timeout 300 python scripts/microbench.py --mla --budgets 74,148 --batch 256 --ctx 1024 --layers 4 >> gpurun_out/mla.jsonl 2>&1
timeout 300 python scripts/microbench.py --mla --budgets 74,148 --batch 64 --ctx 4000 --layers 4 >> gpurun_out/mla.jsonl 2>&1
