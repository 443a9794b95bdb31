#!/bin/bash
# one ncu --set full capture per kernel at a given budget (default 74)
cd "$(dirname "$0")/.."
B=${1:-74}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_bf16 -s 2 -c 1 -o gpurun_out/prof_decode python scripts/microbench.py --kernel decode --budgets $B --iters 3 > gpurun_out/ncu_dec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 2 -c 1 -o gpurun_out/prof_prefill python scripts/microbench.py --kernel prefill --budgets $B --iters 3 > gpurun_out/ncu_pre.log 2>&1
ls gpurun_out
