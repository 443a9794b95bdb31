#!/bin/bash
# isolated curves + one ncu --set full capture per kernel
cd "$(dirname "$0")/.."
timeout 300 python scripts/microbench.py --kernel both --budgets 16,37,74,111,148 > gpurun_out/micro.jsonl 2> gpurun_out/micro.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_bf16 -s 2 -c 1 -o gpurun_out/prof_decode python scripts/microbench.py --kernel decode --budgets 74 --iters 3 > gpurun_out/ncu_dec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 2 -c 1 -o gpurun_out/prof_prefill python scripts/microbench.py --kernel prefill --budgets 74 --iters 3 > gpurun_out/ncu_pre.log 2>&1
ls -la gpurun_out
