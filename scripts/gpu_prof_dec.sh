#!/bin/bash
# ncu --set full of the cfg2 decode kernel (bs 64 pages -> head-pair kernel) at budget $1
cd "$(dirname "$0")/.."
B=${1:-89}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_ -s 2 -c 1 -o gpurun_out/prof_dec python scripts/microbench.py --kernel decode --budgets $B --iters 3 --bs 64 > gpurun_out/ncu_dec.log 2>&1
