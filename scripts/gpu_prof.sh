#!/bin/bash
# one ncu --set full capture per cfg2 kernel, bench shapes (bs 64 pages), at the bench's best
# split budgets (default prefill 59, decode 89)
cd "$(dirname "$0")/.."
BP=${1:-59}
BD=${2:-89}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_ -s 2 -c 1 -o gpurun_out/prof_decode python scripts/microbench.py --kernel decode --budgets $BD --iters 3 --bs 64 > gpurun_out/ncu_dec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 2 -c 1 -o gpurun_out/prof_prefill python scripts/microbench.py --kernel prefill --budgets $BP --iters 3 --bs 64 > gpurun_out/ncu_pre.log 2>&1
ls gpurun_out
