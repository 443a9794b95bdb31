#!/bin/bash
# re-measure with back-to-back launch timing: isolated curves, uniform-ctx decode, MLA micro,
# MLA prefill micro, and ncu --set full of the cfg2 prefill / decode kernels at the bench split
cd "$(dirname "$0")/.."
bash scripts/gpu_curves.sh
timeout 300 python scripts/microbench.py --mla --budgets 37,74,148 --batch 256 --ctx 1000 --layers 4 > gpurun_out/mla.jsonl 2>&1
timeout 300 python scripts/microbench.py --mla --budgets 74,148 --batch 64 --ctx 4000 --layers 4 >> gpurun_out/mla.jsonl 2>&1
timeout 300 python scripts/microbench.py --mla-prefill --budgets 74,148 --chunk 2048 --layers 4 >> gpurun_out/mla.jsonl 2>&1
bash scripts/gpu_prof.sh 59 89
python scripts/ncu_summary.py gpurun_out/prof_prefill.ncu-rep 20 > gpurun_out/ncu_prefill_summary.txt 2>&1
python scripts/ncu_summary.py gpurun_out/prof_decode.ncu-rep 20 > gpurun_out/ncu_decode_summary.txt 2>&1
ls gpurun_out
