#!/bin/bash
# FP8 decode: code -> f16 conversion pipe split A/B (SPD_F8_KALU / SPD_F8_VALU), parity + timing
cd "$(dirname "$0")/.."
for v in k0v1 k1v0 k1v1 k0v0; do
  echo "== $v"
  SEMIPD_LIB=paper_2504_19867_b200/libsemipd_v_$v.so timeout 600 python -m pytest tests/test_gpu_fp8.py -q -x -m gpu -k "decode_parity or scales or gqa" 2>&1 | tail -1
done
for rep in 1 2; do
for v in k0v0 k0v1 k1v0 k1v1; do
  echo "== $v"
  SEMIPD_LIB=paper_2504_19867_b200/libsemipd_v_$v.so timeout 300 python scripts/microbench.py --kernel decode --bs 64 --budgets 44,89,148 --iters 20 --layers 8 --fp8 2>&1 | grep '^{'
done
done
