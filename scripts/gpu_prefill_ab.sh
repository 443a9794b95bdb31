#!/bin/bash
# A/B of the prefill kernel with / without the compiled-in epilogue peer stores (n_peers = 0)
cd "$(dirname "$0")/.."
for rep in 1 2 3; do for t in nopeer peer; do
  echo "== $t"; SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 200 python scripts/microbench.py --kernel prefill --bs 64 --iters 15 --budgets 59,148 2>&1 | tail -2 | cut -c1-120
done; done
