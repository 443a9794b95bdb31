cd /root/repo
for t in c36 c2 c4 c8 c36; do
  echo "== $t"
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla --budgets 74,148 --batch 256 --ctx 1000 --layers 4 2>&1 | tail -2
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla --budgets 148 --batch 64 --ctx 4000 --layers 4 2>&1 | tail -1
done
for t in c4; do
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mla" 2>&1 | tail -1
done
