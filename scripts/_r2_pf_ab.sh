cd /root/repo
for t in v4; do
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "decode" -p no:cacheprovider > gpurun_out/pf_$t.log 2>&1; echo "$t tests: $(tail -1 gpurun_out/pf_$t.log)"
done
for rep in 1 2; do for t in v0 v2 v4; do
  echo "== $t"
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --kernel decode --bs 16 --budgets 89,104,148 --layers 8 2>&1 | tail -3
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --kernel decode --bs 64 --budgets 89,148 --layers 8 2>&1 | tail -2
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla --budgets 104,148 --batch 256 --ctx 350 --layers 8 2>&1 | tail -2
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla --budgets 148 --batch 64 --ctx 4000 --layers 4 2>&1 | tail -1
done; done
