cd /root/repo
for t in p00 p10 p01 p11; do
  echo "== $t"
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "prefill_mla" -p no:cacheprovider > gpurun_out/mlap_$t.log 2>&1; tail -1 gpurun_out/mlap_$t.log
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla-prefill --budgets 44,104,148 --layers 4 2>&1 | tail -3
done
for t in p00 p11 p10 p01; do
  echo "== $t"
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla-prefill --budgets 104,148 --layers 4 2>&1 | tail -2
done
