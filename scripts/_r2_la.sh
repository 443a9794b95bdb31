cd /root/repo
SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_la1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py tests/test_gpu_rope_fused.py -q -x -k "mla" -p no:cacheprovider > gpurun_out/la_tests.log 2>&1; echo "la1 tests: $(tail -1 gpurun_out/la_tests.log)"
for rep in 1 2; do for t in la0 la1; do
  echo "== $t"
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla --ctx-lognormal --lpt --budgets 44,104,148 --batch 256 --ctx 350 --layers 8 2>&1 | tail -3
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla --budgets 104,148 --batch 256 --ctx 1000 --layers 4 2>&1 | tail -2
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla --budgets 148 --batch 64 --ctx 4000 --layers 4 2>&1 | tail -1
done; done
