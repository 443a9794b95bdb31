cd /root/repo
for t in c1 c0; do
  echo "== $t"
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py tests/test_gpu_rope_fused.py -q -x -k "decode and not mla" -p no:cacheprovider > gpurun_out/bs16_$t.log 2>&1; tail -1 gpurun_out/bs16_$t.log
done
for rep in 1 2; do for t in c0 c1; do
  echo "== $t"
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --kernel decode --bs 16 --budgets 44,89,104,148 --layers 8 2>&1 | tail -4
done; done
