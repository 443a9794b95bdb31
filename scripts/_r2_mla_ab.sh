cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rope_fused.py tests/test_gpu_parity_large.py -q -x -k "mla" > gpurun_out/mla_tests.log 2>&1; tail -2 gpurun_out/mla_tests.log
for rep in 1 2; do
for t in dq0 dq1; do
  echo "== $t"
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla --budgets 44,104,148 --batch 256 --ctx 350 --layers 8 2>&1 | tail -3
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla --budgets 74,148 --batch 256 --ctx 1000 --layers 4 2>&1 | tail -2
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 300 python scripts/microbench.py --mla --budgets 148 --batch 64 --ctx 4000 --layers 4 2>&1 | tail -1
done
done
