cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "mla or prefill" > gpurun_out/s3d_test.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/s3d_test.log
for v in old new; do
  if [ $v = new ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_old.so; fi
  echo "== $v"
  timeout 300 python scripts/microbench.py --kernel prefill --budgets 59,148 --bs 64 2>&1 | grep -v "^$"
  timeout 300 python scripts/microbench.py --mla --ctx 350 --ctx-lognormal --lpt --batch 256 --budgets 44,104,148 2>&1 | grep -v "^$"
  timeout 300 python scripts/microbench.py --mla --ctx 4000 --batch 64 --budgets 104,148 2>&1 | grep -v "^$"
  timeout 300 python scripts/microbench.py --mla-prefill --budgets 104,148 --layers 4 2>&1 | grep -v "^$"
done
