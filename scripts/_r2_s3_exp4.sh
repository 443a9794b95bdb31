cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3e4_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_mla_expanded.py -q -x > gpurun_out/s3e4_test.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/s3e4_test.log
timeout 300 python scripts/microbench.py --mla-exp --budgets 44,74,104,148 --layers 4 > gpurun_out/s3e4_micro.jsonl 2>&1
timeout 300 python scripts/microbench.py --mla-exp --budgets 44,74,148 --layers 4 --prefix 4096 >> gpurun_out/s3e4_micro.jsonl 2>&1
cat gpurun_out/s3e4_micro.jsonl
