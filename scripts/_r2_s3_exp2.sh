cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3e_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_mla_expanded.py -q > gpurun_out/s3e_test.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/s3e_test.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_exp -c 3 -o gpurun_out/s3_ncu_mlaexp python scripts/microbench.py --mla-exp --budgets 104 --layers 1 --iters 1 > gpurun_out/s3e_ncu.log 2>&1; echo "ncu rc $?"
