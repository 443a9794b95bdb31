cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py tests/test_gpu_rope_fused.py -q -x -k "mla" -p no:cacheprovider > gpurun_out/mlad_tests.log 2>&1; tail -1 gpurun_out/mlad_tests.log
for rep in 1 2; do
timeout 300 python scripts/microbench.py --mla --budgets 44,104,148 --batch 256 --ctx 350 --layers 8 2>&1 | tail -3
timeout 300 python scripts/microbench.py --mla --budgets 74,148 --batch 256 --ctx 1000 --layers 4 2>&1 | tail -2
timeout 300 python scripts/microbench.py --mla --budgets 148 --batch 64 --ctx 4000 --layers 4 2>&1 | tail -1
done
