cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_rope_fused.py tests/test_gpu_parity_large.py -q -x -k "not cfg4 and not bench_config" -p no:cacheprovider > gpurun_out/r2_memcheck.log 2>&1; echo "memcheck rc $?"
tail -5 gpurun_out/r2_memcheck.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "mla or block_sizes" -p no:cacheprovider > gpurun_out/r2_memcheck_mla.log 2>&1; echo "memcheck2 rc $?"
tail -5 gpurun_out/r2_memcheck_mla.log
