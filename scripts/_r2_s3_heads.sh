cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_mla_expanded.py -q > gpurun_out/s3h_test.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/s3h_test.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_mla_expanded.py -q -x -k "head_counts or bad_block or too_small or (parity and FLAT) or (parity and 0-chunks2)" > gpurun_out/s3h_memcheck.log 2>&1; echo "memcheck rc $?"; tail -5 gpurun_out/s3h_memcheck.log
