set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity_large.py tests/test_gpu_peer_gather.py tests/test_gpu_rope.py -x -q -m gpu > gpurun_out/r2_t1.log 2>&1; echo "pytest rc $?"
timeout 900 python bench.py > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo "bench rc $?"
tail -5 gpurun_out/r2_t1.log
