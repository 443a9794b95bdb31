python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_rope_fused.py -x -q > gpurun_out/r2_rope_fused.log 2>&1; echo "rope rc $?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest_all.log 2>&1; echo "all rc $?"
tail -3 gpurun_out/r2_rope_fused.log gpurun_out/r2_gputest_all.log
