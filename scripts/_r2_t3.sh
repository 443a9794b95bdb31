python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_controller_loop.py tests/test_gpu_multi_nccl.py -x -q -s > gpurun_out/r2_ctl.log 2>&1; echo "ctl rc $?"
tail -5 gpurun_out/r2_ctl.log
