cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_nccl_graph.py -x -q > gpurun_out/r2_ncclg.log 2>&1; echo "rc $?"
tail -30 gpurun_out/r2_ncclg.log
