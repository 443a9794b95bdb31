cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3t_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_trace.py -q -x > gpurun_out/s3t_tests.log 2>&1; echo "engine tests rc $?"; tail -2 gpurun_out/s3t_tests.log
timeout 1200 python scripts/mla_trace.py --requests 2000 --layers 27 --expanded --out gpurun_out/s3t_trace_expanded.json > gpurun_out/s3t_trace_expanded.log 2>&1; echo "trace rc $?"
tail -1 gpurun_out/s3t_trace_expanded.log
timeout 1500 python scripts/bench_field.py cfg5_mla_expanded > gpurun_out/s3t_field.jsonl 2> gpurun_out/s3t_field.err; echo "field rc $?"
