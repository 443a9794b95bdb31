set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc $?"
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc $?"
tail -3 gpurun_out/r2_gputest.log
