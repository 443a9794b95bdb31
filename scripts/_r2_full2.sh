cd /root/repo
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc $?"
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/r2g_gputest.log 2>&1; echo "pytest rc $?"
timeout 900 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc $?"
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2g_ref.json 2>&1; echo "ref rc $?"
tail -2 gpurun_out/r2g_gputest.log
