cd /root/repo
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc $?"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2f_gputest.log 2>&1; echo "pytest rc $?"
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc $?"
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2f_ref.json 2>&1; echo "ref rc $?"
tail -2 gpurun_out/r2f_gputest.log
