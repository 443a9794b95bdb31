cd /root/repo
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo "smoke rc $?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s4_gputest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/s4_gputest.log
timeout 1500 python bench.py > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err; echo "bench rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s4_launches.csv python bench.py --steps 1 --warmup 3 --split 30 --no-secondary --no-cpu --no-e2e --no-extra --sustained 0 > gpurun_out/s4_ncu.log 2>&1; echo "ncu rc $?"
