cd /root/repo
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3z_smoke.log 2>&1; echo "smoke rc $?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s3z_gputest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/s3z_gputest.log
timeout 1500 python bench.py > gpurun_out/s3z_bench.json 2> gpurun_out/s3z_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s3z_ref.json 2>&1; echo "ref rc $?"
