cd /root/repo
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo "smoke rc $?"
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/s3_gputest.log 2>&1; echo "pytest rc $?"
timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo "bench rc $?"
tail -3 gpurun_out/s3_gputest.log
