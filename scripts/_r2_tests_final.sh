cd /root/repo
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo "smoke rc $?"
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/r2j_gputest.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/r2j_gputest.log
