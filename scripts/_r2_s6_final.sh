cd /root/repo
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s6_smoke.log 2>&1; echo "smoke rc $?"
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/s6_gputest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/s6_gputest.log
