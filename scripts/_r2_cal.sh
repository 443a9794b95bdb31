cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --no-secondary --no-cpu --no-e2e > gpurun_out/r2_cal.json 2> gpurun_out/r2_cal.err; echo "rc $?"
tail -3 gpurun_out/r2_cal.err
