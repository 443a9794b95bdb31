cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --no-secondary --no-cpu > gpurun_out/r2_tail.json 2> gpurun_out/r2_tail.err; echo "rc $?"
tail -3 gpurun_out/r2_tail.err
