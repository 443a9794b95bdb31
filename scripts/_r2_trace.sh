cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python scripts/mla_trace.py --requests 2000 --layers 27 --out gpurun_out/r2_mla_trace.json > gpurun_out/r2_mla_trace.log 2>&1; echo "trace rc $?"
tail -1 gpurun_out/r2_mla_trace.log | cut -c1-1500
