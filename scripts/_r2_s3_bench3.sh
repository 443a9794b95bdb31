cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python bench.py > gpurun_out/s3y_bench.json 2> gpurun_out/s3y_bench.err; echo "bench rc $?"
