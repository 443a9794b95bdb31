cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python bench.py > gpurun_out/s3b2_bench.json 2> gpurun_out/s3b2_bench.err; echo "bench rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_bf16|decode_pair|prefill_tc|alloc_kernel|free_kernel" -c 300 --csv --log-file gpurun_out/s3b2_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-secondary --no-extra --sweep 40 > gpurun_out/s3b2_ncu.log 2>&1; echo "ncu rc $?"
