cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/microbench.py --mla-exp --budgets 44,74,104,148 --layers 4 > gpurun_out/s3c_micro.jsonl 2>&1
timeout 300 python scripts/microbench.py --mla-exp --budgets 44,74,148 --layers 4 --prefix 4096 >> gpurun_out/s3c_micro.jsonl 2>&1
timeout 1500 python scripts/bench_field.py cfg5_mla_expanded cfg5_mla > gpurun_out/s3c_fields.jsonl 2> gpurun_out/s3c_fields.err; echo "fields rc $?"
timeout 1200 python scripts/mla_trace.py --requests 2000 --layers 27 --expanded --out gpurun_out/s3c_trace_expanded.json > gpurun_out/s3c_trace_expanded.log 2>&1; echo "trace exp rc $?"
timeout 1200 python scripts/mla_trace.py --requests 2000 --layers 27 --out gpurun_out/s3c_trace_absorbed.json > gpurun_out/s3c_trace_absorbed.log 2>&1; echo "trace abs rc $?"
tail -1 gpurun_out/s3c_trace_expanded.log | cut -c1-600
tail -1 gpurun_out/s3c_trace_absorbed.log | cut -c1-600
