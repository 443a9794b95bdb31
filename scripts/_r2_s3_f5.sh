cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3f_build.log 2>&1
timeout 300 python scripts/microbench.py --mla-exp --budgets 44,74,148 --layers 4 > gpurun_out/s3f_micro.jsonl 2>&1; echo "micro rc $?"
cat gpurun_out/s3f_micro.jsonl
timeout 900 python scripts/bench_field.py cfg5_mla_expanded cfg5_mla > gpurun_out/s3f_fields.jsonl 2> gpurun_out/s3f_fields.err; echo "fields rc $?"
tail -3 gpurun_out/s3f_fields.err
