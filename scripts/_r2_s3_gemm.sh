cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3g_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_mla_expanded.py -q -x > gpurun_out/s3g_test.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/s3g_test.log
timeout 300 python scripts/microbench.py --mla-exp --budgets 44,74,104,148 --layers 4 > gpurun_out/s3g_micro.jsonl 2>&1
timeout 300 python scripts/microbench.py --mla-exp --budgets 44,74,148 --layers 4 --prefix 4096 >> gpurun_out/s3g_micro.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/s3g_micro.jsonl'):
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['budget'], d['P'], 'graph', round(d['ms_graph'],4), 'prep', round(d['prep_ms'],4), 'gemm', round(d['gemm_ms'],4), round(d['gemm_TFLOP_s']), 'attn', round(d['attn_ms'],4))
PY
