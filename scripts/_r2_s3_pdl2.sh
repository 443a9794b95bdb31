cd /root/repo
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3q_smoke.log 2>&1; echo "smoke rc $?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s3q_gputest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/s3q_gputest.log
timeout 1500 python scripts/bench_field.py cfg5_mla_expanded cfg5_mla > gpurun_out/s3q_fields.jsonl 2> gpurun_out/s3q_fields.err; echo "fields rc $?"
python - <<'PY'
import json
for line in open('gpurun_out/s3q_fields.jsonl'):
    d=json.loads(line)
    print(d['field'], 'best', d['best']['x'], round(d['best']['tokens_per_s']), 'target', d['best_target']['x'], round(d['best_target']['target_score'],3))
PY
