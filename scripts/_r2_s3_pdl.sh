cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -q -x -k "corun or decode or prefill or bitwise or stress" > gpurun_out/s3p_test.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/s3p_test.log
for v in pdl nopdl pdl nopdl; do
  if [ $v = nopdl ]; then export SEMIPD_NO_PDL=1; else unset SEMIPD_NO_PDL; fi
  timeout 600 python bench.py --no-secondary --no-e2e --no-cpu --no-extra --sweep 30,35,40,45,50 > gpurun_out/s3p_bench_$v.json 2> gpurun_out/s3p_bench_$v.err
  python - <<PY
import json
d=json.loads(open('gpurun_out/s3p_bench_$v.json').read().strip().splitlines()[-1])
print('$v', round(d['value']), round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), d.get('corun_streams'))
for r in d['sweep']: print('  ', r['x'], round(r['tokens_per_s']), round(r['decode_frac'],3), round(r['prefill_frac_share_burst'],3), round(r['overlap'],3))
PY
done
