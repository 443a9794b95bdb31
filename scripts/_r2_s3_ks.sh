cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -q -x -k "decode or corun or stress or bitwise" > gpurun_out/s3k_test.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/s3k_test.log
for rep in 1 2; do
for v in ks noks; do
  if [ $v = ks ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; fi
  echo "== $v"
  timeout 300 python scripts/microbench.py --kernel decode --budgets 44,74,89,104,148 --bs 64 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['budget'], round(d['ms'],4), round(d['GB_s']))"
done
done
for v in ks noks; do
  if [ $v = ks ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; fi
  timeout 600 python bench.py --no-secondary --no-e2e --no-cpu --no-extra --sweep 35,40,45 > gpurun_out/s3k_bench_$v.json 2>/dev/null
  python - <<PY
import json
d=json.loads(open('gpurun_out/s3k_bench_$v.json').read().strip().splitlines()[-1])
print('$v bench', round(d['value']), round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))
for r in d['sweep']: print('  ', r['x'], round(r['tokens_per_s']), round(r['decode_frac'],3), round(r['prefill_frac_share_burst'],3))
PY
done
