cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_ks2.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -q -x -k "decode or corun or stress or bitwise" > gpurun_out/s3k2_test.log 2>&1; echo "pytest ks2 rc $?"; tail -2 gpurun_out/s3k2_test.log
for rep in 1 2; do
for v in base ks2; do
  if [ $v = base ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; fi
  echo "== $v"
  timeout 300 python scripts/microbench.py --kernel decode --budgets 44,74,89,104,148 --bs 64 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['budget'], round(d['ms'],4), round(d['GB_s']))"
done
done
