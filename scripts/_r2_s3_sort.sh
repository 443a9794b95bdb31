cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py tests/test_gpu_mla_expanded.py tests/test_gpu_trace.py -q -x -k "mla or trace" > gpurun_out/s3so_def.log 2>&1; echo "pytest default rc $?"; tail -2 gpurun_out/s3so_def.log
SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_s10.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -q -x -k "mla" > gpurun_out/s3so_test.log 2>&1; echo "pytest s10 rc $?"; tail -2 gpurun_out/s3so_test.log
for v in default nosort s10 s14; do
  if [ $v = default ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; fi
  echo "== $v"
  timeout 300 python scripts/microbench.py --mla --ctx 350 --ctx-lognormal --lpt --batch 256 --budgets 44,74,104,148 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print('lognormal', d['budget'], round(d['ms'],4), round(d['GB_s']))"
  timeout 300 python scripts/microbench.py --mla --ctx 1000 --batch 256 --budgets 74,104,148 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print('ctx1000', d['budget'], round(d['ms'],4), round(d['GB_s']))"
  timeout 300 python scripts/microbench.py --mla --ctx 4000 --batch 64 --budgets 104,148 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print('B64ctx4000', d['budget'], round(d['ms'],4), round(d['GB_s']))"
done
