cd /root/repo
timeout 900 python -m pytest tests/test_gpu_mla_expanded.py -q -x > gpurun_out/s3ab2_test.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/s3ab2_test.log
for v in default nosplit; do
  if [ $v = default ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; fi
  echo "== $v"
  for P in 0 4096; do
  timeout 300 python scripts/microbench.py --mla-exp --budgets 44,74,104,148 --layers 4 --prefix $P 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['budget'], d['P'], 'graph', round(d['ms_graph'],4), 'gemm', round(d['gemm_ms'],4), 'attn', round(d['attn_ms'],4))"
  done
done
