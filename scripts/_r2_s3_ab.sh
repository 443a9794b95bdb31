cd /root/repo
for v in default nosplit nosplit32 split32; do
  if [ $v = default ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; fi
  echo "== $v"
  timeout 300 python scripts/microbench.py --mla-exp --budgets 44,104,148 --layers 4 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['budget'], d['P'], 'graph', round(d['ms_graph'],4), 'gemm', round(d['gemm_ms'],4), 'attn', round(d['attn_ms'],4))"
  timeout 300 python scripts/microbench.py --mla-exp --budgets 148 --layers 4 --prefix 4096 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['budget'], d['P'], 'graph', round(d['ms_graph'],4), 'gemm', round(d['gemm_ms'],4), 'attn', round(d['attn_ms'],4))"
done
