cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_mla_expanded.py -q -x > gpurun_out/s3sg_test.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/s3sg_test.log
for v in single nosingle; do
  if [ $v = single ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; fi
  echo "== $v"
  for P in 0 4096; do
  timeout 300 python scripts/microbench.py --mla-exp --budgets 74,89,104,118,148 --layers 4 --prefix $P 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['budget'], d['P'], 'graph', round(d['ms_graph'],4), 'attn', round(d['attn_ms'],4))"
  done
done
