cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for v in default p0 p55 p33 p77; do
  if [ $v = default ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; fi
  echo "== $v"
  timeout 300 python scripts/microbench.py --kernel prefill --budgets 44,59,148 --bs 64 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['budget'], round(d['ms'],4), round(d['TFLOP_s']))"
done
done
