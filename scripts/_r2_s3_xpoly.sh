cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for v in default xp0 xp55; do
  if [ $v = default ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; fi
  echo "== $v"
  for P in 0 4096; do
  timeout 300 python scripts/microbench.py --mla-exp --budgets 59,104,148 --layers 4 --prefix $P 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print(d['budget'], d['P'], 'attn', round(d['attn_ms'],4))"
  done
done
done
