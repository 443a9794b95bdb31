cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in default bm20 bm12 bm10 bm8; do
  if [ $v = default ]; then unset SEMIPD_LIB; else export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; fi
  echo "== $v"
  timeout 300 python scripts/microbench.py --mla --ctx 350 --ctx-lognormal --lpt --batch 256 --budgets 44,74,104,148 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l.strip()); continue
    print('lognormal', d['budget'], round(d['ms'],4), round(d['GB_s']))"
  timeout 300 python scripts/microbench.py --mla --ctx 1000 --batch 256 --budgets 74,148 2>&1 | python -c "
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
