cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { timeout 300 python scripts/microbench.py --kernel decode --bs 64 --batch 64 --ctx 2048 --budgets 74,89,104,148 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print('$1', d['budget'], round(d['ms'],4), round(d.get('GB_s',0)))"; }
unset SEMIPD_LIB; unset SEMIPD_DECODE_PAIR64; run default
export SEMIPD_DECODE_PAIR64=1; run pair
for v in sk1024 sk2048; do export SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$v.so; unset SEMIPD_DECODE_PAIR64; run $v; export SEMIPD_DECODE_PAIR64=1; run ${v}_pair; done
