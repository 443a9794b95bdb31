cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
echo "== single (default at B=64)"; timeout 300 python scripts/microbench.py --kernel decode --bs 64 --budgets 59,74,89,104,148 --layers 8 2>&1 | tail -5
echo "== pair64 forced"; SEMIPD_DECODE_PAIR64=1 timeout 300 python scripts/microbench.py --kernel decode --bs 64 --budgets 59,74,89,104,148 --layers 8 2>&1 | tail -5
done
