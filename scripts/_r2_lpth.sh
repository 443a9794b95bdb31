cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
timeout 300 python scripts/microbench.py --mla --ctx-lognormal --budgets 44,104,148 --batch 256 --ctx 350 --layers 8 2>&1 | tail -3
timeout 300 python scripts/microbench.py --mla --ctx-lognormal --lpt --budgets 44,104,148 --batch 256 --ctx 350 --layers 8 2>&1 | tail -3
done
