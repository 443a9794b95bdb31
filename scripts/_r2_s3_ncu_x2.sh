cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_exp_attn -c 1 -o gpurun_out/s3x2_ncu_attn_p4096 python scripts/microbench.py --mla-exp --budgets 148 --layers 1 --iters 1 --prefix 4096 > /dev/null 2>&1; echo "ncu rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_exp_attn -c 1 -o gpurun_out/s3x2_ncu_attn_p0 python scripts/microbench.py --mla-exp --budgets 74 --layers 1 --iters 1 > /dev/null 2>&1; echo "ncu rc $?"
