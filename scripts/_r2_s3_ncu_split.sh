cd /root/repo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_exp_attn -c 1 -o gpurun_out/s3_ncu_split python scripts/microbench.py --mla-exp --budgets 44 --layers 1 --iters 1 > gpurun_out/s3_ncu_split.log 2>&1; echo "ncu rc $?"
