cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in gemm attn prep; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_exp_$k -c 1 -o gpurun_out/s3f_ncu_$k python scripts/microbench.py --mla-exp --budgets 104 --layers 1 --iters 1 > gpurun_out/s3f_ncu_$k.log 2>&1; echo "ncu $k rc $?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_exp_attn -c 1 -o gpurun_out/s3f_ncu_attn_p4096 python scripts/microbench.py --mla-exp --budgets 148 --layers 1 --iters 1 --prefix 4096 > gpurun_out/s3f_ncu_attn4096.log 2>&1; echo "ncu attn4096 rc $?"
