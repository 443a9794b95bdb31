cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_bf16 -c 1 -o gpurun_out/s3_ncu_dec89 python scripts/microbench.py --kernel decode --budgets 89 --bs 64 --iters 1 --layers 2 > gpurun_out/s3_ncu_dec.log 2>&1; echo "ncu rc $?"
