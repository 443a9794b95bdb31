cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mla_tc -c 1 -o gpurun_out/s3_ncu_mlad python scripts/microbench.py --mla --ctx 350 --ctx-lognormal --lpt --batch 256 --budgets 104 --iters 1 --layers 1 > gpurun_out/s3_ncu_mlad.log 2>&1; echo "ncu rc $?"
