cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_ -s 2 -c 1 -o gpurun_out/prof_dec16 python scripts/microbench.py --kernel decode --budgets 104 --iters 3 --bs 16 > gpurun_out/ncu_dec16.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_ -s 2 -c 1 -o gpurun_out/prof_dec64 python scripts/microbench.py --kernel decode --budgets 104 --iters 3 --bs 64 > gpurun_out/ncu_dec64.log 2>&1
for f in prof_dec16 prof_dec64; do python scripts/ncu_summary.py gpurun_out/$f.ncu-rep 12 > gpurun_out/${f}_summary.txt 2>&1; done
ncu -i gpurun_out/prof_dec16.ncu-rep --page raw --csv > gpurun_out/dec16_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_dec64.ncu-rep --page raw --csv > gpurun_out/dec64_raw.csv 2>/dev/null
