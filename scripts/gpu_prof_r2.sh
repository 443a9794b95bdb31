#!/bin/bash
# Round-2 profiles: the bench step's launch list (cold, serialised) + ncu --set full captures
# of the cfg2 kernels at the bench split and of the cfg5 MLA kernels.  Writes gpurun_out/.
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --split 40 \
  --no-secondary --no-cpu --no-e2e --no-extra > gpurun_out/r2_launches_bench.log 2>&1
echo "launches rc $?"
bash scripts/gpu_prof.sh 59 89; echo "cfg2 full rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_mla -s 2 -c 1 \
  -o gpurun_out/prof_mla_prefill python scripts/microbench.py --mla-prefill --budgets 104 --iters 3 \
  --layers 2 > gpurun_out/ncu_mla_pre.log 2>&1; echo "mla prefill rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mla -s 2 -c 1 \
  -o gpurun_out/prof_mla_dec python scripts/microbench.py --mla --budgets 104 --batch 256 --ctx 350 \
  --iters 3 --layers 2 > gpurun_out/ncu_mla_dec.log 2>&1; echo "mla decode rc $?"
for f in prof_decode prof_prefill prof_mla_prefill prof_mla_dec; do
  python scripts/ncu_summary.py gpurun_out/$f.ncu-rep 20 > gpurun_out/${f}_summary.txt 2>&1
done
ls -la gpurun_out
