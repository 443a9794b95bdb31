#!/bin/bash
# Final round-2 ncu captures: launch list of a bench step + ncu --set full of every hot kernel
# in its final form (cfg2 decode / prefill at the bench split, 16-token head-pair decode,
# MLA prefill with the 2-page ring, MLA decode on the lognormal longest-first batch).
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|prefill|alloc|free" -c 300 --csv \
  --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 3 --split 40 \
  --no-secondary --no-cpu --no-e2e --no-extra > gpurun_out/r2f_launches_bench.log 2>&1
echo "launches rc $?"
bash scripts/gpu_prof.sh 59 89; echo "cfg2 full rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_pair -s 2 -c 1 \
  -o gpurun_out/prof_dec16pair python scripts/microbench.py --kernel decode --bs 16 --budgets 89 --iters 3 --layers 2 > gpurun_out/ncu_dec16pair.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_mla -s 2 -c 1 \
  -o gpurun_out/prof_mla_prefill python scripts/microbench.py --mla-prefill --budgets 104 --iters 3 --layers 2 > gpurun_out/ncu_mla_pre.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mla -s 2 -c 1 \
  -o gpurun_out/prof_mla_dec python scripts/microbench.py --mla --ctx-lognormal --lpt --budgets 104 --batch 256 --ctx 350 \
  --iters 3 --layers 2 > gpurun_out/ncu_mla_dec.log 2>&1
for f in prof_decode prof_prefill prof_dec16pair prof_mla_prefill prof_mla_dec; do
  python scripts/ncu_summary.py gpurun_out/$f.ncu-rep 12 > gpurun_out/${f}_summary.txt 2>&1
done
ls gpurun_out/*summary.txt
