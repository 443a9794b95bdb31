#!/bin/bash
# full GPU round: all -m gpu tests, smoke, bench (+ncu launch list), isolated curves
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/test_all.log 2>&1; echo "tests exit $?" >> gpurun_out/summary.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/summary.txt
timeout 900 python bench.py --extra > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/summary.txt
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?" >> gpurun_out/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_bf16|prefill_tc|kv_write|alloc_kernel|free_kernel" -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --sweep 40 > gpurun_out/ncu_bench.log 2>&1; echo "ncu exit $?" >> gpurun_out/summary.txt
timeout 300 python scripts/microbench.py --kernel both --budgets 16,37,59,74,89,111,148 --bs 64 > gpurun_out/micro.jsonl 2>&1
cat gpurun_out/summary.txt
