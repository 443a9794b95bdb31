#!/bin/bash
# smoke + co-run test + bench + ncu launch list; logs to gpurun_out/
cd "$(dirname "$0")/.."
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/summary.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k corun -s --timeout 150 > gpurun_out/test_corun.log 2>&1; echo "corun exit $?" >> gpurun_out/summary.txt
timeout 900 python bench.py --steps 10 --warmup 3 --extra > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/summary.txt
if [ "$1" == "ncu" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_bf16|prefill_tc|kv_write|alloc_kernel|free_kernel" -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --sweep 50 > gpurun_out/ncu_bench.log 2>&1; echo "ncu exit $?" >> gpurun_out/summary.txt
fi
cat gpurun_out/summary.txt
