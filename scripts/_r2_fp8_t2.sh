#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fp8_build.log 2>&1 || { tail -30 gpurun_out/fp8_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fp8.py -q -x -m gpu -k "prefill or host" > gpurun_out/fp8_t2.log 2>&1
echo "fp8 prefill tests rc $?"; tail -3 gpurun_out/fp8_t2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "prefill" > gpurun_out/fp8_t2_bf16.log 2>&1
echo "bf16 prefill tests rc $?"; tail -3 gpurun_out/fp8_t2_bf16.log
for b in 44 89 104 148; do
  timeout 300 python scripts/microbench.py --kernel decode --bs 64 --budgets $b --iters 20 --layers 8 --fp8
  timeout 300 python scripts/microbench.py --kernel decode --bs 64 --budgets $b --iters 20 --layers 8
done 2>&1 | grep '^{' > gpurun_out/fp8_micro.jsonl
cat gpurun_out/fp8_micro.jsonl
timeout 300 python scripts/microbench.py --kernel prefill --bs 64 --budgets 59,148 --iters 10 --layers 4 --fp8 --prefix 4096 | grep '^{'
timeout 300 python scripts/microbench.py --kernel prefill --bs 64 --budgets 59,148 --iters 10 --layers 4 --prefix 4096 | grep '^{'
