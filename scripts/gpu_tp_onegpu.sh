#!/bin/bash
# The driver's N > 1 bench command shape (default flags: e2e + extra on), every rank on the
# box's one GPU (dev overrides; gloo since NCCL refuses two ranks per device).  Plumbing check.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for n in 2 8; do
  SPD_BENCH_ONE_GPU=1 SPD_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --steps 3 --warmup 3 > gpurun_out/bench_tp${n}_onegpu.json 2> gpurun_out/bench_tp${n}_onegpu.err
  echo "tp$n exit $?" >> gpurun_out/summary_tp.txt
done
cat gpurun_out/summary_tp.txt
