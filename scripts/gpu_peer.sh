#!/bin/bash
# peer (copy-engine) all-gather: GPU tests (two processes on the box's one GPU) and the
# N = 2 bench path on one GPU (dev overrides: both ranks on cuda:0, gloo for the host plumbing)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python scripts/probe_memops.py > gpurun_out/probe_memops.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_peer_gather.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/test_peer.log 2>&1; echo "peer tests exit $?" >> gpurun_out/summary_peer.txt
tail -5 gpurun_out/test_peer.log
SPD_BENCH_ONE_GPU=1 SPD_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --gather peer --steps 3 --warmup 3 --sweep 40 --no-e2e --no-extra > gpurun_out/bench_tp2_peer_onegpu.json 2> gpurun_out/bench_tp2_peer_onegpu.err; echo "bench peer exit $?" >> gpurun_out/summary_peer.txt
tail -3 gpurun_out/bench_tp2_peer_onegpu.err
cat gpurun_out/summary_peer.txt
