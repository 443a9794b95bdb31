cd /root/repo
timeout 600 python -m pytest tests/test_gpu_rope.py -q -p no:cacheprovider > gpurun_out/rope.log 2>&1; tail -3 gpurun_out/rope.log
SPD_BENCH_ONE_GPU=1 SPD_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --steps 3 --warmup 3 --no-extra --sweep 40 > gpurun_out/bench_tp2_onegpu.json 2> gpurun_out/bench_tp2_onegpu.err; echo "tp2 exit $?"
