cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export SPD_BENCH_ONE_GPU=1 SPD_BENCH_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --split 40 --no-cpu --no-secondary > gpurun_out/r2_tp2_gloo.json 2> gpurun_out/r2_tp2_gloo.err; echo "tp2 dependent rc $?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --split 40 --no-cpu --no-secondary --no-e2e --tp-mode pipelined > gpurun_out/r2_tp2_gloo_pipe.json 2> gpurun_out/r2_tp2_gloo_pipe.err; echo "tp2 pipelined rc $?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --steps 3 --warmup 3 --split 40 --no-cpu --no-secondary --no-e2e --gather fused > gpurun_out/r2_tp2_fused.json 2> gpurun_out/r2_tp2_fused.err; echo "tp2 fused rc $?"
tail -c 600 gpurun_out/r2_tp2_gloo.json; tail -3 gpurun_out/r2_tp2_gloo.err
