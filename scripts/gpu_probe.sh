set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_mufu scripts/probe_mufu.cu && /tmp/probe_mufu > gpurun_out/mufu.jsonl
timeout 300 python scripts/timeline.py 59 > gpurun_out/tl.log 2>&1
TL_OUT=timeline148.json timeout 300 python scripts/timeline.py 148 >> gpurun_out/tl.log 2>&1
cat gpurun_out/mufu.jsonl
