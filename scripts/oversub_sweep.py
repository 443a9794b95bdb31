"""Co-run step time at (x, y) partitions with x + y > 100 (P:216 / P:522: the two workers may
"compete for the resources"): persistent grids of n_p + n_d > 148 CTAs, where the CTAs that do
not fit start as the other phase's CTAs exit.  cfg-2 workload of bench.py, graph replay."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
import dataclasses  # noqa: E402
w = bench.Workload(dataclasses.replace(bench.MODELS["llama3-8b"], block_size=64), 1, dev)
for _ in range(2):
    w.corun_step(50, 50)
pairs = [(40, 60), (40, 65), (40, 70), (40, 80), (35, 70), (45, 65), (50, 60), (30, 80), (60, 60),
         (100, 100), (40, 60)]
for x, y in pairs:
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        w.corun_step(x, y)
    g.replay()
    t = bench.time_steps(g.replay, 10, dev) / 10
    n_p, n_d = w.pool.sm_budgets()
    print(json.dumps({"x": x, "y": y, "n_p": n_p, "n_d": n_d, "ms": t * 1e3,
                      "tokens_per_s": (bench.PREFILL_TOKENS + bench.DECODE_BATCH) / t}), flush=True)
