"""Co-run step at disjoint and oversubscribed partitions with the prefill stream at HIGH
priority (the block scheduler then hands freed SMs to pending prefill CTAs first), cfg 2,
graph replay.  Compares against default-priority streams in the same process."""
import dataclasses
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
w = bench.Workload(dataclasses.replace(bench.MODELS["llama3-8b"], block_size=64), 1, dev)
lo, hi = torch.cuda.Stream.priority_range()  # (0 = low ... hi = most negative = highest)
streams = {"default": (w.sP, w.sD),
           "prefill_high": (torch.cuda.Stream(dev, priority=-1), torch.cuda.Stream(dev, priority=0)),
           "decode_high": (torch.cuda.Stream(dev, priority=0), torch.cuda.Stream(dev, priority=-1))}
for _ in range(2):
    w.corun_step(50, 50)
for name, (sp, sd) in streams.items():
    w.sP, w.sD = sp, sd
    for x, y in [(40, 60), (40, 70), (40, 80), (40, 100), (50, 100), (30, 100), (100, 100)]:
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            w.corun_step(x, y)
        g.replay()
        t = min(bench.time_steps(g.replay, 10, dev) / 10 for _ in range(2))
        n_p, n_d = w.pool.sm_budgets()
        print(json.dumps({"streams": name, "x": x, "y": y, "n_p": n_p, "n_d": n_d, "ms": t * 1e3,
                          "tokens_per_s": (bench.PREFILL_TOKENS + bench.DECODE_BATCH) / t}), flush=True)
