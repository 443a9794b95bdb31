#!/usr/bin/env python
"""Dev probe: per-launch device timeline (span records [5] / [6]: first CTA entry after the PDL
wait, last CTA exit) of one replay of the cfg2 co-run step at split x, both streams: launch
durations and the gaps between consecutive launches of each stream."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses
import numpy as np
import torch
import bench


def main():
    x = float(sys.argv[1]) if len(sys.argv) > 1 else 30.0
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    shape = dataclasses.replace(bench.MODELS["llama3-8b"], block_size=64)
    w = bench.Workload(shape, 1, dev)
    run = bench.Runner(w, dev)
    for _ in range(2):
        w.corun_step(50, 50)
    step = run.capture(lambda: w.corun_step(x, 100 - x, 0, 0))
    for _ in range(4):
        step()
    torch.cuda.synchronize()
    sp = w.spans.cpu().numpy().astype(np.float64)
    L = w.L
    t0 = min(sp[:2 * L, 5])
    for ph, off in (("prefill", 0), ("decode", L)):
        if w.span_order[0] != "prefill":
            off = L - off
        r = sp[off:off + L]
        st, en = (r[:, 5] - t0) / 1e3, (r[:, 6] - t0) / 1e3
        dur = en - st
        gap = st[1:] - en[:-1]
        print(f"{ph}: first start {st[0]:.1f} us, last end {en[-1]:.1f} us, mean launch {dur.mean():.1f} us, "
              f"gaps mean {gap.mean():.2f} min {gap.min():.2f} max {gap.max():.2f} us, sum {gap.sum():.1f} us")
        print("  starts", " ".join(f"{v:.0f}" for v in st[:8]), "...")
        print("  durs  ", " ".join(f"{v:.1f}" for v in dur[:8]), "...")
        print("  gaps  ", " ".join(f"{v:.1f}" for v in gap[:12]), "...")


if __name__ == "__main__":
    main()
