#!/usr/bin/env python
"""Dev probe: kernel-to-kernel gaps on one stream.  32 cfg-2 decode launches (one per layer) at
a given budget captured in a CUDA graph; graph time per launch vs the launches' own spans."""
import os, sys, json
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = bench.Workload(synth.CFG2_LLAMA8B, 1, dev, seed=1020)
    for budget in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "89,148").split(",")]:
        for phase in ("decode", "prefill"):
            w.span_order = (phase,)
            run = bench.Runner(w, dev)
            fn = (lambda: w.phase_decode(budget, stream=torch.cuda.current_stream(dev))) if phase == "decode" \
                else (lambda: w.phase_prefill(budget, stream=torch.cuda.current_stream(dev)))
            step = run.capture(fn)
            t, ks = run.time(step, 5)
            k = ks[phase]
            print(json.dumps({"phase": phase, "budget": budget, "graph_ms": t * 1e3, "kernel_ms_per_launch": k["ms"],
                              "launches": w.L, "sum_kernels_ms": k["ms"] * w.L,
                              "gap_us_per_launch": (t * 1e3 - k["ms"] * w.L) / w.L * 1e3,
                              "stream_ms": k["stream_ms"]}), flush=True)


if __name__ == "__main__":
    main()
