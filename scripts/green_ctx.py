#!/usr/bin/env python
"""N3: hard SM isolation with CUDA green contexts vs. this repo's grid capping.

For splits x in --splits, the 148 SMs are partitioned with cuDevSmResourceSplitByCount into a
prefill green context and a decode green context; the cfg-2 co-run step (32 layers of one
2048-token chunk + a 64-request decode step, bs 64) then runs with each phase on a stream of
its own green context, either as persistent grids sized to the partition or as non-persistent
grids (one CTA per work unit, confined by the hardware).  The same step with grid capping on
ordinary streams (the repo's mechanism, P:195 realised as sm_budget) is timed alongside.
Eager launches and host wall-clock timing over --steps steps for all three (same overheads).

  python scripts/green_ctx.py --splits 30,40,50 --steps 20 --out profiles/r1_green_ctx.json
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (workload builder; no oracle involved)
from cuda.bindings import driver as cu  # noqa: E402


def check(res):
    err = res[0] if isinstance(res, tuple) else res
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"driver call failed: {err}")
    return res[1:] if isinstance(res, tuple) and len(res) > 2 else (res[1] if isinstance(res, tuple) else None)


def green_streams(n_p: int):
    (dev,) = [check(cu.cuDeviceGet(0))]
    sm = check(cu.cuDeviceGetDevResource(dev, cu.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
    groups, nb, rem = check(cu.cuDevSmResourceSplitByCount(1, sm, 0, n_p))
    out = []
    for r in (groups[0], rem):
        desc = check(cu.cuDevResourceGenerateDesc([r], 1))
        g = check(cu.cuGreenCtxCreate(desc, dev, cu.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
        st = check(cu.cuGreenCtxStreamCreate(g, cu.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
        out.append((g, st, r.sm.smCount))
    return out


def timed(fn, streams, steps):
    for _ in range(3):
        fn()
    for s in streams:
        s.synchronize()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    for s in streams:
        s.synchronize()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--splits", default="30,40,50")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    import dataclasses
    shape = dataclasses.replace(bench.MODELS["llama3-8b"], block_size=64)
    w = bench.Workload(shape, 1, dev)
    rows = []
    for x in [float(v) for v in args.splits.split(",")]:
        n_req = int(148 * x / 100 + 0.5)
        (gp, sp_h, n_p), (gd, sd_h, n_d) = green_streams(n_req)
        sP = torch.cuda.ExternalStream(int(sp_h))
        sD = torch.cuda.ExternalStream(int(sd_h))

        def step_green(persistent: bool):
            w.phase_prefill(n_p if persistent else -1, stream=sP)
            w.phase_decode(n_d if persistent else -1, stream=sD)

        t_gp = timed(lambda: step_green(True), (sP, sD), args.steps)
        t_gn = timed(lambda: step_green(False), (sP, sD), args.steps)
        # grid capping on ordinary streams at the same SM counts
        w.pool.set_partition(100.0 * n_p / 148, 100.0 * n_d / 148)
        t_cap = timed(lambda: w.corun_step(100.0 * n_p / 148, 100.0 * n_d / 148), (w.sP, w.sD), args.steps)
        rec = {"x_requested": x, "n_prefill_sms": n_p, "n_decode_sms": n_d,
               "green_persistent_ms": t_gp, "green_nonpersistent_ms": t_gn, "grid_cap_ms": t_cap}
        print(json.dumps(rec), flush=True)
        rows.append(rec)
        for g in (gp, gd):
            cu.cuGreenCtxDestroy(g)
    if args.out:
        json.dump({"what": "cfg2 co-run step (ms, eager launches, host wall clock) with green-context SM "
                           "partitions vs grid capping", "rows": rows}, open(args.out, "w"), indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
