#!/usr/bin/env python
"""Isolated per-kernel timing (CUDA events) for the cfg2 shapes at chosen SM budgets.

  python scripts/microbench.py --kernel decode --budgets 37,74,148
  python scripts/microbench.py --kernel prefill --budgets 74 --iters 3   (under ncu)

Decode: B=64 requests, ctx 2048, Hq 32 / Hkv 8, d 128, bs 16; rotates over L layers
of distinct pool memory (L x 537 MB >> L2).  Prefill: one 2048-token chunk, P=0.
Prints one JSON line per (kernel, budget): median ms, GB/s (decode, algorithmic
bytes), TFLOP/s (prefill, unmasked pairs).
"""
import argparse
import json
import math
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2504_19867_b200 import KVPool, PoolConfig  # noqa: E402


def timed_ms(run, iters, L, reps=5):
    """Median over `reps` of the mean time per launch of `iters` back-to-back launches
    (rotating over L layers).  Launches are queued without a host sync between them, so the
    host's per-call work (ctypes marshalling, tensor-map encodes) overlaps the previous kernel
    instead of sitting between two events; a synchronised per-call loop over-counts short
    kernels by that host time (~15 us)."""
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for it in range(iters):
            run(it % L)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / iters)
    return statistics.median(out), min(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="decode", choices=["decode", "prefill", "both"])
    ap.add_argument("--budgets", default="74,148")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--chunk", type=int, default=2048)
    ap.add_argument("--prefix", type=int, default=0)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--bs", type=int, default=16)
    ap.add_argument("--ctx-uniform", default=None,
                    help="lo,hi: decode contexts ~ U[lo, hi] (seed 2002) instead of all = --ctx "
                         "(SURVEY §8(d) item 7, load balance)")
    ap.add_argument("--mla", action="store_true", help="cfg5 absorbed-MLA decode (576/512, 16 heads)")
    ap.add_argument("--mla-prefill", action="store_true", help="cfg5 absorbed-MLA prefill chunk")
    ap.add_argument("--mla-exp", action="store_true",
                    help="cfg5 expanded-form MLA prefill chunk (R32): prep + up-projection GEMM + attention")
    ap.add_argument("--lpt", action="store_true", help="--ctx-lognormal: batch longest first")
    ap.add_argument("--fp8", action="store_true",
                    help="E4M3 pool (reading R31; bs must be 64): decode reads 1-byte codes")
    ap.add_argument("--ctx-lognormal", action="store_true",
                    help="--mla: contexts lognormal around --ctx (sigma 0.5, seed 5005), as bench.py cfg5")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    if args.mla:
        return mla(args, dev)
    if args.mla_prefill:
        return mla_prefill(args, dev)
    if args.mla_exp:
        return mla_exp(args, dev)
    L, B, ctx, C, P = args.layers, args.batch, args.ctx, args.chunk, args.prefix
    Hq, Hkv, d, bs = args.hq, args.hkv, 128, args.bs
    if args.ctx_uniform:
        import numpy as np
        lo, hi = (int(v) for v in args.ctx_uniform.split(","))
        ctx_list = [int(v) for v in np.random.default_rng(2002).integers(lo, hi + 1, size=B)]
    else:
        ctx_list = [ctx] * B
    ctx = max(ctx_list)
    nb_dec = ctx // bs + 1
    nb_pre = -(-(C + P) // bs)
    cfg = PoolConfig(L, B * nb_dec + nb_pre + 8, bs, Hkv, d, d, B + 2, max(nb_dec, nb_pre) + 2,
                     dtype=torch.float8_e4m3fn if args.fp8 else torch.bfloat16)
    pool = KVPool(cfg, dev)
    if args.fp8:
        pool.set_kv_scales(0.05, 0.02)
        pool.attach_fp8_prefill_scratch(1)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32(list(range(B))), i32([c // bs + 1 for c in ctx_list]))
    pool.alloc_blocks(i32([B]), i32([nb_pre]))
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for l in range(L):
        K, V, _, _ = pool.views(l)
        if args.fp8:  # random finite E4M3 codes of magnitude < 2^7
            K.copy_(torch.randint(0, 0x70, K.shape, device=dev, generator=g, dtype=torch.int32).to(torch.uint8) |
                    (torch.randint(0, 2, K.shape, device=dev, generator=g, dtype=torch.int32) * 128).to(torch.uint8))
            V.copy_(torch.randint(0, 0x70, V.shape, device=dev, generator=g, dtype=torch.int32).to(torch.uint8))
        else:
            K.normal_(generator=g)
            V.normal_(generator=g)
    rnd = lambda *s: torch.randn(*s, device=dev, generator=g).bfloat16()  # noqa: E731
    sc = 1 / math.sqrt(d)
    qd, kd, vd = rnd(B, Hq, d), rnd(B, Hkv, d), rnd(B, Hkv, d)
    od = torch.empty(B, Hq, d, dtype=torch.bfloat16, device=dev)
    ws = pool.new_decode_workspace(B, Hq, ctx)
    rid, ctxs = i32(list(range(B))), i32(ctx_list)
    qp, kp, vp = rnd(C, Hq, d), rnd(C, Hkv, d), rnd(C, Hkv, d)
    op = torch.empty(C, Hq, d, dtype=torch.bfloat16, device=dev)
    cu, ridp, pre = i32([0, C]), i32([B]), i32([P])
    kv_elem = 1 if args.fp8 else 2
    dec_bytes = sum(c + 1 for c in ctx_list) * Hkv * 2 * d * kv_elem + B * Hq * 2 * d * 2
    pairs = C * P + C * (C + 1) / 2
    pre_flops = 2 * Hq * 2 * d * pairs
    kernels = ["decode", "prefill"] if args.kernel == "both" else [args.kernel]
    for kern in kernels:
        for bud in [int(x) for x in args.budgets.split(",")]:
            def run(l):
                if kern == "decode":
                    pool.decode_attn(l, qd, kd, vd, rid, ctxs, ctx, sc, od, ws, sm_budget=bud)
                else:
                    pool.prefill_attn(l, qp, kp, vp, cu, ridp, pre, C, C, sc, op, sm_budget=bud)
            for l in range(min(L, 3)):
                run(l)
            torch.cuda.synchronize()
            ms, ms_min = timed_ms(run, args.iters, L)
            rec = {"kernel": kern, "budget": bud, "ms": ms, "min_ms": ms_min}
            if kern == "decode":
                rec["GB_s"] = dec_bytes / (ms / 1e3) / 1e9
            else:
                rec["TFLOP_s"] = pre_flops / (ms / 1e3) / 1e12
            print(json.dumps(rec), flush=True)


def mla(args, dev):
    """MLA decode: B requests at ctx, latent 576 (V = first 512), 16 heads, bs 64."""
    L, B, ctx, bs = args.layers, args.batch, args.ctx, 64
    if args.ctx_lognormal:  # the bench's cfg-5 mix: lognormal around --ctx (sigma 0.5, seed 5005)
        import numpy as np
        rng = np.random.default_rng(5005)
        ctx_list = [int(c) for c in np.clip(rng.lognormal(math.log(ctx) - 0.125, 0.5, B), 64, 4096)]
        if args.lpt:
            ctx_list.sort(reverse=True)
    else:
        ctx_list = [ctx] * B
    ctx = max(ctx_list)
    nbs = [c // bs + 1 for c in ctx_list]
    nb = max(nbs)
    cfg = PoolConfig(L, sum(nbs) + 4, bs, 1, 576, 512, B + 1, nb + 1, kv_shared=True)
    pool = KVPool(cfg, dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32(list(range(B))), i32(nbs))
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for l in range(L):
        K, _, _, _ = pool.views(l)
        K.normal_(generator=g)
    q = torch.randn(B, 16, 576, device=dev, generator=g).bfloat16()
    kn = torch.randn(B, 1, 576, device=dev, generator=g).bfloat16()
    out = torch.empty(B, 16, 512, dtype=torch.bfloat16, device=dev)
    ws = pool.new_decode_workspace(B, 16, ctx)
    rid, ctxs = i32(list(range(B))), i32(ctx_list)
    byts = sum(c + 1 for c in ctx_list) * 576 * 2 + B * 16 * (576 + 512) * 2
    flops = 2 * sum(c + 1 for c in ctx_list) * 16 * (576 + 512)
    for bud in [int(x) for x in args.budgets.split(",")]:
        for l in range(min(L, 3)):
            pool.decode_attn(l, q, kn, None, rid, ctxs, ctx, 1 / math.sqrt(192), out, ws, sm_budget=bud)
        torch.cuda.synchronize()
        ms, _ = timed_ms(lambda l: pool.decode_attn(l, q, kn, None, rid, ctxs, ctx, 1 / math.sqrt(192),
                                                    out, ws, sm_budget=bud), args.iters, L)
        print(json.dumps({"kernel": "decode_mla", "budget": bud, "B": B, "ctx": ctx, "ms": ms,
                          "GB_s": byts / (ms / 1e3) / 1e9, "TFLOP_s": flops / (ms / 1e3) / 1e12}),
              flush=True)


def mla_prefill(args, dev):
    """MLA prefill: one chunk of C tokens after a prefix P, 16 heads over the latent (bs 64)."""
    L, C, P = args.layers, args.chunk, args.prefix
    nb = -(-(C + P) // 64)
    pool = KVPool(PoolConfig(L, nb + 4, 64, 1, 576, 512, 2, nb + 1, kv_shared=True), dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32([0]), i32([nb]))
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for l in range(L):
        K, _, _, _ = pool.views(l)
        K.normal_(generator=g)
    q = torch.randn(C, 16, 576, device=dev, generator=g).bfloat16()
    k = torch.randn(C, 1, 576, device=dev, generator=g).bfloat16()
    out = torch.empty(C, 16, 512, dtype=torch.bfloat16, device=dev)
    flops = 2 * 16 * (576 + 512) * (C * P + C * (C + 1) / 2)
    for bud in [int(x) for x in args.budgets.split(",")]:
        run = lambda l: pool.prefill_attn(l, q, k, None, i32([0, C]), i32([0]), i32([P]), C, C,  # noqa: E731
                                          1 / math.sqrt(192), out, sm_budget=bud)
        for l in range(min(L, 2)):
            run(l)
        torch.cuda.synchronize()
        ms, _ = timed_ms(run, args.iters, L)
        print(json.dumps({"kernel": "prefill_mla", "budget": bud, "C": C, "P": P, "ms": ms,
                          "TFLOP_s": flops / (ms / 1e3) / 1e12}), flush=True)


def mla_exp(args, dev):
    """Expanded-form MLA prefill (R32): one chunk of C tokens after a prefix P, 16 heads, bs 64.
    Reports the call's time, the GEMM / attention kernels' span-timed shares, TFLOP/s of each
    against its own algorithmic flops, and the absorbed-equivalent rate (the absorbed form's flops
    for the same tokens / this call's time) for comparison with --mla-prefill."""
    L, C, P, H = args.layers, args.chunk, args.prefix, 16
    nb = -(-(C + P) // 64)
    pool = KVPool(PoolConfig(L, nb + 4, 64, 1, 576, 512, 2, nb + 1, kv_shared=True), dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32([0]), i32([nb]))
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for l in range(L):
        K, _, _, _ = pool.views(l)
        K.normal_(generator=g)
    q = torch.randn(C, H, 192, device=dev, generator=g).bfloat16()
    kv = torch.randn(C, 576, device=dev, generator=g).bfloat16()
    w_uk = [(torch.randn(H, 128, 512, device=dev, generator=g) / 22.6).bfloat16() for _ in range(L)]
    w_uv = [(torch.randn(H, 128, 512, device=dev, generator=g) / 22.6).bfloat16() for _ in range(L)]
    out = torch.empty(C, H, 128, dtype=torch.bfloat16, device=dev)
    ws = pool.new_mla_expanded_workspace(1, C + P, H)
    pairs = C * P + C * (C + 1) / 2
    f_attn = 2 * H * (192 + 128) * pairs
    f_gemm = 2 * (C + P) * 512 * 2 * H * 128
    f_abs = 2 * H * (576 + 512) * pairs
    spans = torch.zeros(3, 8, dtype=torch.int64, device=dev)  # prep, GEMM, attention
    cu_t, rid_t, pre_t = i32([0, C]), i32([0]), i32([P])
    for bud in [int(x) for x in args.budgets.split(",")]:
        run = lambda l: pool.prefill_mla_expanded(l, q, kv, w_uk[l], w_uv[l], cu_t, rid_t,  # noqa: E731
                                                  pre_t, C, C, C + P, 1 / math.sqrt(192), out, ws,
                                                  sm_budget=bud)
        for l in range(min(L, 2)):
            run(l)
        torch.cuda.synchronize()
        ms, _ = timed_ms(run, args.iters, L)
        # the same calls captured into a CUDA graph (no host work between launches: the bench's
        # co-run step is graph-replayed too)
        gs = torch.cuda.Stream(device=dev)
        gs.wait_stream(torch.cuda.current_stream(dev))
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            for it in range(L):
                pool.prefill_mla_expanded(it, q, kv, w_uk[it], w_uv[it], cu_t, rid_t,
                                          pre_t, C, C, C + P, 1 / math.sqrt(192), out, ws,
                                          sm_budget=bud, stream=gs)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ms_graph = e0.elapsed_time(e1) / (5 * L)
        spans.zero_()
        pool.set_spans(spans)
        for it in range(args.iters):
            run(it % L)
        torch.cuda.synchronize()
        pool.set_spans(None)
        sp = spans.cpu()
        pms = float(sp[0, 2]) / max(1, int(sp[0, 3])) / 1e6
        gms = float(sp[1, 2]) / max(1, int(sp[1, 3])) / 1e6
        ams = float(sp[2, 2]) / max(1, int(sp[2, 3])) / 1e6
        print(json.dumps({"kernel": "prefill_mla_expanded", "budget": bud, "C": C, "P": P, "ms": ms,
                          "ms_graph": ms_graph, "TFLOP_s_graph": (f_gemm + f_attn) / (ms_graph / 1e3) / 1e12,
                          "prep_ms": pms, "gemm_ms": gms, "attn_ms": ams,
                          "gemm_TFLOP_s": f_gemm / (gms / 1e3) / 1e12 if gms > 0 else None,
                          "attn_TFLOP_s": f_attn / (ams / 1e3) / 1e12 if ams > 0 else None,
                          "TFLOP_s": (f_gemm + f_attn) / (ms / 1e3) / 1e12,
                          "absorbed_equiv_TFLOP_s": f_abs / (ms / 1e3) / 1e12}), flush=True)


if __name__ == "__main__":
    main()
