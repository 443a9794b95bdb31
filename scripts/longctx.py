#!/usr/bin/env python
"""cfg4 long-context mix (BASELINE.json configs[3]): 16 decode requests at ctx 32768 co-run
with 8192-token prefill chunks of a 32k prompt (P = 0, 8192, 16384, 24576), while the
partition cycles (30,70) -> (50,50) -> (70,30) every 8 iterations (P:211-216 delayed /
asynchronous switching: each phase adopts the new budget at its next launch).

Reports per-iteration device time, the partition-switch cost (first iteration after a
switch vs the steady state at the new split), decode GB/s and prefill TFLOP/s, and checks
that switching moves no KV (pool pointer + a checksum of every page untouched by the
iteration stay unchanged).  Llama-3-8B attention shapes, bs 64, --layers per iteration.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--iters", type=int, default=24)
    ap.add_argument("--bs", type=int, default=64)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "longctx.json"))
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    L, B, ctx, C, prompt = a.layers, 16, 32768, 8192, 32768
    Hq, Hkv, d, bs = 32, 8, 128, a.bs
    nb_dec, nb_pre = ctx // bs + 1, prompt // bs
    cfg = PoolConfig(L, B * nb_dec + nb_pre + 8, bs, Hkv, d, d, B + 2, max(nb_dec, nb_pre) + 2)
    pool = KVPool(cfg, dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32(list(range(B))), i32([nb_dec] * B))
    pool.alloc_blocks(i32([B]), i32([nb_pre]))
    g = torch.Generator(device=dev)
    g.manual_seed(4)
    for l in range(L):
        K, V, _, _ = pool.views(l)
        K.normal_(generator=g)
        V.normal_(generator=g)
    rnd = lambda *s: torch.randn(*s, device=dev, generator=g).bfloat16()  # noqa: E731
    qd = [rnd(B, Hq, d) for _ in range(L)]
    kd = [rnd(B, Hkv, d) for _ in range(L)]
    vd = [rnd(B, Hkv, d) for _ in range(L)]
    qp = [rnd(C, Hq, d) for _ in range(L)]
    kp = [rnd(C, Hkv, d) for _ in range(L)]
    vp = [rnd(C, Hkv, d) for _ in range(L)]
    od = torch.empty(B, Hq, d, dtype=torch.bfloat16, device=dev)
    op = torch.empty(C, Hq, d, dtype=torch.bfloat16, device=dev)
    ws = pool.new_decode_workspace(B, Hq, ctx)
    rid, ctxs = i32(list(range(B))), i32([ctx] * B)
    cu, ridp = i32([0, C]), i32([B])
    sc = 1 / math.sqrt(d)
    sP, sD = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    schedule = [(30, 70), (50, 50), (70, 30)]
    ptr0 = pool.mem.data_ptr()
    # checksum of the decode requests' cached pages (never written by an iteration: the
    # decode append rewrites slot ctx with the same bits, prefill writes only its blocks)
    K0, V0, BT, _ = pool.views(0)
    dec_blocks = BT[:B, :nb_dec - 1].reshape(-1).long()
    chk0 = int(K0[dec_blocks].view(torch.int16).sum().item())

    def iteration(it):
        x, y = schedule[(it // 8) % len(schedule)]
        pool.set_partition(x, y)
        P = (it % 4) * C
        pre = i32([P])
        main = torch.cuda.current_stream(dev)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        e[0].record(main)
        sP.wait_stream(main)
        sD.wait_stream(main)
        with torch.cuda.stream(sP):
            e[1].record(sP)
            for l in range(L):
                pool.prefill_attn(l, qp[l], kp[l], vp[l], cu, ridp, pre, C, C, sc, op, stream=sP)
            e[2].record(sP)
        with torch.cuda.stream(sD):
            e[3].record(sD)
            for l in range(L):
                pool.decode_attn(l, qd[l], kd[l], vd[l], rid, ctxs, ctx, sc, od, ws, stream=sD)
            e[4].record(sD)
        main.wait_stream(sP)
        main.wait_stream(sD)
        e[5].record(main)
        torch.cuda.synchronize(dev)
        pairs = C * P + C * (C + 1) / 2
        pre_ms, dec_ms = e[1].elapsed_time(e[2]), e[3].elapsed_time(e[4])
        return {"it": it, "x": x, "y": y, "budgets": pool.sm_budgets(), "P": P,
                "ms": e[0].elapsed_time(e[5]), "prefill_ms": pre_ms, "decode_ms": dec_ms,
                "prefill_tflops": L * 2 * Hq * 2 * d * pairs / (pre_ms / 1e3) / 1e12,
                "decode_gbs": L * B * (ctx + 1) * Hkv * 2 * d * 2 / (dec_ms / 1e3) / 1e9}

    for it in range(4):   # warm-up
        iteration(it)
    recs = [iteration(it) for it in range(a.iters)]
    chk1 = int(K0[dec_blocks].view(torch.int16).sum().item())
    # switch cost: first iteration of each 8-iteration block vs the median of the same P at
    # the same split inside the block
    sw = []
    for r in recs:
        if r["it"] % 8 == 0 and r["it"] > 0:
            same = [q["ms"] for q in recs if q["x"] == r["x"] and q["P"] == r["P"] and q["it"] != r["it"]]
            if same:
                sw.append(r["ms"] - statistics.median(same))
    out = {"config": "cfg4 long-context mix (Llama-3-8B attention, bs %d, %d layers/iter)" % (bs, L),
           "iterations": recs, "switch_cost_ms": sw,
           "kv_moved": pool.mem.data_ptr() != ptr0 or chk0 != chk1,
           "pool_checksum_before": chk0, "pool_checksum_after": chk1}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    for r in recs:
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}))
    print("switch cost ms:", [round(s, 3) for s in sw], "kv_moved:", out["kv_moved"])


if __name__ == "__main__":
    main()
