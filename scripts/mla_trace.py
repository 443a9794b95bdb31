#!/usr/bin/env python
"""cfg-5 synthetic trace: DeepSeek-V2-Lite absorbed-MLA attention (27 layers,
16 heads, latent 576 / 512, 64-token pages, 3072-block pool) driven by the co-run engine
(paper_2504_19867_b200.engine) over a Poisson(3.0)-per-iteration trace of 2000 requests
(lognormal input mean 251, output mean 200, seed 5).

Measures attention time per iteration, allocator op count and pool high-water; parity is
sampled at --samples iterations against the fp64 oracle (layer 0: every 64th prefill row +
16 decode requests), and the whole device op log is replayed bit-exactly at the end.

  python scripts/mla_trace.py --requests 2000 --layers 27 --out profiles/r1_mla_trace.json
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402  (test infrastructure: parity sampling only)
import synth  # noqa: E402
from paper_2504_19867_b200 import KVPool, PoolConfig  # noqa: E402
from paper_2504_19867_b200.engine import CoRunEngine  # noqa: E402

TOL = (2e-2, 1e-2)


def bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def check(got: np.ndarray, ref: np.ndarray, what: str):
    diff = np.abs(got - ref)
    max_abs = float(diff.max()) if diff.size else 0.0
    den = float(np.linalg.norm(ref))
    fro = float(np.linalg.norm(got - ref) / den) if den > 0 else 0.0
    ok = bool(np.all(np.isfinite(got)) and max_abs <= TOL[0] and fro <= TOL[1])
    return {"what": what, "max_abs": max_abs, "fro_rel": fro, "ok": ok}


def replay(words, N_B, R, MBR):
    ref = oracle.Allocator(N_B, R, MBR)
    i, n_ops = 0, 0
    while i < len(words):
        seq, kind, n, status = words[i:i + 4]
        ids = words[i + 4:i + 4 + n]
        if kind == 1:
            st = ref.alloc(ids, words[i + 4 + n:i + 4 + 2 * n])
            i += 4 + 2 * n
        else:
            st = ref.free(ids)
            i += 4 + n
        assert st == status, f"op {seq}: device status {status}, replay {st}"
        assert seq == n_ops, "op log out of linearisation order"
        n_ops += 1
    return ref, n_ops


def nearest_rank_(vals, p):
    vals = sorted(vals)
    return vals[max(1, math.ceil(p * len(vals))) - 1] if vals else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=2000)
    ap.add_argument("--lam", type=float, default=3.0)
    ap.add_argument("--layers", type=int, default=27)
    ap.add_argument("--blocks", type=int, default=3072)
    ap.add_argument("--x", type=float, default=50.0, help="prefill SM percent (y = 100 - x)")
    ap.add_argument("--samples", type=int, default=10)
    ap.add_argument("--max-iters", type=int, default=100000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--expanded", action="store_true",
                    help="expanded-form MLA prefill (semipd_prefill_mla_expanded, reading R32)")
    ap.add_argument("--controller", action="store_true",
                    help="N1: adjust (x, y) every --window iterations with Alg. 1 + the Eq. 4 fit")
    ap.add_argument("--window", type=int, default=100)
    ap.add_argument("--ttft-slo", type=float, default=0.25, help="seconds (attention-only clock)")
    ap.add_argument("--tpot-slo", type=float, default=0.0045, help="seconds (attention-only clock)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    shape = synth.CFG5_MLA
    L, Hq, dk, dv, bs = args.layers, shape.num_q_heads, shape.head_dim_k, shape.head_dim_v, 64
    R, MBR = 1024, (8192 + 2048) // bs + 2
    pool = KVPool(PoolConfig(L, args.blocks, bs, 1, dk, dv, R, MBR, kv_shared=True,
                             oplog_words=1 << 22), dev)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    for l in range(L):
        pool.views(l)[0].normal_(generator=g)
    eng = CoRunEngine(pool, Hq, shape.softmax_scale, partition=(args.x, 100.0 - args.x), seed=5,
                      mla_expanded=args.expanded)
    pre_keys = 0  # sum over iterations of the prefill calls' keys (P + C), for the expanded flops
    trace = synth.mla_trace(args.requests, args.lam, seed=5)
    last_arrival = trace[-1].arrival_iter
    sample_its = set(int(x) for x in np.linspace(5, max(6, last_arrival), args.samples))
    stats, parity, idx = [], [], 0
    # latency bookkeeping on a device clock: the sum of measured iteration times
    now, arrive_t, first_dec_t = 0.0, {}, {}
    ttft, tpot, win_ttft, win_tpot, splits = {}, {}, [], [], []
    x_cur, y_cur = args.x, 100.0 - args.x
    ctl = None
    if args.controller:
        from paper_2504_19867_b200.controller import (ControllerConfig, Observation, SloConfig,
                                                      SloController, nearest_rank)
        ctl = SloController(SloConfig(args.ttft_slo, args.tpot_slo, 0.9),
                            ControllerConfig(window_size=args.window))
    t0 = time.perf_counter()
    while (idx < len(trace) or not eng.idle) and eng.it < args.max_iters:
        arr = []
        while idx < len(trace) and trace[idx].arrival_iter <= eng.it:
            arr.append(trace[idx])
            idx += 1
        sample = eng.it in sample_its
        if sample:
            torch.cuda.synchronize()
            k_pre = bits(pool.views(0)[0])  # layer-0 latent pool before this iteration
        for r in arr:
            arrive_t[r.rid] = now
        s, plan = eng.step(arr)
        stats.append(s)
        pre_keys += sum(ch + pf for _, ch, pf in plan.prefill)
        now += s.t_iter_ms / 1e3
        for r, ch, pf in plan.prefill:
            if r.prefilled == r.input_len and r.trace_id not in ttft:
                ttft[r.trace_id] = now - arrive_t[r.trace_id]
                win_ttft.append(ttft[r.trace_id])
        for r, _ in plan.decode:
            if r.generated == 1:
                first_dec_t[r.trace_id] = now
            if r.slot < 0 and r.generated == r.output_len:  # finished this iteration
                tp = (now - first_dec_t[r.trace_id]) / max(1, r.output_len - 1)
                tpot[r.trace_id] = tp
                win_tpot.append(tp)
        if ctl is not None and s.it > 0 and s.it % args.window == 0:
            p_tt = nearest_rank(win_ttft, 0.9)
            p_tp = nearest_rank(win_tpot, 0.9)
            ctl.update_estimate_model(Observation(100 * x_cur / (x_cur + y_cur),
                                                  100 * y_cur / (x_cur + y_cur), p_tt, p_tp))
            nx, ny = ctl.adjust(s.it, x_cur, y_cur, p_tt, p_tp)
            splits.append({"it": s.it, "x": x_cur, "y": y_cur, "p90_ttft_s": p_tt, "p90_tpot_s": p_tp,
                           "next": [nx, ny]})
            if (nx, ny) != (x_cur, y_cur):
                x_cur, y_cur = nx, ny
                pool.set_partition(x_cur, y_cur)  # adopted at each phase's next launch (R15)
            win_ttft, win_tpot = [], []
        if sample and (plan.prefill or plan.decode):
            bt = pool.views(0)[2].cpu().numpy()
            rec = {"it": s.it}
            kp = k_pre.copy()
            if plan.prefill:
                T = s.prefill_tokens
                cu = [0]
                for _, ch, _ in plan.prefill:
                    cu.append(cu[-1] + ch)
                mask = np.zeros(T, np.uint8)
                mask[::64] = 1
                mask[-1] = 1
                rids = [r.slot if r.slot >= 0 else -1 for r, _, _ in plan.prefill]
                pfx = [pf for _, _, pf in plan.prefill]
                if args.expanded:
                    ref = oracle.prefill_mla_expanded(
                        bits(eng.q_pre[:T]), bits(eng.k_pre[:T, 0]), kp.reshape(kp.shape[0], 1, bs, dk),
                        bt, cu, rids, pfx, bits(eng.w_uk[0]), bits(eng.w_uv[0]), 1 / math.sqrt(192),
                        rows_mask=mask)
                else:
                    ref = oracle.prefill(bits(eng.q_pre[:T]), bits(eng.k_pre[:T]), None, kp, None, bt, cu,
                                         rids, pfx, shape.softmax_scale, kv_shared=True, rows_mask=mask,
                                         dv=dv)
                got = eng.o_pre[0][:T].float().cpu().double().numpy()
                sel = mask.astype(bool)
                rec["prefill"] = check(got[sel], ref[sel], f"it {s.it} prefill rows")
            live = [(j, r, ctx) for j, (r, ctx) in enumerate(plan.decode) if r.slot >= 0][:16]
            if live:
                sel = [j for j, _, _ in live]
                ref = oracle.decode(bits(eng.q_dec[sel]), bits(eng.k_dec[sel]), None, kp, None, bt,
                                    [r.slot for _, r, _ in live], [ctx for _, _, ctx in live],
                                    shape.softmax_scale, kv_shared=True, dv=dv)
                got = eng.o_dec[0][sel].float().cpu().double().numpy()
                rec["decode"] = check(got, ref, f"it {s.it} decode ({len(live)} requests)")
            parity.append(rec)
            print(json.dumps(rec), flush=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    words, dropped = pool.oplog()
    ref, n_ops = replay(words, args.blocks, R, MBR) if dropped == 0 else (None, -1)
    bt, nb = pool.views(0)[2].cpu().numpy(), pool.views(0)[3].cpu().numpy()
    tables_ok = ref is not None and bool(np.array_equal(bt, ref.bt) and np.array_equal(nb, ref.nblk))
    free_now, min_free = pool.stats()
    fl_pair = 2.0 * Hq * (dk + dv)
    t_att = sum(max(x.t_prefill_ms, x.t_decode_ms) for x in stats) / 1e3
    t_iter = sum(x.t_iter_ms for x in stats) / 1e3
    pre_tok = sum(x.prefill_tokens for x in stats)
    dec_tok = sum(x.decode_reqs for x in stats)
    if args.expanded:  # causal MHA at dqk 192 / dv 128 + the up-projection of every key
        pre_fl = (sum(x.prefill_pairs for x in stats) * 2.0 * Hq * (192 + 128) +
                  pre_keys * 2.0 * 512 * 2 * Hq * 128) * L
    else:
        pre_fl = sum(x.prefill_pairs for x in stats) * fl_pair * L
    dec_bytes = sum(x.decode_keys for x in stats) * dk * 2 * L
    t_pre = sum(x.t_prefill_ms for x in stats) / 1e3
    t_dec = sum(x.t_decode_ms for x in stats) / 1e3
    summary = {
        "config": f"cfg5 DeepSeek-V2-Lite MLA attention ({L} layers, 16 heads, latent 576/512, bs 64, "
                  f"{args.blocks}-block pool), Poisson({args.lam})/iteration trace of {args.requests} "
                  f"requests (seed 5), 2048-token chunked prefill, decode cap 512, split "
                  f"({args.x:g},{100 - args.x:g})",
        "prefill_form": "expanded (R32)" if args.expanded else "absorbed",
        "iterations": len(stats), "finished": len(eng.finished),
        "preemptions": sum(x.preempted for x in stats),
        "prefill_tokens": pre_tok, "decode_tokens": dec_tok,
        "attention_s": t_att, "iteration_device_s": t_iter, "wall_s": wall,
        "tokens_per_s_attention": (pre_tok + dec_tok) / t_att if t_att else None,
        "prefill_tflops_while_running": pre_fl / t_pre / 1e12 if t_pre else None,
        "decode_gbs_while_running": dec_bytes / t_dec / 1e9 if t_dec else None,
        "mean_decode_batch": float(np.mean([x.decode_reqs for x in stats if x.decode_reqs] or [0])),
        "max_decode_batch": max(x.decode_reqs for x in stats),
        "alloc_calls": sum(x.alloc_calls for x in stats), "free_calls": sum(x.free_calls for x in stats),
        "op_log_ops": n_ops, "op_log_dropped": dropped, "op_log_replay_tables_equal": tables_ok,
        "pool_blocks": args.blocks, "pool_min_free": min_free,
        "pool_high_water_blocks": args.blocks - min_free, "pool_free_end": free_now,
        "p90_ttft_s": nearest_rank_(list(ttft.values()), 0.9),
        "p90_tpot_s": nearest_rank_(list(tpot.values()), 0.9),
        "controller": ({"ttft_slo_s": args.ttft_slo, "tpot_slo_s": args.tpot_slo, "window": args.window,
                        "trajectory": splits,
                        "ttft_slo_attainment": sum(v <= args.ttft_slo for v in ttft.values()) / max(1, len(ttft)),
                        "tpot_slo_attainment": sum(v <= args.tpot_slo for v in tpot.values()) / max(1, len(tpot)),
                        "model": None if ctl is None else ctl.model.__dict__}
                       if args.controller else None),
        "parity_samples": parity,
        "parity_all_ok": all(v["ok"] for rec in parity for k, v in rec.items() if k != "it"),
    }
    print(json.dumps({k: v for k, v in summary.items() if k != "parity_samples"}))
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"summary": summary,
                       "iterations": [s.__dict__ for s in stats]}, f)
    return 0 if (summary["parity_all_ok"] and tables_ok) else 1


if __name__ == "__main__":
    sys.exit(main())
