"""One-GPU emulation of the cfg-3 decode step at TP = 2/4/8 (ranks = streams of one process,
graph replay): per-rank decode (B 64, ctx 2048) followed by its head gather, three ways:
  none   : decode only (no gather),
  copy   : decode, then semipd_peer_gather (copy-engine pushes + 2 handshakes),
  fused  : ready handshake, decode with epilogue peer stores, landed handshake.
All ranks share one GPU (HBM, SMs, copy engines), so absolute times are not a multi-GPU
number; the differences show what each gather adds on the device."""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from paper_2504_19867_b200 import lib, tp  # noqa: E402
from test_gpu_peer_gather import _decode_pool  # noqa: E402

dev = torch.device("cuda", 0)
L = lib()
shape = synth.AttnShape("llama3-70b", 64, 8, 128, 128, 64, torch.bfloat16)
B, C = 64, 2048
ctx = [C] * B
cd = synth.decode_case(shape, ctx, seed=5050)
i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
rid, ctx_d = i32(list(range(B))), i32(ctx)
vp = ctypes.c_void_p
for tpn in (2, 4, 8):
    hq = 64 // tpn
    pools, outs, flags, streams, wss, ins, locs = [], [], [], [], [], [], []
    for r in range(tpn):
        pools.append(_decode_pool(shape, ctx, cd, tp.head_range(8, tpn, r), dev))
        outs.append(torch.zeros(64, B, 128, dtype=torch.bfloat16, device=dev))
        flags.append(torch.zeros(2 * tpn, dtype=torch.int32, device=dev))
        streams.append(torch.cuda.Stream(dev))
        wss.append(pools[r].new_decode_workspace(B, hq, C))
        ql, qh = tp.head_range(64, tpn, r)
        kl, kh = tp.head_range(8, tpn, r)
        ins.append((cd.q[:, ql:qh].contiguous().to(dev), cd.k_new[:, kl:kh].contiguous().to(dev),
                    cd.v_new[:, kl:kh].contiguous().to(dev), ql, qh))
        locs.append(torch.empty(hq, B, 128, dtype=torch.bfloat16, device=dev))
    fl = (vp * tpn)(*[f.data_ptr() for f in flags])
    shard = hq * B * 128 * 2
    torch.cuda.synchronize()

    def round_(mode):
        main = torch.cuda.current_stream(dev)
        for s in streams:
            s.wait_stream(main)
        for r in range(tpn):
            qs, ks, vs, ql, qh = ins[r]
            s = streams[r]
            cs = vp(s.cuda_stream)
            if mode == "fused":
                assert L.semipd_peer_handshake(fl, vp(flags[r].data_ptr()), tpn, r, 0, cs) == 0
            out = outs[r][ql:qh] if mode == "fused" else locs[r]
            pools[r].decode_attn(0, qs, ks, vs, rid, ctx_d, C, shape.softmax_scale, out, wss[r],
                                 out_head_major=True, stream=s)
            if mode == "fused":
                assert L.semipd_peer_handshake(fl, vp(flags[r].data_ptr()), tpn, r, 1, cs) == 0
            elif mode == "copy":
                dsts = (vp * tpn)(*[outs[k].data_ptr() + r * shard for k in range(tpn)])
                assert L.semipd_peer_gather(vp(locs[r].data_ptr()), shard, dsts, fl,
                                            vp(flags[r].data_ptr()), tpn, r, cs) == 0
        for s in streams:
            main.wait_stream(s)

    res = {"phase": "decode", "tp": tpn, "B": B, "ctx": C}
    for mode in ("none", "copy", "fused"):
        for r in range(tpn):
            pools[r].set_decode_peers([outs[k].data_ptr() + r * shard for k in range(tpn) if k != r]
                                      if mode == "fused" else [], B)
        round_(mode)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            round_(mode)
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[mode + "_us"] = e0.elapsed_time(e1) * 1e3 / 20
    print(json.dumps(res), flush=True)
    del pools, outs, wss
    torch.cuda.empty_cache()

# ---- prefill: a 2k chunk (P = 0) per rank, the same three ways
from paper_2504_19867_b200 import KVPool, PoolConfig  # noqa: E402
Cp = 2048
pc = synth.prefill_case(shape, [Cp], [0], seed=5051)
cu, rid1, pre0 = i32([0, Cp]), i32([0]), i32([0])
nbp = Cp // 64
for tpn in (2, 4, 8):
    hq = 64 // tpn
    pools, outs, flags, streams, ins, locs = [], [], [], [], [], []
    for r in range(tpn):
        kl, kh = tp.head_range(8, tpn, r)
        ql, qh = tp.head_range(64, tpn, r)
        pool = KVPool(PoolConfig(1, nbp + 1, 64, kh - kl, 128, 128, 1, nbp), dev)
        pool.alloc_blocks(i32([0]), i32([nbp]))
        pools.append(pool)
        outs.append(torch.zeros(64, Cp, 128, dtype=torch.bfloat16, device=dev))
        flags.append(torch.zeros(2 * tpn, dtype=torch.int32, device=dev))
        streams.append(torch.cuda.Stream(dev))
        ins.append((pc.q[:, ql:qh].contiguous().to(dev), pc.k_new[:, kl:kh].contiguous().to(dev),
                    pc.v_new[:, kl:kh].contiguous().to(dev), ql, qh))
        locs.append(torch.empty(hq, Cp, 128, dtype=torch.bfloat16, device=dev))
    fl = (vp * tpn)(*[f.data_ptr() for f in flags])
    shard = hq * Cp * 128 * 2
    torch.cuda.synchronize()

    def round_p(mode):
        main = torch.cuda.current_stream(dev)
        for s in streams:
            s.wait_stream(main)
        for r in range(tpn):
            qs, ks, vs, ql, qh = ins[r]
            s = streams[r]
            cs = vp(s.cuda_stream)
            if mode == "fused":
                assert L.semipd_peer_handshake(fl, vp(flags[r].data_ptr()), tpn, r, 0, cs) == 0
            out = outs[r][ql:qh] if mode == "fused" else locs[r]
            pools[r].prefill_attn(0, qs, ks, vs, cu, rid1, pre0, Cp, Cp, shape.softmax_scale, out,
                                  out_head_major=True, stream=s)
            if mode == "fused":
                assert L.semipd_peer_handshake(fl, vp(flags[r].data_ptr()), tpn, r, 1, cs) == 0
            elif mode == "copy":
                dsts = (vp * tpn)(*[outs[k].data_ptr() + r * shard for k in range(tpn)])
                assert L.semipd_peer_gather(vp(locs[r].data_ptr()), shard, dsts, fl,
                                            vp(flags[r].data_ptr()), tpn, r, cs) == 0
        for s in streams:
            main.wait_stream(s)

    res = {"phase": "prefill", "tp": tpn, "C": Cp}
    for mode in ("none", "copy", "fused"):
        for r in range(tpn):
            pools[r].set_prefill_peers([outs[k].data_ptr() + r * shard for k in range(tpn) if k != r]
                                       if mode == "fused" else [], Cp)
        round_p(mode)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            round_p(mode)
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[mode + "_us"] = e0.elapsed_time(e1) * 1e3 / 20
    print(json.dumps(res), flush=True)
    del pools, outs
    torch.cuda.empty_cache()
