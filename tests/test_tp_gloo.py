"""Multi-process (gloo, world size 2, CPU) tests of the TP-by-KV-head host logic:
head sharding, per-phase process groups, head-major all-gather.
The per-rank attention is the oracle on the rank's head shard (no GPU here); the
gathered result must equal the unsharded oracle exactly (attention is independent
per head)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2504_19867_b200 import tp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pool_for(shape, case_k, case_v, ctx, bs, heads):
    """Oracle-side pool holding only `heads` (a kv-head slice) for each request."""
    B = len(ctx)
    nb = [c // bs + 1 for c in ctx]
    bt = np.full((B, max(nb)), -1, np.int32)
    u = 0
    for b in range(B):
        bt[b, :nb[b]] = np.arange(u, u + nb[b])
        u += nb[b]
    lo, hi = heads
    kp = np.zeros((u, hi - lo, bs, shape.head_dim_k), np.uint16)
    vp = np.zeros((u, hi - lo, bs, shape.head_dim_v), np.uint16)
    for b in range(B):
        kb = synth.bits(case_k[b][:, lo:hi])
        vb = synth.bits(case_v[b][:, lo:hi])
        for j in range(ctx[b]):
            kp[bt[b, j // bs], :, j % bs] = kb[j]
            vp[bt[b, j // bs], :, j % bs] = vb[j]
    return kp, vp, bt


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        groups = tp.PhaseGroups.create(backend="gloo")
        shape = synth.AttnShape("70b-mini", 8, 4, 32, 32, 16, torch.bfloat16)
        ctx = [5, 40, 17]
        dc = synth.decode_case(shape, ctx, seed=303)
        # ---- decode shard
        kl, kh = tp.head_range(shape.num_kv_heads, ws, rank)
        ql, qh = tp.head_range(shape.num_q_heads, ws, rank)
        qs, ks, vs = tp.shard_qkv(dc.q, dc.k_new, dc.v_new, ws, rank)
        kp, vp, bt = _pool_for(shape, dc.k_ctx, dc.v_ctx, ctx, 16, (kl, kh))
        out = oracle.decode(synth.bits(qs), synth.bits(ks), synth.bits(vs), kp, vp, bt,
                            [0, 1, 2], ctx, shape.softmax_scale)          # [B, Hq/tp, dv]
        local = torch.from_numpy(out).permute(1, 0, 2).contiguous()      # head-major
        full = torch.empty(shape.num_q_heads, len(ctx), shape.head_dim_v, dtype=torch.float64)
        tp.gather_heads(local, full, groups.decode)
        # ---- prefill shard on the other phase group
        pc = synth.prefill_case(shape, [23], [0], seed=304)
        qs2, ks2, vs2 = tp.shard_qkv(pc.q, pc.k_new, pc.v_new, ws, rank)
        kpp = np.zeros((4, kh - kl, 16, 32), np.uint16)
        vpp = np.zeros_like(kpp)
        outp = oracle.prefill(synth.bits(qs2), synth.bits(ks2), synth.bits(vs2), kpp, vpp,
                              np.array([[0, 1, -1, -1]], np.int32), [0, 23], [0], [0],
                              shape.softmax_scale)
        localp = torch.from_numpy(outp).permute(1, 0, 2).contiguous()
        fullp = torch.empty(shape.num_q_heads, 23, 32, dtype=torch.float64)
        tp.gather_heads(localp, fullp, groups.prefill)
        if rank == 0:
            q.put((full.numpy(), fullp.numpy()))
    finally:
        dist.destroy_process_group()


def test_tp2_gather_equals_unsharded():
    ctx_ = mp.get_context("spawn")
    qq = ctx_.Queue()
    port = _free_port()
    procs = [ctx_.Process(target=_worker, args=(r, 2, port, qq)) for r in range(2)]
    for p in procs:
        p.start()
    full, fullp = qq.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shape = synth.AttnShape("70b-mini", 8, 4, 32, 32, 16, torch.bfloat16)
    ctx = [5, 40, 17]
    dc = synth.decode_case(shape, ctx, seed=303)
    kp, vp, bt = _pool_for(shape, dc.k_ctx, dc.v_ctx, ctx, 16, (0, 4))
    ref = oracle.decode(synth.bits(dc.q), synth.bits(dc.k_new), synth.bits(dc.v_new), kp, vp, bt,
                        [0, 1, 2], ctx, shape.softmax_scale)
    np.testing.assert_array_equal(full.transpose(1, 0, 2), ref)
    pc = synth.prefill_case(shape, [23], [0], seed=304)
    kpp = np.zeros((4, 4, 16, 32), np.uint16)
    refp = oracle.prefill(synth.bits(pc.q), synth.bits(pc.k_new), synth.bits(pc.v_new), kpp,
                          np.zeros_like(kpp), np.array([[0, 1, -1, -1]], np.int32), [0, 23], [0],
                          [0], shape.softmax_scale)
    np.testing.assert_array_equal(fullp.transpose(1, 0, 2), refp)


def test_head_range():
    assert tp.head_range(64, 8, 3) == (24, 32)
    assert tp.head_range(8, 8, 7) == (7, 8)
    with pytest.raises(ValueError):
        tp.head_range(8, 3, 0)
