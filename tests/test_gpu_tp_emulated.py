"""TP-by-KV-head emulated on one GPU: each rank's head shard runs
on its own pool; the head-major shard outputs concatenated in rank order must equal
the unsharded run BITWISE (every work unit is per kv head, so sharding changes no
arithmetic), and match the oracle."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from harness import compare, np_bits
from paper_2504_19867_b200 import KVPool, PoolConfig, tp

pytestmark = pytest.mark.gpu


def _run(shape, ctx, chunk, case_d, case_p, heads_kv, heads_q, dev):
    """Decode + prefill on a pool holding kv heads [heads_kv) only; head-major outputs."""
    kl, kh = heads_kv
    ql, qh = heads_q
    bs = shape.block_size
    nb = [c // bs + 1 for c in ctx]
    nbp = -(-chunk // bs)
    cfg = PoolConfig(1, sum(nb) + nbp + 2, bs, kh - kl, 128, 128, len(ctx) + 1, max(max(nb), nbp))
    pool = KVPool(cfg, dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    for b, n in enumerate(nb):
        pool.alloc_blocks(i32([b]), i32([n]))
    pool.alloc_blocks(i32([len(ctx)]), i32([nbp]))
    K, V, BT, _ = pool.views(0)
    bt = BT.cpu().numpy()
    for b, c in enumerate(ctx):
        pos = torch.arange(c)
        blk = torch.from_numpy(bt[b]).long()[pos // bs].to(dev)
        K[blk, :, (pos % bs).to(dev)] = case_d.k_ctx[b][:, kl:kh].to(dev)
        V[blk, :, (pos % bs).to(dev)] = case_d.v_ctx[b][:, kl:kh].to(dev)
    sc = shape.softmax_scale
    B = len(ctx)
    od = torch.empty(qh - ql, B, 128, dtype=torch.bfloat16, device=dev)
    ws = pool.new_decode_workspace(B, qh - ql, max(ctx))
    pool.decode_attn(0, case_d.q[:, ql:qh].contiguous().to(dev),
                     case_d.k_new[:, kl:kh].contiguous().to(dev),
                     case_d.v_new[:, kl:kh].contiguous().to(dev), i32(list(range(B))), i32(ctx),
                     max(ctx), sc, od, ws, out_head_major=True)
    op = torch.empty(qh - ql, chunk, 128, dtype=torch.bfloat16, device=dev)
    pool.prefill_attn(0, case_p.q[:, ql:qh].contiguous().to(dev),
                      case_p.k_new[:, kl:kh].contiguous().to(dev),
                      case_p.v_new[:, kl:kh].contiguous().to(dev), i32([0, chunk]), i32([B]),
                      i32([0]), chunk, chunk, sc, op, out_head_major=True)
    torch.cuda.synchronize()
    return od.cpu(), op.cpu()


@pytest.mark.parametrize("tpn", [2, 4, 8])
def test_tp_shards_concat_equal_unsharded(tpn):
    dev = torch.device("cuda", 0)
    shape = synth.AttnShape("llama3-70b", 64, 8, 128, 128, 64, torch.bfloat16)  # cfg3 shapes
    ctx, chunk = [300, 2048, 4500], 700
    cd = synth.decode_case(shape, ctx, seed=3030)
    cp = synth.prefill_case(shape, [chunk], [0], seed=3031)
    full_d, full_p = _run(shape, ctx, chunk, cd, cp, (0, 8), (0, 64), dev)
    parts_d, parts_p = [], []
    for r in range(tpn):
        od, op = _run(shape, ctx, chunk, cd, cp, tp.head_range(8, tpn, r),
                      tp.head_range(64, tpn, r), dev)
        parts_d.append(od)
        parts_p.append(op)
    assert torch.equal(torch.cat(parts_d), full_d)
    assert torch.equal(torch.cat(parts_p), full_p)
    # and the unsharded run matches the oracle (decode rows)
    bs = 64
    nb = [c // bs + 1 for c in ctx]
    bt = np.full((3, max(nb)), -1, np.int32)
    u = 0
    for b in range(3):
        bt[b, :nb[b]] = np.arange(u, u + nb[b])
        u += nb[b]
    kp = np.zeros((u, 8, bs, 128), np.uint16)
    vp = np.zeros_like(kp)
    for b, c in enumerate(ctx):
        kb, vb = np_bits(cd.k_ctx[b]), np_bits(cd.v_ctx[b])
        for j in range(c):
            kp[bt[b, j // bs], :, j % bs] = kb[j]
            vp[bt[b, j // bs], :, j % bs] = vb[j]
    ref = oracle.decode(np_bits(cd.q), np_bits(cd.k_new), np_bits(cd.v_new), kp, vp, bt,
                        [0, 1, 2], ctx, shape.softmax_scale)
    compare(full_d.float().double().numpy().transpose(1, 0, 2), ref, torch.bfloat16, "tp decode")
