"""TP by KV head on >= 2 real GPUs (§4.5): one process per GPU, one
process group per phase (NCCL, each communicator capped to 4 CTAs), cfg-3 shapes (Hq 64 /
Hkv 8 split over the ranks).  Every rank runs decode and prefill attention on its head shard
and the head-major outputs are all-gathered three ways — NCCL all_gather_into_tensor, the
copy-engine peer gather over NVLink (semipd_peer_gather), and the epilogue peer stores
(semipd_set_decode_peers / semipd_set_prefill_peers) — and each gathered result is compared
with the fp64 oracle over all 64 heads.  Skipped on a one-GPU box (the round's driver boxes);
the same host logic runs under gloo in tests/test_tp_gloo.py."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    try:
        import numpy as np
        import torch.distributed as dist

        import oracle
        import synth
        from harness import compare, np_bits
        from paper_2504_19867_b200 import KVPool, PoolConfig, tp
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dev = torch.device("cuda", rank)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        groups = tp.PhaseGroups.create(backend="nccl", max_ctas=4)
        full = synth.AttnShape("llama3-70b", 64, 8, 128, 128, 64, torch.bfloat16)
        ctx, C, P = [300, 2048, 4500, 64], 700, 300
        B = len(ctx)
        dc = synth.decode_case(full, ctx, seed=5000)
        pc = synth.prefill_case(full, [C], [P], seed=5001)
        kl, kh = tp.head_range(8, world, rank)
        ql, qh = tp.head_range(64, world, rank)
        i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
        bs = 64
        nb_d = [c // bs + 1 for c in ctx]
        nb_p = -(-(C + P) // bs)
        pool = KVPool(PoolConfig(1, sum(nb_d) + nb_p + 2, bs, kh - kl, 128, 128, B + 1,
                                 max(max(nb_d), nb_p)), dev)
        for b, n in enumerate(nb_d):
            pool.alloc_blocks(i32([b]), i32([n]))
        pool.alloc_blocks(i32([B]), i32([nb_p]))
        K, V, BT, _ = pool.views(0)
        bt = BT.cpu()
        for rid, kt, vt in [(b, dc.k_ctx[b], dc.v_ctx[b]) for b in range(B)] + \
                           [(B, pc.k_prefix[0], pc.v_prefix[0])]:
            pos = torch.arange(kt.shape[0])
            blk = bt[rid].long()[pos // bs].to(dev)
            K[blk, :, (pos % bs).to(dev)] = kt[:, kl:kh].to(dev)
            V[blk, :, (pos % bs).to(dev)] = vt[:, kl:kh].to(dev)
        sc = full.softmax_scale
        ws = pool.new_decode_workspace(B, qh - ql, max(ctx))
        dq = dc.q[:, ql:qh].contiguous().to(dev)
        dk_, dv_ = dc.k_new[:, kl:kh].contiguous().to(dev), dc.v_new[:, kl:kh].contiguous().to(dev)
        pq = pc.q[:, ql:qh].contiguous().to(dev)
        pk_, pv_ = pc.k_new[:, kl:kh].contiguous().to(dev), pc.v_new[:, kl:kh].contiguous().to(dev)
        ref_d = np.concatenate([oracle.attention_contig(
            np_bits(dc.q[b:b + 1]), np_bits(torch.cat([dc.k_ctx[b], dc.k_new[b:b + 1]])),
            np_bits(torch.cat([dc.v_ctx[b], dc.v_new[b:b + 1]])), -1, sc) for b in range(B)])
        ref_p = oracle.attention_contig(np_bits(pc.q), np_bits(torch.cat([pc.k_prefix[0], pc.k_new])),
                                        np_bits(torch.cat([pc.v_prefix[0], pc.v_new])), P, sc)
        hm = lambda t: t.float().cpu().double().numpy().transpose(1, 0, 2)  # noqa: E731

        def run(out_d, out_p):
            # decode appends / prefill rewrites the same bits every time: reruns are idempotent
            pool.decode_attn(0, dq, dk_, dv_, i32(range(B)), i32(ctx), max(ctx), sc, out_d, ws,
                             out_head_major=True)
            pool.prefill_attn(0, pq, pk_, pv_, i32([0, C]), i32([B]), i32([P]), C, C, sc, out_p,
                              out_head_major=True)

        # 1. NCCL all-gather on the phase groups
        od = torch.empty(qh - ql, B, 128, dtype=torch.bfloat16, device=dev)
        op = torch.empty(qh - ql, C, 128, dtype=torch.bfloat16, device=dev)
        run(od, op)
        gd = torch.empty(64, B, 128, dtype=torch.bfloat16, device=dev)
        gp = torch.empty(64, C, 128, dtype=torch.bfloat16, device=dev)
        tp.gather_heads(od, gd, groups.decode)
        tp.gather_heads(op, gp, groups.prefill)
        torch.cuda.synchronize()
        compare(hm(gd), ref_d, torch.bfloat16, f"nccl decode gather rank {rank}")
        compare(hm(gp), ref_p, torch.bfloat16, f"nccl prefill gather rank {rank}")
        # 2. copy-engine peer gather over NVLink
        pg_d = tp.PeerGather((64, B, 128), torch.bfloat16, groups.decode, dev)
        pg_p = tp.PeerGather((64, C, 128), torch.bfloat16, groups.prefill, dev)
        pg_d(od)
        pg_p(op)
        torch.cuda.synchronize()
        compare(hm(pg_d.out()), ref_d, torch.bfloat16, f"peer decode gather rank {rank}")
        compare(hm(pg_p.out()), ref_p, torch.bfloat16, f"peer prefill gather rank {rank}")
        # 3. epilogue peer stores (real NVLink peers)
        pg_d.out().fill_(float("nan"))
        pg_p.out().fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        pool.set_decode_peers(pg_d.peer_shard_ptrs(), B)
        pool.set_prefill_peers(pg_p.peer_shard_ptrs(), C)
        pg_d.handshake(0)
        pg_p.handshake(0)
        run(pg_d.local_view(), pg_p.local_view())
        pg_d.handshake(1)
        pg_p.handshake(1)
        torch.cuda.synchronize()
        compare(hm(pg_d.out()), ref_d, torch.bfloat16, f"fused decode gather rank {rank}")
        compare(hm(pg_p.out()), ref_p, torch.bfloat16, f"fused prefill gather rank {rank}")
        pool.set_decode_peers([])
        pool.set_prefill_peers([])
        dist.barrier()
        pg_d.close()
        pg_p.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover (reported to the parent)
        import traceback
        q.put((rank, "".join(traceback.format_exception(e))[-3000:]))


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs (one process per GPU)")
def test_tp2_nccl_peer_and_fused_gathers_match_oracle():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=900) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
