"""Copy-engine peer all-gather of head-major shards (``semipd_peer_gather``; SURVEY §8(e),
§8(f) N2).  Two processes share the one GPU of the box: IPC handles open across processes
on the same device exactly as across NVLink peers, and the copies / stream memory
operations are the same calls.  Checks are bitwise: a gather moves bytes.

- generic: several rounds of seeded shards with the entry handshake; every rank's gathered
  buffer equals the rank-order concatenation; a shard written in place (local_view) skips
  the local copy and is gathered too;
- kernel outputs: each rank's head-major decode / prefill output for its KV-head shard
  (cfg3 shapes, Hkv 8 -> 4 per rank), gathered, equals the unsharded run bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from harness import compare, np_bits
from paper_2504_19867_b200 import INVALID, SemipdError

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard(rnd, rank, shape_local):
    g = torch.Generator().manual_seed(1000 * rnd + rank)
    return torch.randn(*shape_local, generator=g).to(torch.bfloat16)


def _generic_worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2504_19867_b200 import tp
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    try:
        full = (8, 37, 64)
        loc = (full[0] // ws,) + full[1:]
        pg = tp.PeerGather(full, torch.bfloat16, dist.group.WORLD, dev, n_bufs=2)
        s = torch.cuda.Stream(dev)
        bad = []
        for rnd in range(6):
            buf = rnd % 2
            with torch.cuda.stream(s):
                if rnd % 3 == 2:  # in place: the shard is already in the gathered buffer
                    pg.local_view(buf).copy_(_shard(rnd, rank, loc).to(dev))
                    out = pg(pg.local_view(buf), buf=buf, stream=s)
                else:
                    out = pg(_shard(rnd, rank, loc).to(dev), buf=buf, stream=s)
                got = out.cpu()
            s.synchronize()
            want = torch.cat([_shard(rnd, k, loc) for k in range(ws)])
            if not torch.equal(got.view(torch.int16), want.view(torch.int16)):
                bad.append(rnd)
        # captured once into a CUDA graph, replayed with new shard contents (the flag
        # operations carry no per-call value, so every replay synchronises afresh)
        torch.cuda.synchronize()
        src = torch.empty(loc, dtype=torch.bfloat16, device=dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            pg(src, buf=0, stream=torch.cuda.current_stream())
        for rnd in range(6, 10):
            src.copy_(_shard(rnd, rank, loc).to(dev))
            g.replay()
            got = pg.out(0).cpu()
            want = torch.cat([_shard(rnd, k, loc) for k in range(ws)])
            if not torch.equal(got.view(torch.int16), want.view(torch.int16)):
                bad.append(rnd)
        torch.cuda.synchronize()
        dist.barrier()
        pg.close()
        q.put((rank, bad, pg.calls))
    except Exception as e:  # report instead of leaving the parent waiting
        q.put((rank, repr(e), -1))
        raise
    finally:
        dist.destroy_process_group()


def _run_two(target, timeout):
    """Start two daemon workers; collect one result each; never leave a worker behind (a
    worker whose peer died would wait on its stream forever)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, 2, port, q), daemon=True) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=timeout) for _ in procs]
        for p in procs:
            p.join(timeout=60)
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    return res, procs


def test_peer_gather_generic_two_processes():
    res, procs = _run_two(_generic_worker, 240)
    for rank, bad, calls in res:
        assert bad == [], f"rank {rank}: rounds {bad} gathered wrong bytes"
        assert calls == 7  # 6 eager calls + the one captured
    assert all(p.exitcode == 0 for p in procs)


def _kernel_worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import synth
    from paper_2504_19867_b200 import tp
    from test_gpu_tp_emulated import _run
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    try:
        shape = synth.AttnShape("llama3-70b", 64, 8, 128, 128, 64, torch.bfloat16)
        ctx, chunk = [300, 2048, 4500], 700
        cd = synth.decode_case(shape, ctx, seed=3030)
        cp = synth.prefill_case(shape, [chunk], [0], seed=3031)
        od, op = _run(shape, ctx, chunk, cd, cp, tp.head_range(8, ws, rank),
                      tp.head_range(64, ws, rank), dev)
        groups = tp.PhaseGroups.create(backend="gloo")
        pgd = tp.PeerGather((64, len(ctx), 128), torch.bfloat16, groups.decode, dev)
        pgp = tp.PeerGather((64, chunk, 128), torch.bfloat16, groups.prefill, dev)
        sd, sp = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        with torch.cuda.stream(sd):
            gd = pgd(od.to(dev), stream=sd)
        with torch.cuda.stream(sp):
            gp = pgp(op.to(dev), stream=sp)
        torch.cuda.synchronize()
        gd, gp = gd.cpu(), gp.cpu()
        ok = True
        if rank == 0:
            full_d, full_p = _run(shape, ctx, chunk, cd, cp, (0, 8), (0, 64), dev)
            ok = torch.equal(gd, full_d) and torch.equal(gp, full_p)
        dist.barrier()
        pgd.close()
        pgp.close()
        q.put((rank, ok))
    except Exception as e:
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_peer_gather_kernel_outputs_equal_unsharded():
    res, procs = _run_two(_kernel_worker, 300)
    for rank, ok in res:
        assert ok is True, f"rank {rank}: {ok if isinstance(ok, str) else 'gathered kernel outputs differ from the unsharded run'}"
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_peer_gather_emulated_ranks_one_process(tp):
    """TP ranks emulated as streams of one process (plain device pointers for the peers'
    buffers and flags): bitwise gather, every flag reset afterwards, repeatable."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "scripts"))
    from peer_gather_bench import run
    r = run(tp, (16, 129, 64), iters=3)
    assert r["shard_bytes"] == 16 // tp * 129 * 64 * 2


def _decode_pool(shape, ctx, case, heads_kv, dev):
    """A pool holding kv heads [heads_kv) of the cached contexts (harness bit copies)."""
    from paper_2504_19867_b200 import KVPool, PoolConfig
    kl, kh = heads_kv
    bs = shape.block_size
    nb = [c // bs + 1 for c in ctx]
    pool = KVPool(PoolConfig(1, sum(nb) + 2, bs, kh - kl, 128, 128, len(ctx), max(nb)), dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    for b, n in enumerate(nb):
        pool.alloc_blocks(i32([b]), i32([n]))
    K, V, BT, _ = pool.views(0)
    bt = BT.cpu()
    for b, c in enumerate(ctx):
        pos = torch.arange(c)
        blk = bt[b].long()[pos // bs].to(dev)
        K[blk, :, (pos % bs).to(dev)] = case.k_ctx[b][:, kl:kh].to(dev)
        V[blk, :, (pos % bs).to(dev)] = case.v_ctx[b][:, kl:kh].to(dev)
    return pool


@pytest.mark.parametrize("tpn", [2, 4, 8])
def test_decode_epilogue_peer_stores_emulated(tpn):
    """The TP head gather fused into the decode epilogue (semipd_set_decode_peers +
    semipd_peer_handshake), TP ranks emulated as streams of one process: rank r's decode kernel
    stores its head slice into every rank's gathered buffer; after the landed handshake each
    gathered buffer equals the unsharded decode output bitwise.  Twice, to exercise the flag
    resets and the ready handshake of the second round."""
    import ctypes

    import synth
    from paper_2504_19867_b200 import lib, tp
    dev = torch.device("cuda", 0)
    shape = synth.AttnShape("llama3-70b", 64, 8, 128, 128, 64, torch.bfloat16)
    ctx = [300, 2048, 4500, 64]
    B = len(ctx)
    cd = synth.decode_case(shape, ctx, seed=3040)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    sc = shape.softmax_scale
    # unsharded reference run
    full_pool = _decode_pool(shape, ctx, cd, (0, 8), dev)
    ref = torch.empty(64, B, 128, dtype=torch.bfloat16, device=dev)
    full_pool.decode_attn(0, cd.q.to(dev), cd.k_new.to(dev), cd.v_new.to(dev), i32(list(range(B))),
                          i32(ctx), max(ctx), sc, ref, full_pool.new_decode_workspace(B, 64, max(ctx)),
                          out_head_major=True)
    torch.cuda.synchronize()
    pools, outs, flags, streams, wss = [], [], [], [], []
    for r in range(tpn):
        pools.append(_decode_pool(shape, ctx, cd, tp.head_range(8, tpn, r), dev))
        outs.append(torch.full((64, B, 128), float("nan"), dtype=torch.bfloat16, device=dev))
        flags.append(torch.zeros(2 * tpn, dtype=torch.int32, device=dev))
        streams.append(torch.cuda.Stream(dev))
        wss.append(pools[r].new_decode_workspace(B, 64 // tpn, max(ctx)))
    hq = 64 // tpn
    fl = (ctypes.c_void_p * tpn)(*[f.data_ptr() for f in flags])
    L = lib()
    # every device input exists before the first handshake: a host-to-device copy issued on a
    # rank's stream while it waits for a later rank's flag would block this (single) host thread
    rid, ctx_d = i32(list(range(B))), i32(ctx)
    ins = []
    for r in range(tpn):
        ql, qh = tp.head_range(64, tpn, r)
        kl, kh = tp.head_range(8, tpn, r)
        ins.append((cd.q[:, ql:qh].contiguous().to(dev), cd.k_new[:, kl:kh].contiguous().to(dev),
                    cd.v_new[:, kl:kh].contiguous().to(dev), ql, qh))
    torch.cuda.synchronize()
    for rnd in range(2):
        for o in outs:
            o.fill_(float("nan"))
        torch.cuda.synchronize()
        for r in range(tpn):
            shard = hq * B * 128 * 2
            pools[r].set_decode_peers([outs[k].data_ptr() + r * shard for k in range(tpn) if k != r], B)
        for r in range(tpn):
            qs, ks, vs, ql, qh = ins[r]
            s = streams[r]
            cs = ctypes.c_void_p(s.cuda_stream)
            assert L.semipd_peer_handshake(fl, ctypes.c_void_p(flags[r].data_ptr()), tpn, r, 0, cs) == 0
            # the rank's own slice goes straight into its gathered buffer
            pools[r].decode_attn(0, qs, ks, vs, rid, ctx_d, max(ctx), sc, outs[r][ql:qh], wss[r],
                                 out_head_major=True, stream=s)
            assert L.semipd_peer_handshake(fl, ctypes.c_void_p(flags[r].data_ptr()), tpn, r, 1, cs) == 0
        torch.cuda.synchronize()
        for r in range(tpn):
            assert torch.equal(outs[r].view(torch.int16), ref.view(torch.int16)), (rnd, r)
        assert all(int(f.abs().sum()) == 0 for f in flags)
    # the gathered buffers against the fp64 oracle (the plain definition over each request's
    # contiguous keys: cached context + the appended row), not only against the unsharded run
    ref64 = np.concatenate([oracle.attention_contig(
        np_bits(cd.q[b:b + 1]), np_bits(torch.cat([cd.k_ctx[b], cd.k_new[b:b + 1]])),
        np_bits(torch.cat([cd.v_ctx[b], cd.v_new[b:b + 1]])), -1, sc) for b in range(B)])
    for r in range(tpn):
        compare(outs[r].float().cpu().double().numpy().transpose(1, 0, 2), ref64, torch.bfloat16,
                f"fused decode gather tp{tpn} rank {r}")
    # peers need head-major output
    pools[0].set_decode_peers([outs[1].data_ptr()], B)
    with pytest.raises(Exception):
        pools[0].decode_attn(0, ins[0][0], ins[0][1], ins[0][2], rid, ctx_d, max(ctx), sc,
                             torch.empty(B, hq, 128, dtype=torch.bfloat16, device=dev), wss[0],
                             out_head_major=False)
    # the peer offsets were fixed for batch B: another batch is refused, nothing launches
    with pytest.raises(SemipdError) as ei:
        pools[0].decode_attn(0, ins[0][0][:B - 1].contiguous(), ins[0][1][:B - 1].contiguous(),
                             ins[0][2][:B - 1].contiguous(), rid[:B - 1], ctx_d[:B - 1], max(ctx),
                             sc, outs[0][ins[0][3]:ins[0][4], :B - 1], wss[0], out_head_major=True)
    assert ei.value.status == INVALID
    with pytest.raises(SemipdError):  # tokens must be given with peers
        pools[0].set_decode_peers([outs[1].data_ptr()], 0)
    pools[0].set_decode_peers([])


@pytest.mark.parametrize("tpn", [2, 8])
def test_prefill_epilogue_peer_stores_emulated(tpn):
    """The TP head gather fused into the tcgen05 prefill epilogue (semipd_set_prefill_peers):
    ranks emulated as streams of one process, a 700-token chunk (full and ragged q tiles) over
    a 300-token paged prefix; every rank's gathered buffer equals the unsharded prefill bitwise,
    and the unsharded run is unchanged by the peer-store code path being present."""
    import ctypes

    import synth
    from paper_2504_19867_b200 import KVPool, PoolConfig, lib, tp
    dev = torch.device("cuda", 0)
    shape = synth.AttnShape("llama3-70b", 64, 8, 128, 128, 64, torch.bfloat16)
    C, P, bs = 700, 300, 64
    pc = synth.prefill_case(shape, [C], [P], seed=3050)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    sc = shape.softmax_scale
    nb = -(-(C + P) // bs)

    def make(heads):
        kl, kh = heads
        pool = KVPool(PoolConfig(1, nb + 1, bs, kh - kl, 128, 128, 1, nb), dev)
        pool.alloc_blocks(i32([0]), i32([nb]))
        K, V, BT, _ = pool.views(0)
        pos = torch.arange(P)
        blk = BT.cpu()[0].long()[pos // bs].to(dev)
        K[blk, :, (pos % bs).to(dev)] = pc.k_prefix[0][:, kl:kh].to(dev)
        V[blk, :, (pos % bs).to(dev)] = pc.v_prefix[0][:, kl:kh].to(dev)
        return pool

    cu, rid, pre = i32([0, C]), i32([0]), i32([P])
    full = make((0, 8))
    ref = torch.empty(64, C, 128, dtype=torch.bfloat16, device=dev)
    full.prefill_attn(0, pc.q.to(dev), pc.k_new.to(dev), pc.v_new.to(dev), cu, rid, pre, C, C, sc,
                      ref, out_head_major=True)
    hq = 64 // tpn
    pools, outs, flags, streams, ins = [], [], [], [], []
    for r in range(tpn):
        ql, qh = tp.head_range(64, tpn, r)
        kl, kh = tp.head_range(8, tpn, r)
        pools.append(make((kl, kh)))
        outs.append(torch.full((64, C, 128), float("nan"), dtype=torch.bfloat16, device=dev))
        flags.append(torch.zeros(2 * tpn, dtype=torch.int32, device=dev))
        streams.append(torch.cuda.Stream(dev))
        ins.append((pc.q[:, ql:qh].contiguous().to(dev), pc.k_new[:, kl:kh].contiguous().to(dev),
                    pc.v_new[:, kl:kh].contiguous().to(dev), ql, qh))
    shard = hq * C * 128 * 2
    for r in range(tpn):
        pools[r].set_prefill_peers([outs[k].data_ptr() + r * shard for k in range(tpn) if k != r], C)
    fl = (ctypes.c_void_p * tpn)(*[f.data_ptr() for f in flags])
    L = lib()
    torch.cuda.synchronize()
    for r in range(tpn):
        qs, ks, vs, ql, qh = ins[r]
        s = streams[r]
        cs = ctypes.c_void_p(s.cuda_stream)
        assert L.semipd_peer_handshake(fl, ctypes.c_void_p(flags[r].data_ptr()), tpn, r, 0, cs) == 0
        pools[r].prefill_attn(0, qs, ks, vs, cu, rid, pre, C, C, sc, outs[r][ql:qh],
                              out_head_major=True, stream=s)
        assert L.semipd_peer_handshake(fl, ctypes.c_void_p(flags[r].data_ptr()), tpn, r, 1, cs) == 0
    torch.cuda.synchronize()
    for r in range(tpn):
        assert torch.equal(outs[r].view(torch.int16), ref.view(torch.int16)), r
    assert all(int(f.abs().sum()) == 0 for f in flags)
    # every rank's gathered buffer against the fp64 oracle (bottom-right causal over the
    # paged prefix + the chunk, all 64 heads), not only against the unsharded kernel
    ref64 = oracle.attention_contig(np_bits(pc.q), np_bits(torch.cat([pc.k_prefix[0], pc.k_new])),
                                    np_bits(torch.cat([pc.v_prefix[0], pc.v_new])), P, sc)
    for r in range(tpn):
        compare(outs[r].float().cpu().double().numpy().transpose(1, 0, 2), ref64, torch.bfloat16,
                f"fused prefill gather tp{tpn} rank {r}")
    # another total_q than the gathered buffers hold is refused
    with pytest.raises(SemipdError) as ei:
        qs, ks, vs, ql, qh = ins[0]
        pools[0].prefill_attn(0, qs[:C - 1].contiguous(), ks[:C - 1].contiguous(),
                              vs[:C - 1].contiguous(), i32([0, C - 1]), rid, pre, C - 1, C - 1, sc,
                              outs[0][ql:qh, :C - 1], out_head_major=True)
    assert ei.value.status == INVALID


def _decode_pool_f8(shape, ctx, case, heads_kv, dev, ks, vs):
    """An E4M3 pool (R31) holding kv heads [heads_kv) of the cached contexts as the oracle's codes."""
    from paper_2504_19867_b200 import KVPool, PoolConfig
    kl, kh = heads_kv
    bs = shape.block_size
    nb = [c // bs + 1 for c in ctx]
    pool = KVPool(PoolConfig(1, sum(nb) + 2, bs, kh - kl, 128, 128, len(ctx), max(nb),
                             dtype=torch.float8_e4m3fn), dev)
    pool.set_kv_scales(ks, vs)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    for b, n in enumerate(nb):
        pool.alloc_blocks(i32([b]), i32([n]))
    K, V, BT, _ = pool.views(0)
    bt = BT.cpu()
    for b, c in enumerate(ctx):
        pos = torch.arange(c)
        blk = bt[b].long()[pos // bs].to(dev)
        kc = torch.from_numpy(oracle.e4m3_quantize(np_bits(case.k_ctx[b][:, kl:kh]), ks))
        vc = torch.from_numpy(oracle.e4m3_quantize(np_bits(case.v_ctx[b][:, kl:kh]), vs))
        K[blk, :, (pos % bs).to(dev)] = kc.to(dev)
        V[blk, :, (pos % bs).to(dev)] = vc.to(dev)
    return pool


@pytest.mark.parametrize("tpn", [2, 4])
def test_decode_epilogue_peer_stores_fp8_emulated(tpn):
    """The fused TP head gather on E4M3 pools (N2 x R31): rank r's FP8 decode kernel stores its
    head slice into every rank's gathered buffer; each gathered buffer equals the unsharded FP8
    decode bitwise and the oracle's FP8 decode within the bf16 bar.  (FP8 decode units are head
    pairs, so every rank keeps an even number of kv heads: TP <= 4 for 8 kv heads.)"""
    import ctypes

    import synth
    from paper_2504_19867_b200 import lib, tp
    dev = torch.device("cuda", 0)
    shape = synth.AttnShape("llama3-70b-fp8", 64, 8, 128, 128, 64, torch.bfloat16)
    ks, vs = 0.05, 0.02
    ctx = [300, 2048, 4500, 64]
    B = len(ctx)
    cd = synth.decode_case(shape, ctx, seed=3041)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    sc = shape.softmax_scale
    full_pool = _decode_pool_f8(shape, ctx, cd, (0, 8), dev, ks, vs)
    kp, vp = (t.cpu().numpy().copy() for t in full_pool.views(0)[:2])
    ref = torch.empty(64, B, 128, dtype=torch.bfloat16, device=dev)
    full_pool.decode_attn(0, cd.q.to(dev), cd.k_new.to(dev), cd.v_new.to(dev), i32(list(range(B))),
                          i32(ctx), max(ctx), sc, ref, full_pool.new_decode_workspace(B, 64, max(ctx)),
                          out_head_major=True)
    torch.cuda.synchronize()
    pools, outs, flags, streams, wss, ins = [], [], [], [], [], []
    hq = 64 // tpn
    for r in range(tpn):
        pools.append(_decode_pool_f8(shape, ctx, cd, tp.head_range(8, tpn, r), dev, ks, vs))
        outs.append(torch.full((64, B, 128), float("nan"), dtype=torch.bfloat16, device=dev))
        flags.append(torch.zeros(2 * tpn, dtype=torch.int32, device=dev))
        streams.append(torch.cuda.Stream(dev))
        wss.append(pools[r].new_decode_workspace(B, hq, max(ctx)))
        ql, qh = tp.head_range(64, tpn, r)
        kl, kh = tp.head_range(8, tpn, r)
        ins.append((cd.q[:, ql:qh].contiguous().to(dev), cd.k_new[:, kl:kh].contiguous().to(dev),
                    cd.v_new[:, kl:kh].contiguous().to(dev), ql, qh))
    fl = (ctypes.c_void_p * tpn)(*[f.data_ptr() for f in flags])
    L = lib()
    rid, ctx_d = i32(list(range(B))), i32(ctx)
    torch.cuda.synchronize()
    shard = hq * B * 128 * 2
    for r in range(tpn):
        pools[r].set_decode_peers([outs[k].data_ptr() + r * shard for k in range(tpn) if k != r], B)
    for r in range(tpn):
        qs, kn, vn, ql, qh = ins[r]
        cs = ctypes.c_void_p(streams[r].cuda_stream)
        assert L.semipd_peer_handshake(fl, ctypes.c_void_p(flags[r].data_ptr()), tpn, r, 0, cs) == 0
        pools[r].decode_attn(0, qs, kn, vn, rid, ctx_d, max(ctx), sc, outs[r][ql:qh], wss[r],
                             out_head_major=True, stream=streams[r])
        assert L.semipd_peer_handshake(fl, ctypes.c_void_p(flags[r].data_ptr()), tpn, r, 1, cs) == 0
    torch.cuda.synchronize()
    for r in range(tpn):
        assert torch.equal(outs[r].view(torch.int16), ref.view(torch.int16)), r
    ref64 = oracle.decode_fp8(np_bits(cd.q), np_bits(cd.k_new), np_bits(cd.v_new), kp, vp,
                              full_pool.views(0)[2].cpu().numpy(), np.arange(B), ctx, sc, ks, vs)
    for r in range(tpn):
        compare(outs[r].float().cpu().double().numpy().transpose(1, 0, 2), ref64, torch.bfloat16,
                f"fused fp8 decode gather tp{tpn} rank {r}")
    for p in pools:
        p.set_decode_peers([])
