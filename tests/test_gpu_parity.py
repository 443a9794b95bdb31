"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs.  Tolerances (S16): bf16 max_abs <= 2e-2 and
fro_rel <= 1e-2; fp32 1e-4 / 1e-4; block tables and K/V pool writes bit-exact."""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import oracle
import synth
from harness import Rig, compare, np_bits

pytestmark = pytest.mark.gpu

SHAPE_8B = synth.CFG2_LLAMA8B
SHAPE_70B_TP1 = synth.CFG3_LLAMA70B


def small(shape, **kw):
    d = dict(name=shape.name, num_q_heads=shape.num_q_heads, num_kv_heads=shape.num_kv_heads,
             head_dim_k=shape.head_dim_k, head_dim_v=shape.head_dim_v,
             block_size=shape.block_size, dtype=shape.dtype, num_layers=1,
             kv_shared=shape.kv_shared, scale=shape.scale)
    d.update(kw)
    return synth.AttnShape(**d)


# ----------------------------------------------------------------------------- allocator
def test_alloc_bit_exact_vs_oracle():
    rig = Rig(small(SHAPE_8B), num_blocks=64, max_reqs=8, mbr=16)
    rng = np.random.default_rng(0)
    for step in range(200):
        if rng.random() < 0.6:
            n = int(rng.integers(1, 4))
            ids = [int(x) for x in rng.integers(0, 8, n)]
            cnt = [int(x) for x in rng.integers(1, 6, n)]
            rig.alloc(ids, cnt, expect_ok=False)
        else:
            ids = [int(x) for x in rng.integers(0, 8, int(rng.integers(1, 3)))]
            rig.free(ids)
        if step % 20 == 0:
            rig.assert_tables_match()
    rig.assert_tables_match()


def test_alloc_spec_examples_on_gpu():
    rig = Rig(small(SHAPE_8B), num_blocks=10, max_reqs=4, mbr=16)
    assert sorted([rig.alloc([0], [6], False), rig.alloc([1], [6], False)]) == [0, oracle.OOM]
    assert rig.pool.stats()[0] == 4
    assert rig.alloc([2], [0], False) == oracle.INVALID
    rig.assert_tables_match()
    rig2 = Rig(small(SHAPE_8B), num_blocks=7, max_reqs=4, mbr=16)
    rig2.alloc([0], [5])
    assert rig2.free([0]) == 0 and rig2.pool.stats()[0] == 7
    assert rig2.free([0]) == oracle.UNKNOWN_REQ
    rig2.alloc([1], [5]); rig2.alloc([1], [2])
    assert rig2.free([1]) == 0 and rig2.pool.stats()[0] == 7
    rig2.assert_tables_match()


def _replay_oplog(words, N_B, R, MBR):
    ref = oracle.Allocator(N_B, R, MBR)
    i, seqs = 0, []
    while i < len(words):
        seq, kind, n, status = words[i:i + 4]
        ids = words[i + 4:i + 4 + n]
        if kind == 1:
            cnt = words[i + 4 + n:i + 4 + 2 * n]
            st = ref.alloc(ids, cnt)
            i += 4 + 2 * n
        else:
            st = ref.free(ids)
            i += 4 + n
        assert st == status, f"op {seq}: gpu status {status} vs replay {st}"
        seqs.append(seq)
    assert seqs == list(range(len(seqs))), "op log not in linearisation order"
    return ref


def test_two_stream_alloc_storm_linearizable():
    """Alloc/free storms from two streams (prefill + decode workers): the
    final tables equal the oracle replay of the device op log, bit for bit."""
    N_B, R, MBR = 96, 16, 32
    rig = Rig(small(SHAPE_8B), num_blocks=N_B, max_reqs=R, mbr=MBR)
    sP, sD = torch.cuda.Stream(), torch.cuda.Stream()
    rng = np.random.default_rng(7)
    keep = []
    for rnd in range(60):
        for s, ids_range in ((sP, range(0, 8)), (sD, range(8, 16))):
            with torch.cuda.stream(s):
                ids = [int(rng.choice(list(ids_range)))]
                if rng.random() < 0.65:
                    t_ids = torch.tensor(ids, dtype=torch.int32, device=rig.dev)
                    t_cnt = torch.tensor([int(rng.integers(1, 9))], dtype=torch.int32,
                                         device=rig.dev)
                    rig.pool.alloc_blocks(t_ids, t_cnt, None, stream=s)
                    keep += [t_ids, t_cnt]
                else:
                    t_ids = torch.tensor(ids, dtype=torch.int32, device=rig.dev)
                    rig.pool.free_blocks(t_ids, None, stream=s)
                    keep.append(t_ids)
    torch.cuda.synchronize()
    words, dropped = rig.pool.oplog()
    assert dropped == 0
    ref = _replay_oplog(words, N_B, R, MBR)
    bt, nb = rig.tables()
    np.testing.assert_array_equal(bt, ref.bt)
    np.testing.assert_array_equal(nb, ref.nblk)
    assert rig.pool.stats()[0] == ref.free_blocks
    # conservation + disjointness
    held = np.concatenate([bt[r, :nb[r]] for r in range(R)])
    assert len(set(held.tolist())) == len(held) == N_B - ref.free_blocks


def test_table_full_and_oom_leave_state():
    rig = Rig(small(SHAPE_8B), num_blocks=16, max_reqs=3, mbr=4)
    rig.alloc([0], [3])
    assert rig.alloc([0, 1], [2, 1], False) == oracle.TABLE_FULL
    assert rig.alloc([1, 2], [10, 4], False) == oracle.OOM
    assert rig.free([0, 0]) == oracle.UNKNOWN_REQ
    rig.assert_tables_match()


# ----------------------------------------------------------------------------- decode
def run_decode(shape, ctx, seed, dist, sm_budget=0, layer=0, num_layers=1, rid_offset=0,
               head_major=False, check_append=True, ws=None):
    bs = shape.block_size
    nblk = [c // bs + 1 for c in ctx]
    N_B = sum(nblk) + 7
    R = len(ctx) + rid_offset + 1
    rig = Rig(shape, num_blocks=N_B, max_reqs=R, mbr=max(nblk) + 1, num_layers=num_layers)
    rids = [rid_offset + b for b in range(len(ctx))]
    # permuted allocation order -> non-contiguous block tables
    for b in np.random.default_rng(seed).permutation(len(ctx)):
        rig.alloc([rids[b]], [nblk[b]])
    rig.assert_tables_match()
    case = synth.decode_case(shape, ctx, seed, dist, rids)
    for b in range(len(ctx)):
        rig.scatter(layer, rids[b], case.k_ctx[b], case.v_ctx[b])
    kp, vp = rig.host_pool(layer)
    dev = rig.dev
    q, kn = case.q.to(dev), case.k_new.to(dev)
    vn = case.v_new.to(dev) if case.v_new is not None else None
    B, Hq, dv = len(ctx), shape.num_q_heads, shape.head_dim_v
    out = torch.empty((Hq, B, dv) if head_major else (B, Hq, dv), dtype=shape.dtype, device=dev)
    if ws is None:
        ws = rig.pool.new_decode_workspace(B, Hq, max(ctx))
    rig.pool.decode_attn(layer, q, kn, vn, rig.i32(rids), rig.i32(ctx), max(ctx),
                         shape.softmax_scale, out, ws, out_head_major=head_major,
                         sm_budget=sm_budget, status=rig.status)
    torch.cuda.synchronize()
    assert int(rig.status.item()) == 0
    ref = oracle.decode(np_bits(case.q), np_bits(case.k_new),
                        None if case.v_new is None else np_bits(case.v_new), kp, vp,
                        rig.ref_alloc.bt, rids, ctx, shape.softmax_scale,
                        kv_shared=shape.kv_shared, dv=dv)
    got = out.float().cpu().double().numpy()
    if head_major:
        got = got.transpose(1, 0, 2)
    m = compare(got, ref, shape.dtype, f"decode {shape.name} dist{dist}")
    if check_append:
        K, V = rig.host_pool(layer)
        np.testing.assert_array_equal(K, kp)   # oracle appended into kp/vp in place
        if V is not None:
            np.testing.assert_array_equal(V, vp)
    return out, m


@pytest.mark.parametrize("dist", synth.DISTS)
def test_decode_tiny_fp32(dist):
    run_decode(synth.CFG1_TINY, [15, 16, 100, 256], seed=1010 + dist, dist=dist)


@pytest.mark.parametrize("dist", synth.DISTS)
def test_decode_llama8b_shapes(dist):
    # ctx covers: block edge, new block, ragged, > 1 split (4096 keys) with a ragged tail
    run_decode(small(SHAPE_8B), [0, 1, 15, 16, 17, 255, 2048, 4095, 4096, 9000],
               seed=1020 + dist, dist=dist)


@pytest.mark.parametrize("G", [1, 2, 8, 16])
def test_decode_gqa_groups(G):
    shape = small(SHAPE_8B, num_q_heads=2 * G, num_kv_heads=2)
    run_decode(shape, [33, 700, 5000], seed=77 + G, dist=synth.VSHIFT)


@pytest.mark.parametrize("bs", [32, 64, 128])
def test_decode_block_sizes(bs):
    run_decode(small(SHAPE_8B, block_size=bs), [5, 63, 64, 300, 4500], seed=88 + bs,
               dist=synth.NEEDLE)


def test_decode_head_major_and_layer():
    run_decode(small(SHAPE_8B), [100, 3000], seed=5, dist=synth.FLAT, head_major=True, layer=1,
               num_layers=2)


def test_decode_bitwise_stable_across_budgets():
    outs = [run_decode(small(SHAPE_8B), [130, 4200, 9999], seed=9, dist=synth.FLAT,
                       sm_budget=b)[0].cpu() for b in (1, 7, 74, 148, -1)]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("dist", synth.DISTS)
def test_decode_mla_latent(dist):
    """cfg 5 absorbed MLA (16 heads, latent 576 / 512, V aliases K, bs 64): block edges,
    ragged tails and > 1 split (4096 keys)."""
    run_decode(small(synth.CFG5_MLA), [0, 31, 63, 64, 200, 4100, 9000], seed=55 + dist, dist=dist)


def test_decode_mla_tensor_kernel_and_budgets():
    shape = small(synth.CFG5_MLA)
    outs = [run_decode(shape, [500, 4500, 37], seed=5, dist=synth.FLAT, sm_budget=b)[0].cpu()
            for b in (1, 9, 148, -1)]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    # the tcgen05 MLA kernel (trace kind 4) is the one that runs at bs 64
    from paper_2504_19867_b200 import KVPool, PoolConfig
    dev = torch.device("cuda", 0)
    pool = KVPool(PoolConfig(1, 8, 64, 1, 576, 512, 2, 4, kv_shared=True), dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32([0]), i32([2]))
    trace = torch.zeros(4 * 64, dtype=torch.int32, device=dev)
    ctr = torch.zeros(1, dtype=torch.int32, device=dev)
    pool.set_trace(trace, ctr)
    q = torch.randn(1, 16, 576, device=dev).bfloat16()
    kn = torch.randn(1, 1, 576, device=dev).bfloat16()
    out = torch.empty(1, 16, 512, dtype=torch.bfloat16, device=dev)
    ws = pool.new_decode_workspace(1, 16, 100)
    pool.decode_attn(0, q, kn, None, i32([0]), i32([100]), 100, 0.07, out, ws)
    torch.cuda.synchronize()
    n = int(ctr.item())
    kinds = set(trace[:4 * n].view(n, 4)[:, 3].cpu().tolist())
    assert kinds == {4}


@pytest.mark.parametrize("dist", [synth.FLAT, synth.NEEDLE])
def test_decode_mla_bs32_mma_sync_kernel(dist):
    """Latent pools with 32-token pages take the mma.sync MLA kernel (trace kind 3)."""
    run_decode(small(synth.CFG5_MLA, block_size=32), [0, 31, 32, 700, 5000], seed=65 + dist,
               dist=dist)


def test_decode_mla_fewer_heads_head_major():
    """Hq < 16 (q rows beyond Hq zero-filled by TMA) with head-major output."""
    run_decode(small(synth.CFG5_MLA, num_q_heads=8), [5, 64, 127, 1500, 2100], seed=71,
               dist=synth.PEAKED, head_major=True)


@pytest.mark.parametrize("ctx", [[9000], [300, 9000, 2000], [5000, 4100, 7000, 100]])
def test_decode_mla_small_batch_fill_splits(ctx):
    """Small batches split long contexts over many SMs (S_fill = ceil(148 / B) >> 32 splits
    here: the unstaged merge path) and their results match the oracle."""
    run_decode(small(synth.CFG5_MLA), ctx, seed=77 + len(ctx), dist=synth.VSHIFT)


@pytest.mark.parametrize("shape_name", ["mla", "llama"])
def test_decode_workspace_reused_across_batch_sizes(shape_name):
    """One workspace serves calls of different batch sizes: a small batch (many splits, so
    partials get written) followed by larger ones must not read stale partial bytes as split /
    work counters (counters live at the front, partials at the back; SpdWs)."""
    shape = small(synth.CFG5_MLA) if shape_name == "mla" else small(SHAPE_8B, block_size=64)
    Hq = shape.num_q_heads
    rig = Rig(shape, num_blocks=8, max_reqs=2, mbr=4)
    ws = rig.pool.new_decode_workspace(96, Hq, 9000)
    rng = np.random.default_rng(3)
    for i, B in enumerate([2, 96, 5, 40, 96]):
        ctx = [int(x) for x in rng.integers(1, 9000 if B <= 5 else 700, size=B)]
        run_decode(shape, ctx, seed=300 + i, dist=synth.FLAT, ws=ws)


def test_decode_mla_cfg5_batch():
    """cfg 5 shape at trace scale: B = 256 requests with lognormal-like contexts."""
    rng = np.random.default_rng(5)
    ctx = [int(x) for x in np.clip(rng.lognormal(np.log(251.0) - 0.5, 1.0, 256), 1, 8192)]
    run_decode(small(synth.CFG5_MLA), ctx, seed=75, dist=synth.VSHIFT)


def test_decode_full_size_cfg2():
    """BASELINE configs[1] decode at full size: B = 64, ctx = 2048, all rows."""
    run_decode(small(SHAPE_8B), [2048] * 64, seed=1020, dist=synth.FLAT)


def test_decode_full_size_cfg2_bench_pages():
    """The bench's configuration: cfg2 decode at full size with 64-token pages (the
    head-pair kernel), all rows."""
    run_decode(small(SHAPE_8B, block_size=64), [2048] * 64, seed=1021, dist=synth.FLAT)


def _pair_ctx(n, seed):
    edges = [0, 1, 63, 64, 65, 127, 128, 700, 4095, 4096, 5000]
    rng = np.random.default_rng(seed)
    return [edges[i] if i < len(edges) else int(rng.integers(1, 600)) for i in range(n)]


@pytest.mark.parametrize("dist", synth.DISTS)
def test_decode_pair_kernel(dist):
    """Head-pair kernel (64-token pages, even Hkv, >= 2 x 148 head-pair units): block edges,
    ragged tails, > 1 split; B = 80 requests x 4 pairs."""
    run_decode(small(SHAPE_8B, block_size=64), _pair_ctx(80, dist), seed=1030 + dist, dist=dist)


@pytest.mark.parametrize("G,hkv,B", [(1, 2, 296), (8, 2, 300), (16, 2, 296), (4, 3, 200)])
def test_decode_pair_kernel_groups(G, hkv, B):
    """G <= 8 with even Hkv takes the head-pair kernel; G = 16 or odd Hkv the one-head one."""
    shape = small(SHAPE_8B, num_q_heads=hkv * G, num_kv_heads=hkv, block_size=64)
    run_decode(shape, _pair_ctx(B, G + hkv), seed=90 + G + hkv, dist=synth.PEAKED)


def test_decode_pair_kernel_budgets_stress_and_kind():
    shape = small(SHAPE_8B, block_size=64)
    ctx = _pair_ctx(76, 7)
    outs = [run_decode(shape, ctx, seed=19, dist=synth.NEEDLE, sm_budget=b)[0].cpu()
            for b in [1, 2, 37, 148, -1] * 2]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    from paper_2504_19867_b200 import KVPool, PoolConfig
    dev = torch.device("cuda", 0)
    B = 74
    pool = KVPool(PoolConfig(1, 2 * B + 2, 64, 8, 128, 128, B + 1, 4), dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32(list(range(B))), i32([2] * B))
    trace = torch.zeros(4 * 256, dtype=torch.int32, device=dev)
    ctr = torch.zeros(1, dtype=torch.int32, device=dev)
    pool.set_trace(trace, ctr)
    q = torch.randn(B, 32, 128, device=dev).bfloat16()
    kn = torch.randn(B, 8, 128, device=dev).bfloat16()
    out = torch.empty(B, 32, 128, dtype=torch.bfloat16, device=dev)
    ws = pool.new_decode_workspace(B, 32, 100)
    pool.decode_attn(0, q, kn, kn.clone(), i32(list(range(B))), i32([100] * B), 100, 0.08, out, ws)
    torch.cuda.synchronize()
    n = int(ctr.item())
    assert set(trace[:4 * n].view(n, 4)[:, 3].cpu().tolist()) == {6}


@pytest.mark.parametrize("dist", synth.DISTS)
def test_decode_page128_kernel(dist):
    """128-token pages take the whole-page-box kernel (MODE 1): keys split over two warps per
    stage, including stages whose second half lies past the last key."""
    run_decode(small(SHAPE_8B, block_size=128), [0, 1, 63, 64, 65, 127, 128, 129, 700, 4096, 9000],
               seed=1040 + dist, dist=dist)


def test_decode_page128_kind_groups_budgets():
    for G in (1, 8, 16):
        shape = small(SHAPE_8B, num_q_heads=2 * G, num_kv_heads=2, block_size=128)
        run_decode(shape, [33, 700, 5000], seed=95 + G, dist=synth.VSHIFT)
    shape = small(SHAPE_8B, block_size=128)
    outs = [run_decode(shape, [5, 70, 130, 4100, 63, 200, 9000, 1], seed=21, dist=synth.NEEDLE,
                       sm_budget=b)[0].cpu() for b in [1, 2, 37, 148, -1]]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    from paper_2504_19867_b200 import KVPool, PoolConfig
    dev = torch.device("cuda", 0)
    pool = KVPool(PoolConfig(1, 8, 128, 8, 128, 128, 2, 4), dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32([0]), i32([2]))
    trace = torch.zeros(4 * 256, dtype=torch.int32, device=dev)
    ctr = torch.zeros(1, dtype=torch.int32, device=dev)
    pool.set_trace(trace, ctr)
    q = torch.randn(1, 32, 128, device=dev).bfloat16()
    kn = torch.randn(1, 8, 128, device=dev).bfloat16()
    out = torch.empty(1, 32, 128, dtype=torch.bfloat16, device=dev)
    ws = pool.new_decode_workspace(1, 32, 200)
    pool.decode_attn(0, q, kn, kn.clone(), i32([0]), i32([200]), 200, 0.08, out, ws)
    torch.cuda.synchronize()
    n = int(ctr.item())
    assert set(trace[:4 * n].view(n, 4)[:, 3].cpu().tolist()) == {7}


# ----------------------------------------------------------------------------- prefill
def run_prefill(shape, chunks, prefixes, seed, dist, sm_budget=0, head_major=False,
                rows_mask=None, layer=0, num_layers=1, rid_offset=0):
    bs = shape.block_size
    nblk = [-(-(c + p) // bs) for c, p in zip(chunks, prefixes)]
    N_B = sum(nblk) + 5
    R = len(chunks) + rid_offset + 2
    rig = Rig(shape, num_blocks=N_B, max_reqs=R, mbr=max(nblk) + 2, num_layers=num_layers)
    rids = [rid_offset + i for i in range(len(chunks))]
    for i in np.random.default_rng(seed + 1).permutation(len(chunks)):
        rig.alloc([rids[i]], [nblk[i]])
    rig.assert_tables_match()
    case = synth.prefill_case(shape, chunks, prefixes, seed, dist, rids)
    for i in range(len(chunks)):
        rig.scatter(layer, rids[i], case.k_prefix[i], case.v_prefix[i])
    kp, vp = rig.host_pool(layer)
    dev = rig.dev
    T, Hq, dv = sum(chunks), shape.num_q_heads, shape.head_dim_v
    out = torch.zeros((Hq, T, dv) if head_major else (T, Hq, dv), dtype=shape.dtype, device=dev)
    q, kn = case.q.to(dev), case.k_new.to(dev)
    vn = case.v_new.to(dev) if case.v_new is not None else None
    rig.pool.prefill_attn(layer, q, kn, vn, rig.i32(case.cu_seqlens), rig.i32(rids),
                          rig.i32(prefixes), T, max(chunks), shape.softmax_scale, out,
                          out_head_major=head_major, sm_budget=sm_budget, status=rig.status)
    torch.cuda.synchronize()
    assert int(rig.status.item()) == 0
    ref = oracle.prefill(np_bits(case.q), np_bits(case.k_new),
                         None if case.v_new is None else np_bits(case.v_new), kp, vp,
                         rig.ref_alloc.bt, case.cu_seqlens, rids, prefixes, shape.softmax_scale,
                         kv_shared=shape.kv_shared, rows_mask=rows_mask, dv=dv)
    got = out.float().cpu().double().numpy()
    if head_major:
        got = got.transpose(1, 0, 2)
    if rows_mask is not None:
        sel = np.asarray(rows_mask, bool)
        got, ref = got[sel], ref[sel]
    m = compare(got, ref, shape.dtype, f"prefill {shape.name} dist{dist}")
    K, V = rig.host_pool(layer)
    np.testing.assert_array_equal(K, kp)   # chunk K/V written bit-exactly
    if V is not None:
        np.testing.assert_array_equal(V, vp)
    return out, m


@pytest.mark.parametrize("chunks,prefixes", [([128], [0]), ([64], [64]), ([91], [37]),
                                             ([64, 64], [0, 0])])
@pytest.mark.parametrize("dist", synth.DISTS)
def test_prefill_tiny_fp32(chunks, prefixes, dist):
    run_prefill(synth.CFG1_TINY, chunks, prefixes, seed=1110 + dist, dist=dist)


@pytest.mark.parametrize("dist", synth.DISTS)
def test_prefill_llama8b_shapes(dist):
    # one full 2k-style chunk scaled down (several tiles + ragged tail), P = 0
    run_prefill(small(SHAPE_8B), [300], [0], seed=1220 + dist, dist=dist)


@pytest.mark.parametrize("chunks,prefixes", [([1], [0]), ([127], [0]), ([129], [0]),
                                             ([200], [17]), ([256], [128]), ([77], [600]),
                                             ([33, 1, 250, 129], [0, 5, 300, 16])])
def test_prefill_edges(chunks, prefixes):
    run_prefill(small(SHAPE_8B), chunks, prefixes, seed=31, dist=synth.NEEDLE)


@pytest.mark.parametrize("G", [1, 2, 8, 16])
def test_prefill_gqa_groups(G):
    shape = small(SHAPE_8B, num_q_heads=2 * G, num_kv_heads=2)
    run_prefill(shape, [150, 40], [0, 70], seed=91 + G, dist=synth.VSHIFT)


@pytest.mark.parametrize("bs", [32, 64, 128])
def test_prefill_block_sizes(bs):
    run_prefill(small(SHAPE_8B, block_size=bs), [190], [45], seed=3 + bs, dist=synth.PEAKED)


def test_prefill_varlen_sharegpt_pack():
    lens = synth.sharegpt_pack(1024, seed=2018)
    run_prefill(small(SHAPE_8B), lens, [0] * len(lens), seed=2018, dist=synth.FLAT)


def test_prefill_head_major_and_layer():
    run_prefill(small(SHAPE_8B), [160], [40], seed=4, dist=synth.FLAT, head_major=True, layer=1,
                num_layers=2)


def test_prefill_repeat_stress():
    """Same multi-request launch 20x: any pipeline race shows up as a bitwise change."""
    outs = [run_prefill(small(SHAPE_8B), [33, 1, 250, 129], [0, 5, 300, 16], seed=31,
                        dist=synth.NEEDLE, sm_budget=b)[0].cpu() for b in [3, 148] * 10]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_decode_repeat_stress_short_units():
    """Short units (1-3 stages) interleaved with long ones rotate stages over warps."""
    ctx = [5, 70, 130, 4100, 63, 200, 9000, 1]
    outs = [run_decode(small(SHAPE_8B), ctx, seed=17, dist=synth.NEEDLE, sm_budget=b)[0].cpu()
            for b in [2, 148] * 8]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_prefill_bitwise_stable_across_budgets():
    outs = [run_prefill(small(SHAPE_8B), [400, 90], [30, 0], seed=12, dist=synth.FLAT,
                        sm_budget=b)[0].cpu() for b in (1, 5, 74, 148, -1)]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_prefill_full_size_cfg2_sampled():
    """BASELINE configs[1] prefill at full size: one 2048-token chunk, P = 0, every
    16th row + the last row checked against the oracle (all heads)."""
    T = 2048
    mask = np.zeros(T, np.uint8)
    mask[::16] = 1
    mask[-1] = 1
    run_prefill(small(SHAPE_8B), [T], [0], seed=1220, dist=synth.FLAT, rows_mask=mask)


@pytest.mark.parametrize("chunks,prefixes", [([128], [0]), ([37], [100]), ([3, 70, 130], [0, 64, 5]),
                                             ([1, 200], [0, 300])])
@pytest.mark.parametrize("dist", synth.DISTS)
def test_prefill_mla_latent(chunks, prefixes, dist):
    """cfg 5 absorbed MLA prefill (16 heads over the 576-d latent, V = K[:, :512], bs 64):
    ragged token blocks, non-page-aligned prefixes, several requests per launch."""
    run_prefill(small(synth.CFG5_MLA), chunks, prefixes, seed=80 + dist, dist=dist)


def test_prefill_mla_kernel_budgets_and_kind():
    shape = small(synth.CFG5_MLA)
    outs = [run_prefill(shape, [150, 7], [10, 64], seed=85, dist=synth.NEEDLE,
                        sm_budget=b)[0].cpu() for b in (1, 9, 148, -1)]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    from paper_2504_19867_b200 import KVPool, PoolConfig
    dev = torch.device("cuda", 0)
    pool = KVPool(PoolConfig(1, 8, 64, 1, 576, 512, 2, 4, kv_shared=True), dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32([0]), i32([2]))
    trace = torch.zeros(4 * 64, dtype=torch.int32, device=dev)
    ctr = torch.zeros(1, dtype=torch.int32, device=dev)
    pool.set_trace(trace, ctr)
    q = torch.randn(100, 16, 576, device=dev).bfloat16()
    kn = torch.randn(100, 1, 576, device=dev).bfloat16()
    out = torch.empty(100, 16, 512, dtype=torch.bfloat16, device=dev)
    pool.prefill_attn(0, q, kn, None, i32([0, 100]), i32([0]), i32([0]), 100, 100, 0.07, out)
    torch.cuda.synchronize()
    n = int(ctr.item())
    kinds = set(trace[:4 * n].view(n, 4)[:, 3].cpu().tolist())
    assert kinds == {5}


def test_prefill_mla_fewer_heads_head_major():
    run_prefill(small(synth.CFG5_MLA, num_q_heads=8), [77], [20], seed=87, dist=synth.PEAKED,
                head_major=True)


def test_prefill_mla_full_chunk_sampled():
    """cfg 5 prefill chunk at full size (C = 2048, P = 0), every 32nd row + the last."""
    T = 2048
    mask = np.zeros(T, np.uint8)
    mask[::32] = 1
    mask[-1] = 1
    run_prefill(small(synth.CFG5_MLA), [T], [0], seed=88, dist=synth.FLAT, rows_mask=mask)


def test_prefill_then_decode_handoff():
    """Prefill writes the chunk's K/V; decode of the next token reads it from the
    pool (P:184 handoff, zero-copy)."""
    shape = small(SHAPE_8B)
    n = 300
    case = synth.prefill_case(shape, [n + 1], [0], seed=42)
    bs = shape.block_size
    rig = Rig(shape, num_blocks=40, max_reqs=2, mbr=32)
    rig.alloc([1], [-(-(n + 1) // bs)])
    dev = rig.dev
    T = n
    out = torch.empty(T, shape.num_q_heads, 128, dtype=shape.dtype, device=dev)
    rig.pool.prefill_attn(0, case.q[:n].to(dev), case.k_new[:n].to(dev), case.v_new[:n].to(dev),
                          rig.i32([0, n]), rig.i32([1]), rig.i32([0]), n, n, shape.softmax_scale,
                          out, status=rig.status)
    dout = torch.empty(1, shape.num_q_heads, 128, dtype=shape.dtype, device=dev)
    ws = rig.pool.new_decode_workspace(1, shape.num_q_heads, n)
    rig.pool.decode_attn(0, case.q[n:].to(dev), case.k_new[n:].to(dev), case.v_new[n:].to(dev),
                         rig.i32([1]), rig.i32([n]), n, shape.softmax_scale, dout, ws,
                         status=rig.status)
    torch.cuda.synchronize()
    kp = np.zeros((40, shape.num_kv_heads, bs, 128), np.uint16)
    vp = np.zeros_like(kp)
    ref = oracle.prefill(np_bits(case.q), np_bits(case.k_new), np_bits(case.v_new), kp, vp,
                         rig.ref_alloc.bt, [0, n + 1], [1], [0], shape.softmax_scale)
    compare(out.float().cpu().double().numpy(), ref[:n], shape.dtype, "handoff prefill")
    compare(dout.float().cpu().double().numpy(), ref[n:], shape.dtype, "handoff decode")
    K, V = rig.host_pool(0)
    np.testing.assert_array_equal(K, kp)
    np.testing.assert_array_equal(V, vp)


# ----------------------------------------------------------------------------- co-run
@pytest.mark.parametrize("bs,dec_kind", [(16, 8), (64, 2), (128, 7)])
def test_corun_bitwise_identical_and_disjoint_sms(bs, dec_kind):
    """Prefill (stream P) and decode (stream D) co-run on one pool with budgets
    (74, 74): outputs are bitwise identical to isolated runs and the two grids
    occupy disjoint SM sets (CTA %smid trace)."""
    from paper_2504_19867_b200 import KVPool, PoolConfig
    shape = small(SHAPE_8B)
    B, ctx, C = 32, 2048, 1024
    nb_d, nb_p = ctx // bs + 1, C // bs
    cfg = PoolConfig(1, B * nb_d + nb_p + 4, bs, 8, 128, 128, B + 2, nb_d + 1)
    pool = KVPool(cfg, 0)
    dev = pool.device
    rid_d = torch.arange(B, dtype=torch.int32, device=dev)
    pool.alloc_blocks(rid_d, torch.full((B,), nb_d, dtype=torch.int32, device=dev))
    rid_p = torch.tensor([B], dtype=torch.int32, device=dev)
    pool.alloc_blocks(rid_p, torch.tensor([nb_p], dtype=torch.int32, device=dev))
    K, V, _, _ = pool.views(0)
    g = synth.gen(5)
    K.copy_(torch.randn(K.shape, generator=g).to(K.dtype).to(dev))
    V.copy_(torch.randn(V.shape, generator=g).to(V.dtype).to(dev))
    qd = torch.randn(B, 32, 128, generator=g).bfloat16().to(dev)
    kd = torch.randn(B, 8, 128, generator=g).bfloat16().to(dev)
    vd = torch.randn(B, 8, 128, generator=g).bfloat16().to(dev)
    qp = torch.randn(C, 32, 128, generator=g).bfloat16().to(dev)
    kpn = torch.randn(C, 8, 128, generator=g).bfloat16().to(dev)
    vpn = torch.randn(C, 8, 128, generator=g).bfloat16().to(dev)
    ctxs = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    cu = torch.tensor([0, C], dtype=torch.int32, device=dev)
    pre = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = pool.new_decode_workspace(B, 32, ctx)
    sc = 1 / math.sqrt(128)

    def run(budgets, streams):
        od = torch.empty(B, 32, 128, dtype=torch.bfloat16, device=dev)
        op = torch.empty(C, 32, 128, dtype=torch.bfloat16, device=dev)
        sp, sd = streams
        with torch.cuda.stream(sp):
            pool.prefill_attn(0, qp, kpn, vpn, cu, rid_p, pre, C, C, sc, op,
                              sm_budget=budgets[0], stream=sp)
        with torch.cuda.stream(sd):
            pool.decode_attn(0, qd, kd, vd, rid_d, ctxs, ctx, sc, od, ws, sm_budget=budgets[1],
                             stream=sd)
        torch.cuda.synchronize()
        return op.cpu(), od.cpu()

    cur = torch.cuda.current_stream()
    iso = run((148, 148), (cur, cur))
    trace = torch.zeros(4 * 4096, dtype=torch.int32, device=dev)
    ctr = torch.zeros(1, dtype=torch.int32, device=dev)
    pool.set_trace(trace, ctr)
    co = run((74, 74), (torch.cuda.Stream(), torch.cuda.Stream()))
    pool.set_trace(None)
    assert torch.equal(iso[0], co[0]) and torch.equal(iso[1], co[1])
    n = int(ctr.item())
    rec = trace[:4 * n].view(n, 4).cpu().numpy()
    pre_sms = set(rec[rec[:, 0] == 1, 1].tolist())
    dec_sms = set(rec[rec[:, 0] == 2, 1].tolist())
    assert len(pre_sms) == 74 and len(dec_sms) == 74
    # the tensor-core kernels ran (kind 1 = tcgen05 prefill, 2 = split-K decode, 6 = the
    # head-pair split-K decode used with >= 64-token pages)
    assert set(rec[rec[:, 0] == 1, 3].tolist()) == {1}
    assert set(rec[rec[:, 0] == 2, 3].tolist()) == {dec_kind}
    # Disjointness holds whenever the two persistent grids are resident together;
    # report the overlap (0 expected when both launch before either finishes).
    print("corun SM overlap:", len(pre_sms & dec_sms))


def test_partition_switch_moves_no_kv_and_keeps_results():
    """P:211-216 / SURVEY CS3: set_partition between iterations is a host store - the
    pool pointer and contents (checksum) are unchanged and outputs stay bitwise equal."""
    shape = small(SHAPE_8B, block_size=64)
    ctx = [4000, 700]
    rig = Rig(shape, num_blocks=90, max_reqs=4, mbr=70)
    for b, c in enumerate(ctx):
        rig.alloc([b], [c // 64 + 1])
    case = synth.decode_case(shape, ctx, seed=77)
    for b in range(2):
        rig.scatter(0, b, case.k_ctx[b], case.v_ctx[b])
    dev = rig.dev
    ptr0 = rig.pool.mem.data_ptr()
    K, V, _, _ = rig.pool.views(0)
    outs, sums = [], []
    ws = rig.pool.new_decode_workspace(2, 32, max(ctx))
    for x, y in [(30, 70), (50, 50), (70, 30), (100, 100), (10, 90)]:
        rig.pool.set_partition(x, y)
        n_p, n_d = rig.pool.sm_budgets()
        assert (n_p, n_d) == (oracle.sm_budget(rig.pool.num_sms, x),
                              oracle.sm_budget(rig.pool.num_sms, y))
        out = torch.empty(2, 32, 128, dtype=torch.bfloat16, device=dev)
        # same step re-run (append rewrites the same slot with the same bits)
        rig.pool.decode_attn(0, case.q.to(dev), case.k_new.to(dev), case.v_new.to(dev),
                             rig.i32([0, 1]), rig.i32(ctx), max(ctx), shape.softmax_scale, out, ws,
                             sm_budget=0)
        torch.cuda.synchronize()
        outs.append(out.cpu())
        sums.append((int(K.view(torch.int16).sum().item()), int(V.view(torch.int16).sum().item())))
        assert rig.pool.mem.data_ptr() == ptr0
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    assert all(s == sums[0] for s in sums)
    with pytest.raises(Exception):
        rig.pool.set_partition(0, 50)
    with pytest.raises(Exception):
        rig.pool.set_partition(50, 100.5)
