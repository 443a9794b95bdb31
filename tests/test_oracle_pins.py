"""Pins for the fp64 oracle (CPU only, -m "not gpu").

The oracle is pinned to things other than itself:
  * an independent library routine: torch.nn.functional.scaled_dot_product_attention
    in float64 on CPU, with an explicit bottom-right causal mask (S4) and the KV
    heads repeated for GQA (S3);
  * brute force with an explicit full score matrix in numpy on tiny inputs;
  * closed forms (single key, equal keys, constant V, dominant key, probability
    vector with known exact values, a hand-computed 1-d case);
  * invariants (paged == contiguous under a permuted block table, chunked ==
    unchunked, prefill + decode == longer prefill, GQA == MHA on repeated KV,
    split-K merge == unsplit, K/V writes bit-exact);
  * the SPEC allocator / partition examples and exhaustive
    two-actor interleavings checked against an independent free-count model.
"""
import itertools
import math

import numpy as np
import pytest
import torch

import oracle
import synth

R64 = dict(rtol=1e-12, atol=1e-12)


def f32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


def sdpa_ref(q, k, v, causal_offset):
    """Library routine: torch SDPA fp64; q [nq,Hq,d], k/v [nk,Hkv,d] (fp64 numpy)."""
    nq, Hq, _ = q.shape
    nk, Hkv, _ = k.shape
    G = Hq // Hkv
    qt = torch.from_numpy(q).permute(1, 0, 2)  # [Hq, nq, d]
    kt = torch.from_numpy(k).permute(1, 0, 2).repeat_interleave(G, dim=0)
    vt = torch.from_numpy(v).permute(1, 0, 2).repeat_interleave(G, dim=0)
    mask = None
    if causal_offset >= 0:
        rows = torch.arange(nq).unsqueeze(1)
        cols = torch.arange(nk).unsqueeze(0)
        mask = cols <= rows + causal_offset
    scale = 1.0 / math.sqrt(q.shape[2])
    o = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=mask, scale=scale)
    return o.permute(1, 0, 2).numpy()


def scatter_pool(k_tok, v_tok, bt_row, bs, k_pool, v_pool):
    """Harness layout step: write token j's K/V into pool[bt[j//bs]][:, j%bs]."""
    for j in range(k_tok.shape[0]):
        k_pool[bt_row[j // bs], :, j % bs] = k_tok[j]
        if v_pool is not None:
            v_pool[bt_row[j // bs], :, j % bs] = v_tok[j]


# --------------------------------------------------------------------------- attention
@pytest.mark.parametrize("Hq,Hkv,d,nq,nk,off", [(4, 2, 16, 5, 9, 4), (8, 8, 8, 7, 7, 0),
                                                (6, 1, 32, 3, 20, 17), (4, 2, 16, 4, 6, -1)])
def test_contig_matches_torch_sdpa(Hq, Hkv, d, nq, nk, off):
    rng = np.random.default_rng(1)
    q, k, v = (f32(rng.standard_normal(s)) for s in [(nq, Hq, d), (nk, Hkv, d), (nk, Hkv, d)])
    out = oracle.attention_contig(q, k, v, off, 1.0 / math.sqrt(d))
    ref = sdpa_ref(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64), off)
    np.testing.assert_allclose(out, ref, rtol=1e-11, atol=1e-12)


def test_bf16_inputs_widen_exactly():
    """bf16 bit patterns are widened exactly: result equals fp32 path on the same values."""
    g = synth.gen(3)
    q = torch.randn(3, 2, 16, generator=g).bfloat16()
    k = torch.randn(6, 1, 16, generator=g).bfloat16()
    v = torch.randn(6, 1, 16, generator=g).bfloat16()
    a = oracle.attention_contig(synth.bits(q), synth.bits(k), synth.bits(v), 3, 0.25)
    b = oracle.attention_contig(f32(q.float()), f32(k.float()), f32(v.float()), 3, 0.25)
    np.testing.assert_array_equal(a, b)


def test_brute_force_full_matrix():
    rng = np.random.default_rng(7)
    nq, nk, d = 4, 6, 8
    q, k, v = (f32(rng.standard_normal(s)) for s in [(nq, 1, d), (nk, 1, d), (nk, 1, d)])
    s = 0.3
    out = oracle.attention_contig(q, k, v, 2, s)
    Q, K, V = (a[:, 0].astype(np.float64) for a in (q, k, v))
    S = s * (Q @ K.T)
    S[np.arange(nk)[None, :] > np.arange(nq)[:, None] + 2] = -np.inf
    P = np.exp(S - S.max(1, keepdims=True))
    P /= P.sum(1, keepdims=True)
    np.testing.assert_allclose(out[:, 0], P @ V, **R64)


def test_hand_computed_1d():
    # Hq=Hkv=d=1: z = [0, ln 3] -> weights 1:3 ; v = [0, 4] -> o = 3 exactly.
    q, k, v = f32([[[1.0]]]), f32([[[0.0]], [[1.0]]]), f32([[[0.0]], [[4.0]]])
    out = oracle.attention_contig(q, k, v, -1, math.log(3.0))
    assert abs(out[0, 0, 0] - 3.0) < 1e-14


def test_closed_forms():
    rng = np.random.default_rng(11)
    d = 16
    q = f32(rng.standard_normal((1, 2, d)))
    # single key -> o = v
    k1, v1 = f32(rng.standard_normal((1, 1, d))), f32(rng.standard_normal((1, 1, d)))
    o = oracle.attention_contig(q, k1, v1, -1, 0.25)
    np.testing.assert_allclose(o[0, 0], v1[0, 0], **R64)
    np.testing.assert_allclose(o[0, 1], v1[0, 0], **R64)
    # all keys equal -> mean of visible v
    n = 9
    kk = np.repeat(f32(rng.standard_normal((1, 1, d))), n, axis=0)
    vv = f32(rng.standard_normal((n, 1, d)))
    o = oracle.attention_contig(q, kk, vv, -1, 0.25)
    np.testing.assert_allclose(o[0, 0], vv[:, 0].astype(np.float64).mean(0), **R64)
    # constant V -> V
    vc = np.repeat(f32(rng.standard_normal((1, 1, d))), n, axis=0)
    o = oracle.attention_contig(q, f32(rng.standard_normal((n, 1, d))), vc, -1, 0.25)
    np.testing.assert_allclose(o[0, 1], vc[0, 0], rtol=1e-12, atol=1e-12)
    # dominant key (+40 above the rest) -> its v
    qd = np.zeros((1, 1, d), np.float32)
    qd[0, 0, 0] = 1.0
    kd = np.zeros((n, 1, d), np.float32)
    kd[5, 0, 0] = 40.0
    o = oracle.attention_contig(qd, kd, vv, -1, 1.0)
    np.testing.assert_allclose(o[0, 0], vv[5, 0], rtol=0, atol=1e-15 * n + 1e-16 * 40 + 1e-15)
    # V = identity rows -> o is the probability vector; z = 0, ln2, 2ln2 -> 1/7, 2/7, 4/7
    kp = np.zeros((3, 1, 3), np.float32)
    kp[:, 0, 0] = [0.0, 1.0, 2.0]
    qp = np.zeros((1, 1, 3), np.float32)
    qp[0, 0, 0] = 1.0
    vp = np.eye(3, dtype=np.float32).reshape(3, 1, 3)
    o = oracle.attention_contig(qp, kp, vp, -1, math.log(2.0))
    np.testing.assert_allclose(o[0, 0], [1 / 7, 2 / 7, 4 / 7], rtol=1e-14)
    assert abs(o[0, 0].sum() - 1.0) < 1e-15


def test_gqa_equals_mha_on_repeated_kv():
    rng = np.random.default_rng(5)
    q = f32(rng.standard_normal((5, 8, 16)))
    k = f32(rng.standard_normal((7, 2, 16)))
    v = f32(rng.standard_normal((7, 2, 16)))
    a = oracle.attention_contig(q, k, v, 2, 0.25)
    b = oracle.attention_contig(q, np.repeat(k, 4, axis=1), np.repeat(v, 4, axis=1), 2, 0.25)
    np.testing.assert_array_equal(a, b)


def _prefill_setup(shape, chunk_lens, prefix_lens, seed, N_B=64, MBR=16, dist=synth.FLAT):
    case = synth.prefill_case(shape, chunk_lens, prefix_lens, seed, dist)
    bs = shape.block_size
    rng = np.random.default_rng(seed)
    perm = rng.permutation(N_B).astype(np.int32)
    bt = np.full((len(chunk_lens) + 2, MBR), -1, np.int32)
    used = 0
    for i, (c, p) in enumerate(zip(chunk_lens, prefix_lens)):
        nb = -(-(c + p) // bs)
        bt[i, :nb] = perm[used:used + nb]
        used += nb
    npdt = np.uint16 if shape.dtype == torch.bfloat16 else np.float32
    k_pool = np.zeros((N_B, shape.num_kv_heads, bs, shape.head_dim_k), npdt)
    v_pool = np.zeros((N_B, shape.num_kv_heads, bs, shape.head_dim_v), npdt)
    for i in range(len(chunk_lens)):
        if prefix_lens[i]:
            scatter_pool(synth.bits(case.k_prefix[i]), synth.bits(case.v_prefix[i]), bt[i], bs,
                         k_pool, v_pool)
    return case, bt, k_pool, v_pool


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_paged_prefill_equals_contiguous_sdpa(dtype):
    shape = synth.AttnShape("t", 4, 2, 16, 16, 4, dtype)
    chunk, pre = [5, 11, 1], [0, 7, 13]
    case, bt, kp, vp = _prefill_setup(shape, chunk, pre, seed=21)
    out = oracle.prefill(synth.bits(case.q), synth.bits(case.k_new), synth.bits(case.v_new), kp,
                         vp, bt, case.cu_seqlens, [0, 1, 2], pre, shape.softmax_scale)
    cu = case.cu_seqlens
    for i in range(3):
        kc = torch.cat([case.k_prefix[i], case.k_new[cu[i]:cu[i + 1]]]).double().numpy()
        vc = torch.cat([case.v_prefix[i], case.v_new[cu[i]:cu[i + 1]]]).double().numpy()
        ref = sdpa_ref(case.q[cu[i]:cu[i + 1]].double().numpy(), kc, vc, pre[i])
        np.testing.assert_allclose(out[cu[i]:cu[i + 1]], ref, rtol=1e-11, atol=1e-12)
    # K/V written bit-exactly at positions P..P+C-1
    for i in range(3):
        for t in range(chunk[i]):
            pos = pre[i] + t
            blk, slot = bt[i, pos // 4], pos % 4
            np.testing.assert_array_equal(kp[blk, :, slot], synth.bits(case.k_new[cu[i] + t]))
            np.testing.assert_array_equal(vp[blk, :, slot], synth.bits(case.v_new[cu[i] + t]))


def test_paged_is_permutation_invariant():
    shape = synth.AttnShape("t", 4, 2, 16, 16, 4, torch.float32)
    outs = []
    for seed_perm in (1, 2, 3):
        case, bt, kp, vp = _prefill_setup(shape, [9], [10], seed=33)
        # re-map with a different permutation of physical blocks
        rng = np.random.default_rng(seed_perm)
        perm = rng.permutation(kp.shape[0]).astype(np.int32)
        bt2 = np.where(bt >= 0, perm[np.maximum(bt, 0)], -1).astype(np.int32)
        kp2, vp2 = np.zeros_like(kp), np.zeros_like(vp)
        kp2[perm] = kp
        vp2[perm] = vp
        outs.append(oracle.prefill(synth.bits(case.q), synth.bits(case.k_new),
                                   synth.bits(case.v_new), kp2, vp2, bt2, case.cu_seqlens, [0],
                                   [10], 0.25))
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])


def test_chunked_equals_unchunked_and_decode_continues_prefill():
    shape = synth.AttnShape("t", 4, 2, 16, 16, 4, torch.float32)
    n = 23
    case = synth.prefill_case(shape, [n + 1], [0], seed=44)
    q, k, v = (synth.bits(t) for t in (case.q, case.k_new, case.v_new))
    N_B, MBR = 16, 8
    bt = np.full((1, MBR), -1, np.int32)
    bt[0, :7] = [3, 9, 0, 12, 5, 7, 1]

    def pool():
        return (np.zeros((N_B, 2, 4, 16), np.float32), np.zeros((N_B, 2, 4, 16), np.float32))

    kp, vp = pool()
    full = oracle.prefill(q, k, v, kp, vp, bt, [0, n + 1], [0], [0], 0.25)
    # chunks 0..9 | 10..16 (non-aligned prefix 10) | 17..22  then decode of token 23
    kp2, vp2 = pool()
    parts = []
    for a, b in [(0, 10), (10, 17), (17, n)]:
        parts.append(oracle.prefill(q[a:b], k[a:b], v[a:b], kp2, vp2, bt, [0, b - a], [0], [a],
                                    0.25))
    chunked = np.concatenate(parts)
    np.testing.assert_allclose(chunked, full[:n], rtol=1e-13, atol=1e-14)
    dec = oracle.decode(q[n:n + 1], k[n:n + 1], v[n:n + 1], kp2, vp2, bt, [0], [n], 0.25)
    np.testing.assert_allclose(dec[0], full[n], rtol=1e-13, atol=1e-14)
    np.testing.assert_array_equal(kp2, kp)
    np.testing.assert_array_equal(vp2, vp)


def test_decode_matches_sdpa_and_appends():
    shape = synth.AttnShape("t", 8, 2, 32, 32, 16, torch.bfloat16)
    ctx = [0, 15, 16, 40]
    case = synth.decode_case(shape, ctx, seed=55, dist=synth.VSHIFT)
    N_B, MBR = 32, 4
    bt = np.full((6, MBR), -1, np.int32)
    perm = np.random.default_rng(0).permutation(N_B)
    u = 0
    for b, c in enumerate(ctx):
        nb = c // 16 + 1
        bt[b + 2, :nb] = perm[u:u + nb]
        u += nb
    kp = np.zeros((N_B, 2, 16, 32), np.uint16)
    vp = np.zeros((N_B, 2, 16, 32), np.uint16)
    for b in range(4):
        scatter_pool(synth.bits(case.k_ctx[b]), synth.bits(case.v_ctx[b]), bt[b + 2], 16, kp, vp)
    out = oracle.decode(synth.bits(case.q), synth.bits(case.k_new), synth.bits(case.v_new), kp,
                        vp, bt, [2, 3, 4, 5], ctx, shape.softmax_scale)
    for b, c in enumerate(ctx):
        kc = torch.cat([case.k_ctx[b], case.k_new[b:b + 1]]).double().numpy()
        vc = torch.cat([case.v_ctx[b], case.v_new[b:b + 1]]).double().numpy()
        ref = sdpa_ref(case.q[b:b + 1].double().numpy(), kc, vc, -1)
        np.testing.assert_allclose(out[b], ref[0], rtol=1e-11, atol=1e-12)
        blk, slot = bt[b + 2, c // 16], c % 16
        np.testing.assert_array_equal(kp[blk, :, slot], synth.bits(case.k_new[b]))
    # single key (ctx 0): o = v_new exactly (bf16 widened)
    np.testing.assert_allclose(out[0], np.repeat(case.v_new[0].double().numpy(), 4, axis=0),
                               **R64)


def test_mla_kv_shared_value_aliases_latent():
    """kv_shared: v_j = k_j[:dv] (absorbed MLA, S19) == contiguous with v = k[..., :dv]."""
    shape = synth.AttnShape("mla", 4, 1, 24, 16, 8, torch.float32, kv_shared=True, scale=0.2)
    case = synth.decode_case(shape, [13], seed=66)
    N_B = 8
    bt = np.array([[4, 1, -1]], np.int32)
    kp = np.zeros((N_B, 1, 8, 24), np.float32)
    scatter_pool(synth.bits(case.k_ctx[0]), None, bt[0], 8, kp, None)
    out = oracle.decode(synth.bits(case.q), synth.bits(case.k_new), None, kp, None, bt, [0], [13],
                        0.2, kv_shared=True, dv=16)
    kc = torch.cat([case.k_ctx[0], case.k_new]).numpy()
    ref = oracle.attention_contig(synth.bits(case.q), kc, np.ascontiguousarray(kc[..., :16]), -1,
                                  0.2)
    np.testing.assert_allclose(out, ref, rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("cuts", [[0, 40], [0, 1, 40], [0, 16, 17, 30, 40], [0, 5, 9, 21, 33, 40]])
def test_split_merge_equals_unsplit(cuts):
    rng = np.random.default_rng(9)
    d = 16
    q = rng.standard_normal(d)
    k = rng.standard_normal((40, d))
    v = rng.standard_normal((40, d))
    parts = [oracle.partial(q, k, v, a, b, 0.25) for a, b in zip(cuts[:-1], cuts[1:])]
    merged = oracle.merge([p[0] for p in parts], [p[1] for p in parts], [p[2] for p in parts])
    whole = oracle.attention_contig(f32(q[None, None]), f32(k[:, None]), f32(v[:, None]), -1, 0.25)
    # fp32-rounded inputs for the whole; compare against fp64 partials on same rounding
    q32, k32, v32 = (np.asarray(f32(a), np.float64) for a in (q, k, v))
    parts32 = [oracle.partial(q32, k32, v32, a, b, 0.25) for a, b in zip(cuts[:-1], cuts[1:])]
    merged32 = oracle.merge([p[0] for p in parts32], [p[1] for p in parts32],
                            [p[2] for p in parts32])
    np.testing.assert_allclose(merged32, whole[0, 0], rtol=1e-13, atol=1e-14)
    assert np.all(np.isfinite(merged))


# --------------------------------------------------------------------------- allocator
def test_spec_alloc_examples():
    # S:240 capacity 10, two callers request 6 each -> exactly one granted, free = 4
    a = oracle.Allocator(10, 4, 16)
    r = [a.alloc([0], [6]), a.alloc([1], [6])]
    assert sorted(r) == [oracle.OK, oracle.OOM] and a.free_blocks == 4
    # S:241 request 0 blocks -> contract violation
    assert a.alloc([2], [0]) == oracle.INVALID
    # S:242 grant 4 then free 4 then grant 10 -> granted, free = 0
    b = oracle.Allocator(10, 4, 16)
    assert b.alloc([0], [4]) == oracle.OK and b.free([0]) == oracle.OK
    assert b.alloc([1], [10]) == oracle.OK and b.free_blocks == 0


def test_spec_release_examples():
    a = oracle.Allocator(7, 4, 16)
    assert a.alloc([0], [5]) == oracle.OK and a.free_blocks == 2
    assert a.free([0]) == oracle.OK and a.free_blocks == 7
    assert a.free([0]) == oracle.UNKNOWN_REQ                          # S:250 double release
    assert a.alloc([1], [5]) == oracle.OK and a.alloc([1], [2]) == oracle.OK
    assert a.free_blocks == 0 and a.free([1]) == oracle.OK and a.free_blocks == 7


def test_blocks_for_tokens_spec():
    assert oracle.blocks_for_tokens(251, 16) == 16
    assert oracle.blocks_for_tokens(256, 16) == 16
    assert oracle.blocks_for_tokens(0, 16) == 0
    assert oracle.blocks_for_tokens(257, 16) == 17


def test_lifo_order_and_table_contents():
    a = oracle.Allocator(8, 3, 8)
    assert a.alloc([1, 0], [2, 3]) == oracle.OK
    assert a.bt[1, :2].tolist() == [0, 1] and a.bt[0, :3].tolist() == [2, 3, 4]   # S9
    assert a.free([1]) == oracle.OK                     # pushes 0 then 1 (table order)
    assert a.alloc([2], [3]) == oracle.OK
    assert a.bt[2, :3].tolist() == [1, 0, 5]            # LIFO pops
    assert a.nblk.tolist() == [3, 0, 3] and a.free_blocks == 2


def test_all_or_nothing_and_table_full():
    a = oracle.Allocator(16, 3, 4)
    assert a.alloc([0], [3]) == oracle.OK
    snap = a.snapshot()
    for args in ([[0, 1], [2, 1]], [[1], [5]], [[1, 1], [3, 2]]):    # row overflow -> TABLE_FULL
        assert a.alloc(*args) == oracle.TABLE_FULL
        _same(a, snap)
    assert a.alloc([1, 2], [10, 4]) == oracle.OOM   # 14 > 13 free
    _same(a, snap)
    assert a.alloc([5], [1]) == oracle.INVALID and a.free([7]) == oracle.INVALID
    assert a.free([0, 0]) == oracle.UNKNOWN_REQ and a.free([0, 2]) == oracle.UNKNOWN_REQ
    _same(a, snap)
    assert a.alloc([], []) == oracle.OK and a.free([]) == oracle.OK
    _same(a, snap)


def _same(a, snap):
    fs, top, bt, nb = snap
    assert a.free_blocks == top and np.array_equal(a.bt, bt) and np.array_equal(a.nblk, nb)
    assert np.array_equal(a.free_stack[:top], fs[:top])


def _check_invariants(a):
    top = a.free_blocks
    held = [a.bt[r, :a.nblk[r]] for r in range(a.R)]
    assert top + int(a.nblk.sum()) == a.N_B                     # conservation
    allb = np.concatenate([a.free_stack[:top]] + held)
    assert sorted(allb.tolist()) == list(range(a.N_B))          # disjoint + complete
    for r in range(a.R):
        assert np.all(a.bt[r, a.nblk[r]:] == -1)


def _ops_for_actor(actor, seq):
    return [(actor, op, n) for op, n in seq]


def test_exhaustive_two_actor_interleavings():
    """2 actors x <= 4 ops, N_B <= 8: every interleaving keeps conservation and
    disjointness, and every status equals an independent free-count model."""
    seqs = [
        [("a", 3), ("a", 2), ("f", 0), ("a", 4)],
        [("a", 5), ("f", 0), ("a", 8), ("f", 0)],
        [("a", 1), ("a", 1), ("a", 1), ("f", 0)],
        [("a", 6), ("a", 3), ("f", 0), ("f", 0)],
    ]
    for N_B in (6, 8):
        for s0, s1 in itertools.product(seqs, repeat=2):
            ops0, ops1 = _ops_for_actor(0, s0), _ops_for_actor(1, s1)
            for mask in itertools.combinations(range(8), 4):
                order, i0, i1 = [], 0, 0
                for pos in range(8):
                    if pos in mask:
                        order.append(ops0[i0]); i0 += 1
                    else:
                        order.append(ops1[i1]); i1 += 1
                a = oracle.Allocator(N_B, 2, 16)
                free, held = N_B, [0, 0]           # independent model
                for actor, op, n in order:
                    if op == "a":
                        exp = oracle.OK if n <= free else oracle.OOM
                        if exp == oracle.OK and held[actor] + n > 16:
                            exp = oracle.TABLE_FULL
                        got = a.alloc([actor], [n])
                        if got == oracle.OK:
                            free -= n
                            held[actor] += n
                    else:
                        exp = oracle.OK if held[actor] > 0 else oracle.UNKNOWN_REQ
                        got = a.free([actor])
                        if got == oracle.OK:
                            free += held[actor]
                            held[actor] = 0
                    assert got == exp
                    assert a.free_blocks == free
                    _check_invariants(a)


def test_randomized_linearizability_1e5_ops():
    """>= 1e5 ops, 2-8 actors: invariants hold after every op and the
    free-count model matches; statuses OOM exactly when the model says so."""
    rng = np.random.default_rng(2024)
    total = 0
    while total < 100_000:
        n_act = int(rng.integers(2, 9))
        N_B = int(rng.integers(8, 64))
        a = oracle.Allocator(N_B, n_act, 64)
        free, held = N_B, [0] * n_act
        for _ in range(2500):
            actor = int(rng.integers(n_act))
            if rng.random() < 0.6:
                n = int(rng.integers(1, 9))
                got = a.alloc([actor], [n])
                exp = oracle.OK if n <= free else oracle.OOM
                if exp == oracle.OK and held[actor] + n > 64:
                    exp = oracle.TABLE_FULL
                assert got == exp
                if got == oracle.OK:
                    free -= n
                    held[actor] += n
            else:
                got = a.free([actor])
                assert got == (oracle.OK if held[actor] else oracle.UNKNOWN_REQ)
                if got == oracle.OK:
                    free += held[actor]
                    held[actor] = 0
            assert a.free_blocks == free
            total += 1
        _check_invariants(a)
    assert total >= 100_000


# --------------------------------------------------------------------------- partition
def test_partition_examples():
    assert (oracle.sm_budget(148, 50), oracle.sm_budget(148, 50)) == (74, 74)
    assert (oracle.sm_budget(148, 30), oracle.sm_budget(148, 70)) == (44, 104)
    assert (oracle.sm_budget(148, 100), oracle.sm_budget(148, 100)) == (148, 148)
    assert oracle.sm_budget(148, 0.1) == 1 and oracle.sm_budget(148, 0) == -1
    assert oracle.sm_budget(148, 100.5) == -1
    # SPEC effective_shares: model view only
    assert oracle.effective_shares(30, 70) == (30, 70)
    assert oracle.effective_shares(100, 100) == (50, 50)
    xe, ye = oracle.effective_shares(80, 40)
    assert abs(xe - 66.6667) < 1e-3 and abs(ye - 33.3333) < 1e-3
