"""GPU parity of the expanded-form MLA prefill (R32) against
the fp64 oracle (`oracle.prefill_mla_expanded`, pinned in tests/test_oracle_mla_exp_pins.py):
outputs within the bf16 tolerance (2e-2 max abs, 1e-2 Frobenius-relative), the chunk's latent
rows written to the pool bit for bit, bitwise identical outputs for every SM budget, and the
error paths (BAD_BLOCK, a too-small max_total_keys, UNSUPPORTED pools)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth
from harness import Rig, compare, np_bits

pytestmark = pytest.mark.gpu

H = 16


def _shape(bs, nh=H):
    s = synth.CFG5_MLA
    return synth.AttnShape(s.name, nh, 1, 576, 512, bs, torch.bfloat16, num_layers=1, kv_shared=True,
                           scale=s.scale)


def run_exp(chunks, prefixes, seed, dist=synth.FLAT, bs=64, sm_budget=0, rows_mask=None,
            bad_entry=None, max_total_keys=None, check=True, nh=H):
    case = synth.mla_expanded_case(chunks, prefixes, seed, nh, dist)
    n = len(chunks)
    nk = [p + c for p, c in zip(prefixes, chunks)]
    need = [-(-k // bs) for k in nk]
    mbr = max(need) + 1
    rig = Rig(_shape(bs, nh), num_blocks=sum(need) + 3, max_reqs=n, mbr=mbr)
    for i in range(n):
        rig.alloc([i], [need[i]])
    K, _, BT, _ = rig.pool.views(0)
    bt = BT.cpu().numpy().copy()
    K.zero_()
    for i in range(n):  # the cached prefix rows (bit copies; harness)
        for j in range(prefixes[i]):
            K[bt[i, j // bs], 0, j % bs] = case.lat[i][j].to(rig.dev)
    if bad_entry is not None:  # corrupt one table entry (row, page) -> -1
        BT[bad_entry[0], bad_entry[1]] = -1
        bt[bad_entry[0], bad_entry[1]] = -1
    pool_ref = np_bits(K)
    dev = rig.dev
    T = case.cu[-1]
    mtk = sum(nk) if max_total_keys is None else max_total_keys
    ws = rig.pool.new_mla_expanded_workspace(n, mtk, nh)
    ws.fill_(0xFF)  # NaN patterns: the kernels must not read workspace rows they did not write
    out = torch.full((T, nh, 128), float("nan"), dtype=torch.bfloat16, device=dev)
    rig.pool.prefill_mla_expanded(0, case.q.to(dev), case.kv_new.to(dev), case.w_uk.to(dev),
                                  case.w_uv.to(dev), rig.i32(case.cu), rig.i32(range(n)),
                                  rig.i32(prefixes), T, max(chunks), mtk, case.scale, out, ws,
                                  sm_budget=sm_budget, status=rig.status)
    torch.cuda.synchronize()
    st = int(rig.status.item())
    if not check:
        return out, st, dict(case=case, pool_ref=pool_ref, bt=bt)
    assert st == 0, st
    ref = oracle.prefill_mla_expanded(np_bits(case.q), np_bits(case.kv_new), pool_ref, bt,
                                      np.array(case.cu, np.int32), np.arange(n, dtype=np.int32),
                                      np.array(prefixes, np.int32), np_bits(case.w_uk),
                                      np_bits(case.w_uv), case.scale, rows_mask=rows_mask)
    got = out.float().cpu().double().numpy()
    rows = np.arange(T) if rows_mask is None else np.nonzero(rows_mask)[0]
    compare(got[rows], ref[rows], torch.bfloat16, f"mla_expanded {chunks} {prefixes} bs{bs}")
    # step 1: the pool after the call equals the oracle's pool, bit for bit
    np.testing.assert_array_equal(np_bits(K), pool_ref)
    return out, st, rig


@pytest.mark.parametrize("chunks,prefixes", [([128], [0]), ([37], [100]), ([3, 70, 130], [0, 64, 5]),
                                             ([1, 200], [0, 300]), ([256, 255], [0, 1])])
@pytest.mark.parametrize("dist", synth.DISTS)
def test_mla_expanded_parity(chunks, prefixes, dist):
    run_exp(chunks, prefixes, seed=700 + dist, dist=dist)


@pytest.mark.parametrize("nh", [2, 8, 32])
def test_mla_expanded_head_counts(nh):
    """Other head counts (a TP shard of the 16 heads, a wider model): the GEMM's n-tiles are
    head pairs, the attention's units per head."""
    run_exp([200, 57], [30, 140], seed=750 + nh, nh=nh, dist=synth.PEAKED)


@pytest.mark.parametrize("bs", [16, 32, 128])
def test_mla_expanded_block_sizes(bs):
    run_exp([190, 33], [45, 130], seed=710 + bs, bs=bs, dist=synth.PEAKED)


def test_mla_expanded_bitwise_across_budgets():
    outs = [run_exp([300, 90], [70, 0], seed=720, sm_budget=b)[0].cpu() for b in (1, 7, 74, 148, -1)]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_mla_expanded_full_chunk_sampled():
    """cfg 5 prefill chunk at full size (C = 2048, P = 0): every 32nd row + the last."""
    T = 2048
    mask = np.zeros(T, np.uint8)
    mask[::32] = 1
    mask[-1] = 1
    run_exp([T], [0], seed=730, rows_mask=mask)


def test_mla_expanded_long_prefix_sampled():
    """A 2048-token chunk behind a 6000-token cached prefix (the prefix is re-expanded)."""
    T = 2048
    mask = np.zeros(T, np.uint8)
    mask[::128] = 1
    mask[-1] = 1
    run_exp([T], [6000], seed=731, rows_mask=mask, dist=synth.VSHIFT)


def test_mla_expanded_many_requests():
    rng = np.random.default_rng(732)
    chunks = [int(x) for x in rng.integers(1, 90, 40)]
    prefixes = [int(x) for x in rng.integers(0, 200, 40)]
    run_exp(chunks, prefixes, seed=732)


def test_mla_expanded_bad_block():
    """A -1 table entry inside request 1's prefix: status BAD_BLOCK, no fault, request 0 exact."""
    chunks, prefixes = [60, 50], [10, 150]
    out, st, r = run_exp(chunks, prefixes, seed=740, bad_entry=(1, 1), check=False)
    assert st == 5
    case = r["case"]
    ref = oracle.prefill_mla_expanded(np_bits(case.q[:60]), np_bits(case.kv_new[:60]), r["pool_ref"],
                                      r["bt"], np.array([0, 60], np.int32), np.array([0], np.int32),
                                      np.array([10], np.int32), np_bits(case.w_uk), np_bits(case.w_uv),
                                      case.scale)
    compare(out[:60].float().cpu().double().numpy(), ref, torch.bfloat16, "request 0 beside a bad block")
    assert torch.isfinite(out[60:].float()).all()


def test_mla_expanded_max_total_keys_too_small():
    out, st, _ = run_exp([100, 50], [30, 0], seed=741, max_total_keys=10, check=False)
    assert st == 1  # INVALID, nothing computed


def test_mla_expanded_kernel_kind_and_unsupported_pool():
    from paper_2504_19867_b200 import KVPool, PoolConfig, SemipdError
    dev = torch.device("cuda", 0)
    pool = KVPool(PoolConfig(1, 8, 64, 1, 576, 512, 2, 4, kv_shared=True), dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32([0]), i32([2]))
    trace = torch.zeros(4 * 256, dtype=torch.int32, device=dev)
    ctr = torch.zeros(1, dtype=torch.int32, device=dev)
    pool.set_trace(trace, ctr)
    q = torch.randn(100, H, 192, device=dev).bfloat16()
    kn = torch.randn(100, 576, device=dev).bfloat16()
    w = torch.randn(H, 128, 512, device=dev).bfloat16() / 20
    out = torch.empty(100, H, 128, dtype=torch.bfloat16, device=dev)
    ws = pool.new_mla_expanded_workspace(1, 100, H)
    pool.prefill_mla_expanded(0, q, kn, w, w, i32([0, 100]), i32([0]), i32([0]), 100, 100, 100, 0.07,
                              out, ws)
    torch.cuda.synchronize()
    n = int(ctr.item())
    assert n > 0 and set(trace[:4 * n].view(n, 4)[:, 3].cpu().tolist()) == {10}
    # a GQA (not latent) pool is UNSUPPORTED
    gpool = KVPool(PoolConfig(1, 8, 64, 8, 128, 128, 2, 4), dev)
    assert gpool.mla_expanded_workspace_bytes(1, 100, H) == 0
    with pytest.raises(SemipdError):
        gpool.prefill_mla_expanded(0, q, kn, w, w, i32([0, 100]), i32([0]), i32([0]), 100, 100, 100,
                                   0.07, out, ws)


def test_mla_expanded_total_q_smaller_than_cu():
    """A cu_seqlens_q[n] beyond the host's total_q: status INVALID, nothing read past kv_new and
    nothing stored past out (a guard region after the output stays untouched)."""
    from paper_2504_19867_b200 import KVPool, PoolConfig
    dev = torch.device("cuda", 0)
    pool = KVPool(PoolConfig(1, 8, 64, 1, 576, 512, 2, 4, kv_shared=True), dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32([0]), i32([2]))
    T = 60  # the host says 60 rows; cu says 100
    q = torch.randn(T, H, 192, device=dev).bfloat16()
    kn = torch.randn(T, 576, device=dev).bfloat16()
    w = (torch.randn(H, 128, 512, device=dev) / 22.6).bfloat16()
    buf = torch.full((T + 64, H, 128), 7.0, dtype=torch.bfloat16, device=dev)
    out = buf[:T]
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = pool.new_mla_expanded_workspace(1, 100, H)
    pool.prefill_mla_expanded(0, q, kn, w, w, i32([0, 100]), i32([0]), i32([0]), T, 100, 100, 0.07,
                              out, ws, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 1
    assert torch.all(buf[T:] == 7.0)


@pytest.mark.parametrize("inter", [True, False], ids=["interleaved", "half_split"])
def test_mla_expanded_fused_rope_bitwise(inter):
    """RoPE set on the pool (semipd_set_rope, R28) on the decoupled columns: the call rotates
    q_pe = q[..., 128:192] and k_pe = kv_new[..., 512:576] in place at prefix + t before the
    prep writes the chunk's latent rows.  q, kv_new, the pool and the output equal the composed
    path (semipd_rope on the two column ranges, then the plain call) bit for bit, and the output
    matches the oracle over the rotated rows."""
    from paper_2504_19867_b200 import RopeConfig, rope_
    ds = RopeConfig(theta=10000.0, factor=0.0)
    chunks, prefixes = [100, 37], [0, 70]
    case = synth.mla_expanded_case(chunks, prefixes, 91, H, synth.FLAT)
    n, bs = len(chunks), 64
    need = [-(-(p + c) // bs) for p, c in zip(prefixes, chunks)]
    pos = np.concatenate([np.arange(p, p + c) for c, p in zip(chunks, prefixes)]).astype(np.int32)
    res = []
    for fused in (True, False):
        rig = Rig(_shape(bs), num_blocks=sum(need) + 3, max_reqs=n, mbr=max(need) + 1)
        for i in range(n):
            rig.alloc([i], [need[i]])
        K, _, BT, _ = rig.pool.views(0)
        bt = BT.cpu().numpy().copy()
        K.zero_()
        for i in range(n):
            for j in range(prefixes[i]):
                K[bt[i, j // bs], 0, j % bs] = case.lat[i][j].to(rig.dev)
        pool_ref = np_bits(K)
        dev = rig.dev
        q, kv = case.q.to(dev).contiguous(), case.kv_new.to(dev).contiguous()
        T = case.cu[-1]
        if fused:
            rig.pool.set_rope(ds, rot_offset=512, rot_dim=64, interleaved=inter)
        else:
            p32 = torch.from_numpy(pos).to(dev)
            rope_(q, None, p32, ds, rot_offset=128, rot_dim=64, interleaved=inter)
            rope_(None, kv.view(T, 1, 576), p32, ds, rot_offset=512, rot_dim=64, interleaved=inter)
        ws = rig.pool.new_mla_expanded_workspace(n, sum(need) * bs, H)
        out = torch.empty((T, H, 128), dtype=torch.bfloat16, device=dev)
        rig.pool.prefill_mla_expanded(0, q, kv, case.w_uk.to(dev), case.w_uv.to(dev), rig.i32(case.cu),
                                      rig.i32(range(n)), rig.i32(prefixes), T, max(chunks),
                                      sum(need) * bs, case.scale, out, ws, status=rig.status)
        torch.cuda.synchronize()
        assert int(rig.status.item()) == 0
        res.append((out, q, kv, np_bits(K), pool_ref, bt))
    (of, qf, kf, Kf, pref, bt), (oc, qc, kc, Kc, _, _) = res
    eq = lambda a, b: torch.equal(a.contiguous().view(torch.uint8), b.contiguous().view(torch.uint8))  # noqa: E731
    assert eq(qf, qc) and eq(kf, kc), "rotated rows differ from semipd_rope's"
    assert not eq(qf.cpu(), case.q), "q was not rotated"
    assert eq(qf[..., :128].cpu(), case.q[..., :128]) and eq(kf[..., :512].cpu(), case.kv_new[..., :512])
    np.testing.assert_array_equal(Kf, Kc)
    assert eq(of, oc), "fused output differs from the composed path"
    ref = oracle.prefill_mla_expanded(np_bits(qf), np_bits(kf), pref, bt, np.array(case.cu, np.int32),
                                      np.arange(n, dtype=np.int32), np.array(prefixes, np.int32),
                                      np_bits(case.w_uk), np_bits(case.w_uv), case.scale)
    compare(of.float().cpu().double().numpy(), ref, torch.bfloat16, "mla_expanded + rope vs oracle")
