"""FP8 (E4M3) KV pages on the GPU vs the oracle (reading R31).

Every case runs the CUDA path through the binding and ``oracle.{decode,prefill}_fp8`` on the
same seeded inputs.  Cached context is put in the pool as the oracle's codes of synthetic
bf16 K / V (``oracle.e4m3_quantize``: an input, never a CUDA result).  Checked:
  * pool codes after the quantised append / chunk write: bit-exact;
  * attention outputs: the bf16 tolerance of harness.TOL (decode computes in f16 / fp32:
    E4M3 -> f16 is exact, q rounds bf16 -> f16, P rounds to f16; the prefill prefix stages K
    as value(code) exactly (k_scale goes into the logit scale) and V as bf16(v_scale *
    value(code)) — one relative 2^-9 rounding of V, the order of the P rounding the bf16
    path already has);
  * bitwise identical outputs for every SM budget (R26), BAD_BLOCK without a fault, the
    host error paths, and the trace's kernel kind (9).
"""

import numpy as np
import pytest
import torch

import oracle
import synth
from harness import compare, np_bits

pytestmark = pytest.mark.gpu

F8 = torch.float8_e4m3fn
SHAPE = synth.AttnShape("llama3-8b-fp8", 32, 8, 128, 128, 64, torch.bfloat16)


class F8Rig:
    def __init__(self, shape, num_blocks, max_reqs, mbr, num_layers=1, ks=0.05, vs=0.02):
        from paper_2504_19867_b200 import KVPool, PoolConfig
        self.shape = shape
        self.cfg = PoolConfig(num_layers, num_blocks, shape.block_size, shape.num_kv_heads,
                              shape.head_dim_k, shape.head_dim_v, max_reqs, mbr, dtype=F8)
        self.pool = KVPool(self.cfg, 0)
        self.dev = self.pool.device
        self.ks, self.vs = ks, vs
        self.pool.set_kv_scales(ks, vs)
        self.ref_alloc = oracle.Allocator(num_blocks, max_reqs, mbr)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)

    def i32(self, xs):
        return torch.tensor(list(xs), dtype=torch.int32, device=self.dev)

    def alloc(self, ids, counts):
        self.pool.alloc_blocks(self.i32(ids), self.i32(counts), self.status)
        assert int(self.status.item()) == 0
        assert self.ref_alloc.alloc(ids, counts) == 0

    def put(self, layer, rid, k_tok, v_tok, start=0):
        """Cached context of request rid at positions start..: the oracle's codes."""
        if k_tok.shape[0] == 0:
            return
        K, V, _, _ = self.pool.views(layer)
        kc = torch.from_numpy(oracle.e4m3_quantize(np_bits(k_tok), self.ks))
        vc = torch.from_numpy(oracle.e4m3_quantize(np_bits(v_tok), self.vs))
        bs = self.shape.block_size
        pos = torch.arange(start, start + k_tok.shape[0])
        blk = torch.from_numpy(self.ref_alloc.bt[rid]).long()[pos // bs]
        K[blk.to(self.dev), :, (pos % bs).to(self.dev)] = kc.to(self.dev)
        V[blk.to(self.dev), :, (pos % bs).to(self.dev)] = vc.to(self.dev)

    def host_pool(self, layer=0):
        K, V, _, _ = self.pool.views(layer)
        return K.cpu().numpy().copy(), V.cpu().numpy().copy()


def run_decode(ctx, seed, dist=synth.FLAT, ks=0.05, vs=0.02, sm_budget=0, shape=SHAPE,
               head_major=False, check_append=True, rig=None):
    bs = shape.block_size
    B = len(ctx)
    nb = [c // bs + 1 for c in ctx]
    if rig is None:
        rig = F8Rig(shape, sum(nb) + 3, B + 1, max(nb) + 1, ks=ks, vs=vs)
        rig.alloc(range(B), nb)
    case = synth.decode_case(shape, ctx, seed, dist)
    for b in range(B):
        rig.put(0, b, case.k_ctx[b], case.v_ctx[b])
    kp, vp = rig.host_pool()
    dev = rig.dev
    Hq, dv = shape.num_q_heads, shape.head_dim_v
    out = torch.empty((Hq, B, dv) if head_major else (B, Hq, dv), dtype=torch.bfloat16, device=dev)
    ws = rig.pool.new_decode_workspace(B, Hq, max(ctx))
    rig.pool.decode_attn(0, case.q.to(dev), case.k_new.to(dev), case.v_new.to(dev), rig.i32(range(B)),
                         rig.i32(ctx), max(ctx), shape.softmax_scale, out, ws,
                         out_head_major=head_major, sm_budget=sm_budget, status=rig.status)
    torch.cuda.synchronize()
    assert int(rig.status.item()) == 0
    ref = oracle.decode_fp8(np_bits(case.q), np_bits(case.k_new), np_bits(case.v_new), kp, vp,
                            rig.ref_alloc.bt, np.arange(B), ctx, shape.softmax_scale, rig.ks, rig.vs)
    got = out.float().cpu().double().numpy()
    if head_major:
        got = got.transpose(1, 0, 2)
    m = compare(got, ref, torch.bfloat16, f"fp8 decode dist{dist}")
    if check_append:
        K, V = rig.host_pool()
        np.testing.assert_array_equal(K, kp)  # the oracle appended its codes into kp / vp
        np.testing.assert_array_equal(V, vp)
    return out, m


@pytest.mark.parametrize("dist", synth.DISTS)
def test_fp8_decode_parity(dist):
    # ctx covers: empty context (only the appended key), page edges, ragged tails, > 1 split
    run_decode([0, 1, 63, 64, 65, 255, 2048, 4095, 4096, 9000], seed=3100 + dist, dist=dist)


@pytest.mark.parametrize("ks,vs", [(1.0, 1.0), (0.011, 0.37), (2.0 ** -5, 2.0 ** -3)])
def test_fp8_decode_scales(ks, vs):
    run_decode([5, 300, 4500], seed=3110, dist=synth.VSHIFT, ks=ks, vs=vs)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_fp8_decode_gqa_groups(G):
    shape = synth.AttnShape("fp8-g", 2 * G, 2, 128, 128, 64, torch.bfloat16)
    run_decode([33, 700, 5000], seed=3120 + G, dist=synth.NEEDLE, shape=shape)


def test_fp8_decode_head_major():
    run_decode([100, 3000], seed=3130, head_major=True)


def test_fp8_decode_bitwise_stable_across_budgets():
    outs = [run_decode([130, 4200, 9999], seed=3140, sm_budget=b)[0].cpu() for b in (1, 7, 89, 148, -1)]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_fp8_decode_full_size_cfg2():
    """cfg 2's decode batch (B = 64 at ctx 2048) at the bench's 89-SM budget, every request and
    head against the oracle."""
    run_decode([2048] * 64, seed=3150, sm_budget=89, check_append=True)


def test_fp8_decode_trace_kind_and_bad_block():
    ctx = [100, 200]
    rig = F8Rig(SHAPE, 12, 3, 6)
    rig.alloc([0, 1], [2, 4])
    trace = torch.zeros(4 * 4096, dtype=torch.int32, device=rig.dev)
    ctr = torch.zeros(1, dtype=torch.int32, device=rig.dev)
    rig.pool.set_trace(trace, ctr)
    run_decode(ctx, seed=3160, rig=rig)
    n = int(ctr.item())
    assert n > 0 and set(trace[:4 * n].view(n, 4)[:, 3].cpu().tolist()) == {9}
    rig.pool.set_trace(None)
    # corrupt request 1's first table entry: BAD_BLOCK, request 0 still exact
    _, _, BT, _ = rig.pool.views(0)
    BT[1, 0] = -1
    case = synth.decode_case(SHAPE, ctx, 3161)
    out = torch.empty(2, 32, 128, dtype=torch.bfloat16, device=rig.dev)
    ws = rig.pool.new_decode_workspace(2, 32, 200)
    kp, vp = rig.host_pool()
    rig.pool.decode_attn(0, case.q.cuda(), case.k_new.cuda(), case.v_new.cuda(), rig.i32([0, 1]),
                         rig.i32(ctx), 200, SHAPE.softmax_scale, out, ws, status=rig.status)
    torch.cuda.synchronize()
    assert int(rig.status.item()) == 5
    ref = oracle.decode_fp8(np_bits(case.q[:1]), np_bits(case.k_new[:1]), np_bits(case.v_new[:1]),
                            kp, vp, rig.ref_alloc.bt, [0], ctx[:1], SHAPE.softmax_scale, rig.ks, rig.vs)
    compare(out[:1].float().cpu().double().numpy(), ref, torch.bfloat16, "fp8 decode next to a bad row")


# --------------------------------------------------------------------------- prefill
def run_prefill(chunks, prefix, seed, dist=synth.FLAT, ks=0.05, vs=0.02, sm_budget=0,
                rows_every=1, head_major=False):
    shape = SHAPE
    bs = shape.block_size
    n = len(chunks)
    nb = [(p + c + bs - 1) // bs for p, c in zip(prefix, chunks)]
    rig = F8Rig(shape, sum(nb) + 2, n + 1, max(nb) + 1, ks=ks, vs=vs)
    rig.alloc(range(n), nb)
    rig.pool.attach_fp8_prefill_scratch(n)
    case = synth.prefill_case(shape, chunks, prefix, seed, dist)
    for i in range(n):
        rig.put(0, i, case.k_prefix[i], case.v_prefix[i])
    kp, vp = rig.host_pool()
    dev = rig.dev
    T = sum(chunks)
    cu = np.concatenate([[0], np.cumsum(chunks)]).astype(np.int32)
    Hq = shape.num_q_heads
    out = torch.zeros((Hq, T, 128) if head_major else (T, Hq, 128), dtype=torch.bfloat16, device=dev)
    rig.pool.prefill_attn(0, case.q.to(dev), case.k_new.to(dev), case.v_new.to(dev), rig.i32(cu),
                          rig.i32(range(n)), rig.i32(prefix), T, max(chunks), shape.softmax_scale,
                          out, out_head_major=head_major, sm_budget=sm_budget, status=rig.status)
    torch.cuda.synchronize()
    assert int(rig.status.item()) == 0
    mask = np.zeros(T, np.uint8)
    mask[::rows_every] = 1
    mask[cu[1:] - 1] = 1
    ref = oracle.prefill_fp8(np_bits(case.q), np_bits(case.k_new), np_bits(case.v_new), kp, vp,
                             rig.ref_alloc.bt, cu, np.arange(n), prefix, shape.softmax_scale,
                             rig.ks, rig.vs, rows_mask=mask)
    got = out.float().cpu().double().numpy()
    if head_major:
        got = got.transpose(1, 0, 2)
    rows = mask.astype(bool)
    m = compare(got[rows], ref[rows], torch.bfloat16, f"fp8 prefill {chunks} P={prefix}")
    K, V = rig.host_pool()
    np.testing.assert_array_equal(K, kp)  # the quantised chunk write, bit-exact
    np.testing.assert_array_equal(V, vp)
    return out, m


@pytest.mark.parametrize("dist", synth.DISTS)
def test_fp8_prefill_with_prefix(dist):
    run_prefill([100, 1, 257], [0, 64, 300], seed=3200 + dist, dist=dist)


def test_fp8_prefill_long_prefix_head_major():
    run_prefill([384], [5000], seed=3210, head_major=True, ks=0.013, vs=0.4)


def test_fp8_prefill_full_chunk_cfg2():
    """The bench's prefill chunk (C = 2048, P = 0) at the 59-SM budget; every 16th row."""
    run_prefill([2048], [0], seed=3220, sm_budget=59, rows_every=16)


def test_fp8_prefill_bitwise_stable_across_budgets():
    outs = [run_prefill([300, 77], [129, 0], seed=3230, sm_budget=b)[0].cpu() for b in (3, 59, 148)]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_fp8_host_errors():
    from paper_2504_19867_b200 import KVPool, PoolConfig, RopeConfig, SemipdError
    # geometry the FP8 kernels do not cover
    with pytest.raises(SemipdError, match="UNSUPPORTED"):
        KVPool(PoolConfig(1, 8, 16, 8, 128, 128, 2, 4, dtype=F8), 0)
    rig = F8Rig(SHAPE, 8, 4, 4)
    rig.alloc([0, 1], [1, 1])
    rig.pool.set_rope(RopeConfig(theta=500000.0))  # E4M3 pools take fused RoPE (R28 + R31)
    with pytest.raises(SemipdError, match="INVALID"):
        rig.pool.set_rope(RopeConfig(theta=1.0))
    rig.pool.set_rope(None)
    with pytest.raises(SemipdError, match="INVALID"):
        rig.pool.set_kv_scales(0.0, 1.0)
    q = torch.zeros(2, 32, 128, dtype=torch.bfloat16, device=rig.dev)
    kv = torch.zeros(2, 8, 128, dtype=torch.bfloat16, device=rig.dev)
    out = torch.empty_like(q)
    args = (0, q, kv, kv, rig.i32([0, 1, 2]), rig.i32([0, 1]), rig.i32([0, 0]), 2, 1, 0.1, out)
    with pytest.raises(SemipdError, match="INVALID"):  # no staging scratch
        rig.pool.prefill_attn(*args)
    rig.pool.attach_fp8_prefill_scratch(1)
    with pytest.raises(SemipdError, match="INVALID"):  # more requests than the scratch holds
        rig.pool.prefill_attn(*args)
    q16 = torch.zeros(2, 8 * 16, 128, dtype=torch.bfloat16, device=rig.dev)
    ws = rig.pool.new_decode_workspace(2, 128, 10)
    with pytest.raises(SemipdError, match="UNSUPPORTED"):  # G = 16 > 8
        rig.pool.decode_attn(0, q16, kv, kv, rig.i32([0, 1]), rig.i32([3, 3]), 3, 0.1,
                             torch.empty_like(q16), ws)
