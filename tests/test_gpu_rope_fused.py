"""RoPE fused with the attention calls' K/V write (C ABI ``semipd_set_rope``; SURVEY §8(f) N4,
PAPER P:355 §6, DESIGN R27 / R28).

With RoPE set on the pool, ``prefill_attn`` / ``decode_attn`` rotate the step's q / k_new in
place at the positions the call's layout implies (prefill: prefix + t, R4; decode: ctx, R5)
and write the rotated rows into the pool in the same pass; the attention kernels skip their
own K/V write.  Checks, on the same seeded inputs:
- bitwise: the fused call leaves q, k_new, the pool and the output identical to the composed
  path (semipd_rope at those positions, then the plain call), for the tcgen05 / split-K cfg-2
  kernels, the MLA latent kernels (rope on the 64 decoupled columns, interleaved) and the fp32
  generic path;
- oracle: the fused prefill output equals the oracle's attention over the oracle's rotated
  q / k (fp64 rotation), within the bf16 bar."""
import numpy as np
import pytest
import torch

import oracle
import synth
from harness import Rig, compare, np_bits
from paper_2504_19867_b200 import RopeConfig, rope_

pytestmark = pytest.mark.gpu

LLAMA31 = RopeConfig()
DS = RopeConfig(theta=10000.0, factor=0.0)


def _ocfg(c: RopeConfig):
    return dict(theta=c.theta, factor=c.factor, lf=c.low_freq_factor, hf=c.high_freq_factor,
                L0=float(c.original_max_pos))


def _shape(base, **kw):
    d = dict(name=base.name, num_q_heads=base.num_q_heads, num_kv_heads=base.num_kv_heads,
             head_dim_k=base.head_dim_k, head_dim_v=base.head_dim_v, block_size=base.block_size,
             dtype=base.dtype, num_layers=1, kv_shared=base.kv_shared, scale=base.scale)
    d.update(kw)
    return synth.AttnShape(**d)


def _prefill_pair(shape, chunks, prefixes, cfg, seed, **rk):
    """(fused rig, composed rig) after the same prefill; returns outputs and rotated rows."""
    res = []
    case = synth.prefill_case(shape, chunks, prefixes, seed, synth.FLAT)
    bs = shape.block_size
    nblk = [-(-(c + p) // bs) for c, p in zip(chunks, prefixes)]
    cu = case.cu_seqlens
    pos = np.concatenate([np.arange(p, p + c) for c, p in zip(chunks, prefixes)]).astype(np.int32)
    for fused in (True, False):
        rig = Rig(shape, num_blocks=sum(nblk) + 3, max_reqs=len(chunks) + 1, mbr=max(nblk) + 1)
        for i, n in enumerate(nblk):
            rig.alloc([i], [n])
        for i in range(len(chunks)):
            rig.scatter(0, i, case.k_prefix[i], case.v_prefix[i])
        dev = rig.dev
        q, k = case.q.to(dev).contiguous(), case.k_new.to(dev).contiguous()
        v = None if case.v_new is None else case.v_new.to(dev).contiguous()
        T = sum(chunks)
        out = torch.empty(T, shape.num_q_heads, shape.head_dim_v, dtype=shape.dtype, device=dev)
        if fused:
            rig.pool.set_rope(cfg, **rk)
        else:
            rope_(q, k, torch.from_numpy(pos).to(dev), cfg, **rk)
        rig.pool.prefill_attn(0, q, k, v, rig.i32(cu), rig.i32(range(len(chunks))),
                              rig.i32(prefixes), T, max(chunks), shape.softmax_scale, out,
                              status=rig.status)
        torch.cuda.synchronize()
        assert int(rig.status.item()) == 0
        res.append((rig, out, q, k))
    return case, pos, res


def _bitwise(a, b):
    return torch.equal(a.contiguous().view(torch.uint8), b.contiguous().view(torch.uint8))


@pytest.mark.parametrize("chunks,prefixes", [([300], [0]), ([130, 77, 1], [64, 500, 7])])
def test_fused_rope_prefill_cfg2_bitwise_and_oracle(chunks, prefixes):
    shape = _shape(synth.CFG2_LLAMA8B, block_size=64)
    case, pos, ((rf, of, qf, kf), (rc, oc, qc, kc)) = _prefill_pair(shape, chunks, prefixes,
                                                                     LLAMA31, 61)
    assert _bitwise(qf, qc) and _bitwise(kf, kc), "rotated rows differ from semipd_rope's"
    assert _bitwise(of, oc), "fused output differs from the composed path"
    Kf, Vf = rf.host_pool(0)
    Kc, Vc = rc.host_pool(0)
    assert np.array_equal(Kf, Kc) and np.array_equal(Vf, Vc), "pool pages differ"
    # oracle chain: fp64 rotation of the chunk's q / k (prefix keys are stored unrotated
    # inputs, as cached rows would be), then the oracle's paged prefill
    qr = oracle.rope(np_bits(case.q), pos, **_ocfg(LLAMA31)).astype(np.float32)
    kr = oracle.rope(np_bits(case.k_new), pos, **_ocfg(LLAMA31)).astype(np.float32)
    kp, vp = rf.host_pool(0)
    f32 = lambda a: (a.astype(np.uint32) << 16).view(np.float32)  # noqa: E731 (bf16 bits)
    kp32, vp32 = f32(kp), f32(vp)
    ref = oracle.prefill(qr, kr, case.v_new.float().numpy(), kp32, vp32, rf.ref_alloc.bt,
                         case.cu_seqlens, list(range(len(chunks))), prefixes,
                         shape.softmax_scale)
    compare(of.float().cpu().double().numpy(), ref, torch.bfloat16, "fused rope prefill vs oracle")


@pytest.mark.parametrize("bs", [16, 64])
def test_fused_rope_decode_cfg2_bitwise(bs):
    shape = _shape(synth.CFG2_LLAMA8B, block_size=bs)
    ctx = [0, 15, 64, 700, 4097, 2048]
    case = synth.decode_case(shape, ctx, 62, synth.NEEDLE)
    outs = []
    for fused in (True, False):
        nblk = [c // bs + 1 for c in ctx]
        rig = Rig(shape, num_blocks=sum(nblk) + 2, max_reqs=len(ctx) + 1, mbr=max(nblk) + 1)
        for b, n in enumerate(nblk):
            rig.alloc([b], [n])
        for b in range(len(ctx)):
            rig.scatter(0, b, case.k_ctx[b], case.v_ctx[b])
        dev = rig.dev
        q, k, v = (t.to(dev).contiguous() for t in (case.q, case.k_new, case.v_new))
        out = torch.empty(len(ctx), 32, 128, dtype=torch.bfloat16, device=dev)
        if fused:
            rig.pool.set_rope(LLAMA31)
        else:
            rope_(q, k, rig.i32(ctx), LLAMA31)
        rig.pool.decode_attn(0, q, k, v, rig.i32(range(len(ctx))), rig.i32(ctx), max(ctx),
                             shape.softmax_scale, out, rig.pool.new_decode_workspace(len(ctx), 32, max(ctx)),
                             status=rig.status)
        torch.cuda.synchronize()
        assert int(rig.status.item()) == 0
        outs.append((out, q, k, rig.host_pool(0)))
    (of, qf, kf, (Kf, Vf)), (oc, qc, kc, (Kc, Vc)) = outs
    assert _bitwise(qf, qc) and _bitwise(kf, kc)
    assert _bitwise(of, oc)
    assert np.array_equal(Kf, Kc) and np.array_equal(Vf, Vc)


@pytest.mark.parametrize("inter", [True, False], ids=["interleaved", "half_split"])
def test_fused_rope_mla_prefill_and_decode_bitwise(inter):
    """cfg 5 latent rows: rope on the 64 decoupled columns at 512; the 512 latent columns
    reach the pool untouched."""
    shape = _shape(synth.CFG5_MLA)
    rk = dict(rot_offset=512, rot_dim=64, interleaved=inter)
    case, pos, ((rf, of, qf, kf), (rc, oc, qc, kc)) = _prefill_pair(shape, [100, 33], [0, 70],
                                                                     DS, 63, **rk)
    assert _bitwise(qf, qc) and _bitwise(kf, kc) and _bitwise(of, oc)
    assert np.array_equal(rf.host_pool(0)[0], rc.host_pool(0)[0])
    assert _bitwise(kf[..., :512].cpu(), case.k_new[..., :512])
    # decode on the same pools (ctx = prefix + chunk of each request)
    ctx = [100, 103]
    dc = synth.decode_case(shape, ctx, 64, synth.FLAT, req_ids=[0, 1])
    res = []
    for rig, fused in ((rf, True), (rc, False)):
        dev = rig.dev
        q, k = dc.q.to(dev).contiguous(), dc.k_new.to(dev).contiguous()
        if not fused:
            rope_(q, k, rig.i32(ctx), DS, **rk)
        out = torch.empty(2, 16, 512, dtype=torch.bfloat16, device=dev)
        rig.pool.decode_attn(0, q, k, None, rig.i32([0, 1]), rig.i32(ctx), max(ctx),
                             shape.softmax_scale, out, rig.pool.new_decode_workspace(2, 16, max(ctx)),
                             status=rig.status)
        torch.cuda.synchronize()
        assert int(rig.status.item()) == 0
        res.append((out, q, k, rig.host_pool(0)[0]))
    assert _bitwise(res[0][0], res[1][0]) and _bitwise(res[0][1], res[1][1])
    assert np.array_equal(res[0][3], res[1][3])


def test_fused_rope_fp32_generic_path_bitwise():
    shape = synth.CFG1_TINY
    case, pos, ((rf, of, qf, kf), (rc, oc, qc, kc)) = _prefill_pair(shape, [37, 91], [0, 40],
                                                                     DS, 65)
    assert _bitwise(qf, qc) and _bitwise(kf, kc) and _bitwise(of, oc)
    Kf, Vf = rf.host_pool(0)
    Kc, Vc = rc.host_pool(0)
    assert np.array_equal(Kf, Kc) and np.array_equal(Vf, Vc)


@pytest.mark.parametrize("inter", [False, True], ids=["half_split", "interleaved"])
def test_fused_rope_fp8_decode_and_prefill_bitwise(inter):
    """E4M3 pools (R31): with RoPE set, one pass rotates q / k_new and writes the rotated K and
    the V rows as E4M3 codes; the FP8 kernels skip their own quantised write.  The pool codes,
    the rotated rows and the outputs must equal the composed path's (semipd_rope, then the plain
    FP8 call, whose own write applies the same rule to the rotated k_new) bit for bit."""
    from test_gpu_fp8 import SHAPE, F8Rig
    cfg, rk = LLAMA31, dict(interleaved=inter)
    bs = SHAPE.block_size
    # decode
    ctx = [0, 15, 64, 700, 4097, 2048]
    case = synth.decode_case(SHAPE, ctx, 63, synth.NEEDLE)
    res = []
    for fused in (True, False):
        nb = [c // bs + 1 for c in ctx]
        rig = F8Rig(SHAPE, sum(nb) + 3, len(ctx) + 1, max(nb) + 1)
        rig.alloc(range(len(ctx)), nb)
        for b in range(len(ctx)):
            rig.put(0, b, case.k_ctx[b], case.v_ctx[b])
        dev = rig.dev
        q, k, v = (t.to(dev).contiguous() for t in (case.q, case.k_new, case.v_new))
        out = torch.empty(len(ctx), 32, 128, dtype=torch.bfloat16, device=dev)
        if fused:
            rig.pool.set_rope(cfg, **rk)
        else:
            rope_(q, k, rig.i32(ctx), cfg, **rk)
        rig.pool.decode_attn(0, q, k, v, rig.i32(range(len(ctx))), rig.i32(ctx), max(ctx),
                             SHAPE.softmax_scale, out,
                             rig.pool.new_decode_workspace(len(ctx), 32, max(ctx)), status=rig.status)
        torch.cuda.synchronize()
        assert int(rig.status.item()) == 0
        res.append((out, q, k, rig.host_pool(0)))
    (of, qf, kf, (Kf, Vf)), (oc, qc, kc, (Kc, Vc)) = res
    assert _bitwise(qf, qc) and _bitwise(kf, kc), "decode: rotated rows differ"
    assert np.array_equal(Kf, Kc) and np.array_equal(Vf, Vc), "decode: pool codes differ"
    assert _bitwise(of, oc), "decode: fused output differs from the composed path"
    # prefill (two requests with prefixes, one starting mid-page)
    chunks, prefixes = [130, 77], [64, 500]
    case = synth.prefill_case(SHAPE, chunks, prefixes, 64, synth.FLAT)
    cu = np.concatenate([[0], np.cumsum(chunks)]).astype(np.int32)
    pos = np.concatenate([np.arange(p, p + c) for c, p in zip(chunks, prefixes)]).astype(np.int32)
    res = []
    for fused in (True, False):
        nb = [(p + c + bs - 1) // bs for p, c in zip(prefixes, chunks)]
        rig = F8Rig(SHAPE, sum(nb) + 2, len(chunks) + 1, max(nb) + 1)
        rig.alloc(range(len(chunks)), nb)
        rig.pool.attach_fp8_prefill_scratch(len(chunks))
        for i in range(len(chunks)):
            rig.put(0, i, case.k_prefix[i], case.v_prefix[i])
        dev = rig.dev
        q, k, v = (t.to(dev).contiguous() for t in (case.q, case.k_new, case.v_new))
        T = sum(chunks)
        out = torch.empty(T, 32, 128, dtype=torch.bfloat16, device=dev)
        if fused:
            rig.pool.set_rope(cfg, **rk)
        else:
            rope_(q, k, torch.from_numpy(pos).to(dev), cfg, **rk)
        rig.pool.prefill_attn(0, q, k, v, rig.i32(cu), rig.i32(range(len(chunks))), rig.i32(prefixes),
                              T, max(chunks), SHAPE.softmax_scale, out, status=rig.status)
        torch.cuda.synchronize()
        assert int(rig.status.item()) == 0
        res.append((out, q, k, rig.host_pool(0)))
    (of, qf, kf, (Kf, Vf)), (oc, qc, kc, (Kc, Vc)) = res
    assert _bitwise(qf, qc) and _bitwise(kf, kc), "prefill: rotated rows differ"
    assert np.array_equal(Kf, Kc) and np.array_equal(Vf, Vc), "prefill: pool codes differ"
    assert _bitwise(of, oc), "prefill: fused output differs from the composed path"


def test_set_rope_validation_and_off():
    from paper_2504_19867_b200 import SemipdError
    shape = _shape(synth.CFG2_LLAMA8B, block_size=64)
    rig = Rig(shape, num_blocks=4, max_reqs=2, mbr=4)
    with pytest.raises(SemipdError):
        rig.pool.set_rope(LLAMA31, rot_offset=8, rot_dim=128)   # past the row
    with pytest.raises(SemipdError):
        rig.pool.set_rope(RopeConfig(theta=1.0))                 # theta <= 1
    rig.pool.set_rope(LLAMA31)
    rig.pool.set_rope(None)  # off again: the plain path is unchanged
