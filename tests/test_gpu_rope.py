"""RoPE kernel (C ABI ``semipd_rope``, DESIGN R27) against
the fp64 oracle on the same seeded inputs, element by element.  Tolerances: north_star's
bf16 bar (max abs <= 2e-2, relative Frobenius <= 1e-2) and 1e-4 for fp32; the kernel forms
the angle in fp64, so even 128k-token positions stay at bf16 rounding."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2504_19867_b200 import RopeConfig, SemipdError, rope_

pytestmark = pytest.mark.gpu

LLAMA31 = RopeConfig()
PLAIN = RopeConfig(theta=10000.0, factor=0.0)


def _ocfg(c: RopeConfig):
    return dict(theta=c.theta, factor=c.factor, lf=c.low_freq_factor, hf=c.high_freq_factor,
                L0=float(c.original_max_pos))


def _check(T, Hq, Hkv, d, dtype, cfg, pos, seed):
    g = torch.Generator().manual_seed(seed)
    q = torch.randn(T, Hq, d, generator=g).to(dtype)
    k = torch.randn(T, Hkv, d, generator=g).to(dtype)
    bits = (lambda t: synth.bits(t)) if dtype == torch.bfloat16 else (lambda t: t.numpy())
    ref_q = oracle.rope(bits(q), pos, **_ocfg(cfg))
    ref_k = oracle.rope(bits(k), pos, **_ocfg(cfg))
    dev = torch.device("cuda", 0)
    qd, kd = q.to(dev), k.to(dev)
    rope_(qd, kd, torch.tensor(pos, dtype=torch.int32, device=dev), cfg)
    torch.cuda.synchronize()
    for got, ref in ((qd, ref_q), (kd, ref_k)):
        got = got.cpu().double().numpy()
        err = np.abs(got - ref).max()
        rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
        if dtype == torch.bfloat16:
            assert err <= 2e-2 and rel <= 1e-2, (err, rel)
        else:
            assert err <= 1e-4 and rel <= 1e-4, (err, rel)


@pytest.mark.parametrize("cfg", [LLAMA31, PLAIN], ids=["llama31", "plain"])
def test_rope_cfg2_chunk_bf16(cfg):
    # a 2k prefill chunk at cfg-2 shapes, positions continuing a 6k prefix
    T = 2048
    _check(T, 32, 8, 128, torch.bfloat16, cfg, list(range(6144, 6144 + T)), 11)


def test_rope_long_positions_and_ragged_tokens_bf16():
    # decode-style rows at scattered long-context positions (up to 128k), 37 tokens
    pos = list(np.random.default_rng(3).integers(0, 131072, 37))
    _check(37, 64, 8, 128, torch.bfloat16, LLAMA31, pos, 12)


def test_rope_fp32_head_dim_64():
    _check(129, 4, 2, 64, torch.float32, PLAIN, list(range(129)), 13)


def test_rope_mla_rope_dim_bf16():
    # DeepSeek-style rope part: d = 64, one shared kv head
    _check(100, 16, 1, 64, torch.bfloat16, RopeConfig(theta=10000.0, factor=0.0),
           list(range(500, 600)), 14)


def test_rope_edge_cases():
    dev = torch.device("cuda", 0)
    q = torch.zeros(0, 4, 128, dtype=torch.bfloat16, device=dev)
    rope_(q, None, torch.zeros(0, dtype=torch.int32, device=dev))  # empty: no-op
    # position 0 leaves the rows bit-identical
    x = torch.randn(5, 4, 128, device=dev).to(torch.bfloat16)
    y = x.clone()
    rope_(y, None, torch.zeros(5, dtype=torch.int32, device=dev))
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    # head_dim / 2 not a multiple of the 16-byte vector: refused, nothing written
    z = torch.randn(3, 2, 72, device=dev).to(torch.bfloat16)
    with pytest.raises(SemipdError):
        rope_(z, None, torch.zeros(3, dtype=torch.int32, device=dev))


def test_rope_then_prefill_matches_oracle_chain():
    """The adjacent step composed with the path: semipd_rope on the chunk's q / k, then
    semipd_prefill_attn (which writes the rotated k into the pool) equals the oracle's
    attention over the oracle's rotated q / k (fp64 rotation, fed as fp32), within the bf16
    bar.  The pool must hold exactly the kernel's rotated k rows."""
    from harness import compare
    from paper_2504_19867_b200 import KVPool, PoolConfig
    dev = torch.device("cuda", 0)
    C, Hq, Hkv, d, bs = 300, 32, 8, 128, 64
    g = torch.Generator().manual_seed(21)
    q = torch.randn(C, Hq, d, generator=g).to(torch.bfloat16)
    k = torch.randn(C, Hkv, d, generator=g).to(torch.bfloat16)
    v = torch.randn(C, Hkv, d, generator=g).to(torch.bfloat16)
    pos = list(range(C))
    nb = -(-C // bs)
    pool = KVPool(PoolConfig(1, nb + 1, bs, Hkv, d, d, 1, nb), dev)
    i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
    pool.alloc_blocks(i32([0]), i32([nb]))
    qd, kd, vd = q.to(dev), k.to(dev), v.to(dev)
    rope_(qd, kd, i32(pos), LLAMA31)
    out = torch.empty(C, Hq, d, dtype=torch.bfloat16, device=dev)
    scale = 1.0 / np.sqrt(d)
    pool.prefill_attn(0, qd, kd, vd, i32([0, C]), i32([0]), i32([0]), C, C, scale, out)
    torch.cuda.synchronize()
    K, _, BT, _ = pool.views(0)
    bt = BT.cpu().numpy()
    # the pool holds the kernel's rotated k rows bit for bit (a3 after the rotation)
    posn = np.arange(C)
    pooled = K.cpu()[torch.from_numpy(bt[0][posn // bs]).long(), :, torch.from_numpy(posn % bs)]
    assert torch.equal(pooled.view(torch.int16), kd.cpu().view(torch.int16))
    qr = oracle.rope(synth.bits(q), pos, **_ocfg(LLAMA31)).astype(np.float32)
    kr = oracle.rope(synth.bits(k), pos, **_ocfg(LLAMA31)).astype(np.float32)
    kp = np.zeros((nb + 1, Hkv, bs, d), np.float32)
    vp = np.zeros_like(kp)
    ref = oracle.prefill(qr, kr, v.float().numpy(), kp, vp, bt, [0, C], [0], [0], scale)
    compare(out.float().cpu().double().numpy(), ref, torch.bfloat16, "rope + prefill")


@pytest.mark.parametrize("inter", [True, False], ids=["interleaved", "half_split"])
def test_rope_mla_latent_rows_sub_range(inter):
    """DeepSeek-V2-Lite MLA rows (cfg 5): q [T, 16, 576] and the latent k [T, 1, 576]; only
    the 64 decoupled-rope columns at 512 rotate (interleaved pairs, as DeepSeek lays them out);
    the 512 latent columns stay bit-identical."""
    dev = torch.device("cuda", 0)
    T = 129
    g = torch.Generator().manual_seed(15)
    q = torch.randn(T, 16, 576, generator=g).to(torch.bfloat16)
    k = torch.randn(T, 1, 576, generator=g).to(torch.bfloat16)
    pos = list(range(1000, 1000 + T))
    qd, kd = q.to(dev), k.to(dev)
    cfg = RopeConfig(theta=10000.0, factor=0.0)
    rope_(qd, kd, torch.tensor(pos, dtype=torch.int32, device=dev), cfg, rot_offset=512,
          rot_dim=64, interleaved=inter)
    torch.cuda.synchronize()
    for got, x in ((qd.cpu(), q), (kd.cpu(), k)):
        assert torch.equal(got[..., :512].view(torch.int16), x[..., :512].view(torch.int16))
        ref = oracle.rope(synth.bits(x), pos, **_ocfg(cfg), off=512, rd=64, interleaved=inter)
        diff = np.abs(got.double().numpy() - ref)
        assert diff.max() <= 2e-2
        assert np.linalg.norm(got.double().numpy() - ref) / np.linalg.norm(ref) <= 1e-2
