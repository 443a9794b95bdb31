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
