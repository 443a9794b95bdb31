"""Seeded synthetic input generators shared by tests/, bench.py and smoke().

This module holds NONE of the method's arithmetic: it only draws random
tensors, picks sizes and builds request layouts.  Both the CUDA path and the
oracle consume what it produces; neither is imported here.

Value distributions:
  0 flat    q, k, v ~ N(0, 1)
  1 peaked  q ~ N(0, 1) * 4      (score std ~ 4 at d = 128 with scale 1/sqrt(d))
  2 needle  1% of key positions (seeded) get k = 3*sqrt(d) * q_hat, q_hat the unit
            query of the first q-head of the group (decode) / the chunk's last row
            (prefill): scores ~ 30+ placed anywhere, stressing online-max rescale
  3 vshift  v ~ N(1, 1)          (makes the 2e-2 absolute bound meaningful)

Shapes follow BASELINE.json configs (Llama-3-8B / 70B attention, long-context
mix, DeepSeek-V2-Lite MLA latent).  Seeds: 1000 + 10*cfg_id + dist_id.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

FLAT, PEAKED, NEEDLE, VSHIFT = 0, 1, 2, 3
DISTS = (FLAT, PEAKED, NEEDLE, VSHIFT)


@dataclass
class AttnShape:
    """Attention shapes of one config (per rank for TP)."""
    name: str
    num_q_heads: int
    num_kv_heads: int
    head_dim_k: int
    head_dim_v: int
    block_size: int
    dtype: torch.dtype
    num_layers: int = 1
    kv_shared: bool = False  # MLA latent: V aliases K[..., :head_dim_v]
    scale: float | None = None

    @property
    def softmax_scale(self) -> float:
        return self.scale if self.scale is not None else 1.0 / math.sqrt(self.head_dim_k)


# BASELINE.json configs
CFG1_TINY = AttnShape("tiny-fp32", 4, 2, 64, 64, 16, torch.float32)
CFG2_LLAMA8B = AttnShape("llama3-8b", 32, 8, 128, 128, 16, torch.bfloat16, num_layers=32)
CFG3_LLAMA70B = AttnShape("llama3-70b", 64, 8, 128, 128, 16, torch.bfloat16, num_layers=80)
CFG5_MLA = AttnShape("deepseek-v2-lite-mla", 16, 1, 576, 512, 64, torch.bfloat16,
                     num_layers=27, kv_shared=True, scale=1.0 / math.sqrt(192.0))


def shard_heads(shape: AttnShape, tp: int) -> AttnShape:
    """TP by KV head: a rank holds Hkv/tp KV heads and Hq/tp q heads."""
    assert shape.num_kv_heads % tp == 0 and shape.num_q_heads % tp == 0
    return AttnShape(f"{shape.name}/tp{tp}", shape.num_q_heads // tp, shape.num_kv_heads // tp,
                     shape.head_dim_k, shape.head_dim_v, shape.block_size, shape.dtype,
                     shape.num_layers, shape.kv_shared, shape.scale)


def gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def randn(shape, g: torch.Generator, dtype: torch.dtype, mean: float = 0.0,
          std: float = 1.0) -> torch.Tensor:
    x = torch.randn(shape, generator=g, dtype=torch.float32)
    if std != 1.0:
        x = x * std
    if mean != 0.0:
        x = x + mean
    return x.to(dtype)


def qkv_tokens(n_tok: int, shape: AttnShape, g: torch.Generator, dist: int):
    """q [n, Hq, dk], k [n, Hkv, dk], v [n, Hkv, dv] (v is None for kv_shared)."""
    q = randn((n_tok, shape.num_q_heads, shape.head_dim_k), g, shape.dtype,
              std=4.0 if dist == PEAKED else 1.0)
    k = randn((n_tok, shape.num_kv_heads, shape.head_dim_k), g, shape.dtype)
    v = None
    if not shape.kv_shared:
        v = randn((n_tok, shape.num_kv_heads, shape.head_dim_v), g, shape.dtype,
                  mean=1.0 if dist == VSHIFT else 0.0)
    return q, k, v


def plant_needles(k: torch.Tensor, qhat_per_kv: torch.Tensor, g: torch.Generator,
                  frac: float = 0.01, gain: float = 3.0) -> torch.Tensor:
    """Set `frac` of key positions (seeded) to gain*sqrt(d)*q_hat for each kv head.
    k [n, Hkv, dk]; qhat_per_kv [Hkv, dk] (unit vectors, fp32).  gain = 3 for separate V;
    for the MLA latent cache (V aliases K) gain = 1 keeps the needle's value elements at
    unit scale (with gain 3 |o| reaches ~12, where bf16 output rounding alone exceeds the
    2e-2 absolute bound; R17) while its score still dominates (~40)."""
    n, hkv, d = k.shape
    cnt = max(1, int(round(frac * n)))
    pos = torch.randperm(n, generator=g)[:cnt]
    needle = (gain * math.sqrt(d) * qhat_per_kv).to(k.dtype)
    k = k.clone()
    k[pos] = needle.unsqueeze(0).expand(cnt, hkv, d)
    return k


def unit(x: torch.Tensor) -> torch.Tensor:
    x = x.float()
    return x / x.norm(dim=-1, keepdim=True).clamp_min(1e-12)


@dataclass
class DecodeCase:
    shape: AttnShape
    ctx_lens: list[int]
    req_ids: list[int]
    q: torch.Tensor          # [B, Hq, dk]
    k_new: torch.Tensor      # [B, Hkv, dk]
    v_new: torch.Tensor | None
    k_ctx: list[torch.Tensor] = field(default_factory=list)   # per request [ctx, Hkv, dk]
    v_ctx: list[torch.Tensor | None] = field(default_factory=list)


def decode_case(shape: AttnShape, ctx_lens, seed: int, dist: int = FLAT,
                req_ids=None) -> DecodeCase:
    """A decode step: per-request cached context K/V (to be scattered into the pool
    by the harness) plus the step's q, k_new, v_new."""
    g = gen(seed)
    B = len(ctx_lens)
    q, k_new, v_new = qkv_tokens(B, shape, g, dist)
    G = shape.num_q_heads // shape.num_kv_heads
    k_ctx, v_ctx = [], []
    for b, c in enumerate(ctx_lens):
        _, kc, vc = qkv_tokens(c, shape, g, dist)
        if dist == NEEDLE and c > 0:
            qhat = unit(q[b, ::G, :])  # first q head of each kv group
            kc = plant_needles(kc, qhat, g, gain=1.0 if shape.kv_shared else 3.0)
        k_ctx.append(kc)
        v_ctx.append(vc)
    return DecodeCase(shape, list(ctx_lens), list(req_ids if req_ids is not None else range(B)),
                      q, k_new, v_new, k_ctx, v_ctx)


@dataclass
class PrefillCase:
    shape: AttnShape
    chunk_lens: list[int]
    prefix_lens: list[int]
    req_ids: list[int]
    q: torch.Tensor          # [T, Hq, dk]
    k_new: torch.Tensor      # [T, Hkv, dk]
    v_new: torch.Tensor | None
    k_prefix: list[torch.Tensor] = field(default_factory=list)
    v_prefix: list[torch.Tensor | None] = field(default_factory=list)

    @property
    def cu_seqlens(self) -> list[int]:
        cu = [0]
        for c in self.chunk_lens:
            cu.append(cu[-1] + c)
        return cu


def prefill_case(shape: AttnShape, chunk_lens, prefix_lens, seed: int, dist: int = FLAT,
                 req_ids=None) -> PrefillCase:
    g = gen(seed)
    T = int(sum(chunk_lens))
    q, k_new, v_new = qkv_tokens(T, shape, g, dist)
    G = shape.num_q_heads // shape.num_kv_heads
    kp, vp = [], []
    cu = 0
    for i, (c, p) in enumerate(zip(chunk_lens, prefix_lens)):
        _, k_pre, v_pre = qkv_tokens(p, shape, g, dist)
        if dist == NEEDLE and c > 0:
            qhat = unit(q[cu + c - 1, ::G, :])  # chunk's last row
            gain = 1.0 if shape.kv_shared else 3.0
            if p > 0:
                k_pre = plant_needles(k_pre, qhat, g, gain=gain)
            k_new[cu:cu + c] = plant_needles(k_new[cu:cu + c], qhat, g, gain=gain)
        kp.append(k_pre)
        vp.append(v_pre)
        cu += c
    return PrefillCase(shape, list(chunk_lens), list(prefix_lens),
                       list(req_ids if req_ids is not None else range(len(chunk_lens))),
                       q, k_new, v_new, kp, vp)


def sharegpt_pack(total_tokens: int, seed: int, mean: float = 251.0, sigma: float = 1.0,
                  lo: int = 1, hi: int = 8192) -> list[int]:
    """Varlen chunk lengths, lognormal with the ShareGPT mean input 251,
    filling exactly total_tokens (the last length is truncated)."""
    rng = np.random.default_rng(seed)
    mu = math.log(mean) - sigma * sigma / 2.0
    out, s = [], 0
    while s < total_tokens:
        n = int(np.clip(round(rng.lognormal(mu, sigma)), lo, hi))
        n = min(n, total_tokens - s)
        out.append(n)
        s += n
    return out


def uniform_ctx(batch: int, lo: int, hi: int, seed: int) -> list[int]:
    rng = np.random.default_rng(seed)
    return [int(x) for x in rng.integers(lo, hi + 1, size=batch)]


def bits(t: torch.Tensor) -> np.ndarray:
    """Storage bits of a CPU tensor as numpy (bf16 -> uint16, fp32 -> float32)."""
    t = t.contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    if t.dtype == torch.float32:
        return t.numpy()
    raise TypeError(t.dtype)


@dataclass
class TraceRequest:
    rid: int
    arrival_iter: int
    input_len: int
    output_len: int


def mla_trace(n_req: int = 2000, lam: float = 3.0, seed: int = 5) -> list[TraceRequest]:
    """cfg-5 synthetic trace: Poisson(lam) arrivals per decode
    iteration; lognormal input (mean 251, clamp [1, 8192]) and output (mean 200,
    clamp [1, 2048]) lengths, sigma 1."""
    rng = np.random.default_rng(seed)
    reqs, it, rid = [], 0, 0
    mu_in, mu_out = math.log(251.0) - 0.5, math.log(200.0) - 0.5
    while rid < n_req:
        k = int(rng.poisson(lam))
        for _ in range(k):
            if rid >= n_req:
                break
            il = int(np.clip(round(rng.lognormal(mu_in, 1.0)), 1, 8192))
            ol = int(np.clip(round(rng.lognormal(mu_out, 1.0)), 1, 2048))
            reqs.append(TraceRequest(rid, it, il, ol))
            rid += 1
        it += 1
    return reqs


@dataclass
class MlaExpandedCase:
    """Inputs of an expanded-form MLA prefill call (R32): per
    request the whole latent history lat[i] [P_i + C_i, 576] (rows < P_i are cached, rows >= P_i
    are the call's kv_new), q [T, H, 192], up-projections w_uk / w_uv [H, 128, 512]."""
    q: torch.Tensor
    kv_new: torch.Tensor
    lat: list
    w_uk: torch.Tensor
    w_uv: torch.Tensor
    cu: list
    scale: float


def mla_expanded_case(chunk_lens, prefix_lens, seed: int, num_heads: int = 16, dist: int = FLAT,
                      dn: int = 128, dr: int = 64, dc: int = 512, dv: int = 128) -> MlaExpandedCase:
    """DeepSeek-V2-Lite shapes (16 heads, q_nope 128 | q_pe 64, latent 512 + rope 64, v 128).
    Latent rows ~ N(0, 1) (VSHIFT: N(1, 1), so V has a non-zero mean), q ~ N(0, 1) (PEAKED:
    N(0, 16)), W ~ N(0, 1/dc) so projected K / V are ~unit scale.  NEEDLE: 1 % of each
    request's keys are exact copies of its last key's latent row (repeated keys, a
    degenerate case of the softmax)."""
    g = gen(seed)
    lat = []
    for p, c in zip(prefix_lens, chunk_lens):
        x = randn((p + c, dc + dr), g, torch.bfloat16, mean=1.0 if dist == VSHIFT else 0.0)
        if dist == NEEDLE and p + c > 1:
            cnt = max(1, (p + c) // 100)
            pos = torch.randperm(p + c - 1, generator=g)[:cnt]
            x[pos] = x[-1].clone()
        lat.append(x)
    T = int(sum(chunk_lens))
    q = randn((T, num_heads, dn + dr), g, torch.bfloat16, std=4.0 if dist == PEAKED else 1.0)
    w_uk = randn((num_heads, dn, dc), g, torch.bfloat16, std=1.0 / math.sqrt(dc))
    w_uv = randn((num_heads, dv, dc), g, torch.bfloat16, std=1.0 / math.sqrt(dc))
    kv_new = torch.cat([x[p:] for x, p in zip(lat, prefix_lens)]) if T else torch.zeros(0, dc + dr, dtype=torch.bfloat16)
    cu = [0]
    for c in chunk_lens:
        cu.append(cu[-1] + int(c))
    return MlaExpandedCase(q, kv_new, lat, w_uk, w_uv, cu, 1.0 / math.sqrt(dn + dr))
