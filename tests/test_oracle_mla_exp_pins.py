"""Pins for the oracle's expanded-form MLA prefill (CPU only; SURVEY §8(f) N4, S19,
DESIGN.md reading R32).

  * round_bf16 (the one rounding the form adds: the projected K / V are bf16 activations)
    against torch's float32 -> bfloat16 conversion on fp32-exact inputs, and on exact ties;
  * one-hot up-projections make every projected element an exact copy of a latent coordinate,
    so the expanded prefill must equal plain causal MHA (the pinned attention_contig) over the
    K / V assembled by hand from the latent rows;
  * random up-projections against torch fp64 SDPA over torch-projected K / V (bf16-rounded
    through float32: agreement to the bf16 double-rounding bound);
  * chunked == unchunked, and the chunk's latent rows land in the pool bit for bit.
"""
import math

import numpy as np
import torch

import oracle
import synth

H, DN, DR, DV, DC, BS = 4, 16, 8, 12, 32, 16   # small MLA-shaped case (cfg 5: 16, 128, 64, 128, 512, 64)


def bf(x: torch.Tensor) -> np.ndarray:
    return synth.bits(x.to(torch.bfloat16))


def _case(seed, chunks, prefix, w_kind="random"):
    g = synth.gen(seed)
    n = len(chunks)
    T = sum(chunks)
    nk = [p + c for p, c in zip(prefix, chunks)]
    MBR = max(-(-k // BS) for k in nk) + 1
    N_B = n * MBR
    bt = np.arange(N_B, dtype=np.int32).reshape(n, MBR)
    np.random.default_rng(seed).shuffle(bt.reshape(-1))
    lat_all = [synth.randn((k, DC + DR), g, torch.bfloat16) for k in nk]
    pool = np.zeros((N_B, 1, BS, DC + DR), np.uint16)
    kv_new = []
    for i in range(n):  # prefix rows cached by earlier chunks; chunk rows are the call's input
        for j in range(prefix[i]):
            pool[bt[i, j // BS], 0, j % BS] = bf(lat_all[i][j])
        kv_new.append(lat_all[i][prefix[i]:])
    kv_new = torch.cat(kv_new)
    q = synth.randn((T, H, DN + DR), g, torch.bfloat16)
    if w_kind == "onehot":
        sel_k = torch.randint(0, DC, (H, DN), generator=g)
        sel_v = torch.randint(0, DC, (H, DV), generator=g)
        w_uk = torch.nn.functional.one_hot(sel_k, DC).to(torch.bfloat16)
        w_uv = torch.nn.functional.one_hot(sel_v, DC).to(torch.bfloat16)
    else:
        w_uk = synth.randn((H, DN, DC), g, torch.bfloat16) / math.sqrt(DC)
        w_uv = synth.randn((H, DV, DC), g, torch.bfloat16) / math.sqrt(DC)
        sel_k = sel_v = None
    cu = np.concatenate([[0], np.cumsum(chunks)]).astype(np.int32)
    return dict(q=q, kv_new=kv_new, lat_all=lat_all, pool=pool, bt=bt, cu=cu, n=n,
                w_uk=w_uk.to(torch.bfloat16), w_uv=w_uv.to(torch.bfloat16), sel_k=sel_k, sel_v=sel_v)


def _run(c, prefix, scale, pool=None):
    pool = c["pool"].copy() if pool is None else pool
    out = oracle.prefill_mla_expanded(bf(c["q"]), bf(c["kv_new"]), pool, c["bt"], c["cu"],
                                      np.arange(c["n"]), prefix, bf(c["w_uk"]), bf(c["w_uv"]),
                                      scale, dn=DN, dr=DR)
    return out, pool


def test_round_bf16_matches_torch_on_fp32_inputs_and_ties():
    rng = np.random.default_rng(3)
    x = (rng.standard_normal(3000) * 10.0 ** rng.uniform(-30, 30, 3000)).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).double().numpy()
    ours = np.array([oracle.round_bf16(float(v)) for v in x])
    np.testing.assert_array_equal(ours, ref)
    for m in range(1, 128):  # exact ties between consecutive bf16 values in [1, 2): even wins
        tie = 1.0 + (2 * m - 1) * 2.0 ** -8
        lo, hi = 1.0 + (m - 1) * 2.0 ** -7, 1.0 + m * 2.0 ** -7
        assert oracle.round_bf16(tie) == (lo if (m - 1) % 2 == 0 else hi)


def test_onehot_projection_equals_plain_mha():
    chunks, prefix = [9, 20], [0, 37]
    c = _case(11, chunks, prefix, w_kind="onehot")
    scale = 1 / math.sqrt(DN + DR)
    out, _ = _run(c, prefix, scale)
    for i in range(c["n"]):
        lat = c["lat_all"][i]  # [nk, DC + DR] bf16
        K = torch.cat([lat[:, :DC][:, c["sel_k"]], lat[:, DC:].unsqueeze(1).expand(-1, H, DR)], -1)
        V = lat[:, :DC][:, c["sel_v"]]
        rows = slice(int(c["cu"][i]), int(c["cu"][i + 1]))
        ref = oracle.attention_contig(bf(c["q"][rows]), bf(K), bf(V), prefix[i], scale)
        np.testing.assert_allclose(out[rows], ref, rtol=1e-13, atol=1e-13)


def test_random_projection_matches_torch_sdpa():
    chunks, prefix = [7, 16], [5, 40]
    c = _case(12, chunks, prefix)
    scale = 1 / math.sqrt(DN + DR)
    out, _ = _run(c, prefix, scale)
    for i in range(c["n"]):
        lat = c["lat_all"][i].double()
        kn = torch.einsum("hdc,jc->jhd", c["w_uk"].double(), lat[:, :DC]).float().to(torch.bfloat16).double()
        v = torch.einsum("hdc,jc->jhd", c["w_uv"].double(), lat[:, :DC]).float().to(torch.bfloat16).double()
        K = torch.cat([kn, lat[:, DC:].unsqueeze(1).expand(-1, H, DR)], -1)
        rows = slice(int(c["cu"][i]), int(c["cu"][i + 1]))
        q = c["q"][rows].double()
        C = q.shape[0]
        mask = torch.arange(K.shape[0]).unsqueeze(0) <= torch.arange(C).unsqueeze(1) + prefix[i]
        ref = torch.nn.functional.scaled_dot_product_attention(
            q.transpose(0, 1), K.transpose(0, 1), v.transpose(0, 1), attn_mask=mask, scale=scale)
        np.testing.assert_allclose(out[rows], ref.transpose(0, 1).numpy(), rtol=2e-3, atol=2e-3)


def test_chunked_equals_unchunked_and_pool_rows_written():
    c = _case(13, [30], [0])
    scale = 0.2
    full, pool = _run(c, [0], scale)
    # the chunk's latent rows are in the pool, bit for bit
    for j in range(30):
        assert np.array_equal(pool[c["bt"][0, j // BS], 0, j % BS], bf(c["kv_new"][j]))
    # the same 30 tokens as two chunks: 12 at P = 0, then 18 at P = 12
    c1 = dict(c, cu=np.array([0, 12], np.int32), q=c["q"][:12], kv_new=c["kv_new"][:12])
    o1, pool1 = _run(c1, [0], scale)
    c2 = dict(c, cu=np.array([0, 18], np.int32), q=c["q"][12:], kv_new=c["kv_new"][12:])
    o2, _ = _run(c2, [12], scale, pool=pool1)
    np.testing.assert_allclose(np.concatenate([o1, o2]), full, rtol=1e-13, atol=1e-13)
