"""Pins for the oracle's FP8 (E4M3) KV-page functions (CPU only, -m "not gpu").

DESIGN.md reading R31 (the paper, names FP8 and nothing more): pages hold OCP E4M3
codes, written as E4M3_rne_satfinite(fl32(x / s)) and read as s * value(code); a prefill
chunk's own keys enter attention at input precision, cached keys through the pool.

Pinned against things other than the oracle itself:
  * the OCP OFP8 specification's E4M3 table (tests/golden/e4m3_values.txt, cited there);
  * an independent library routine: torch.float8_e4m3fn (all 256 code values; RNE
    conversion of in-range fp32 values, ties included);
  * saturation / NaN / signed-zero special cases of the spec's "satfinite" rule;
  * reduction to the already-pinned bf16 oracle: when every K/V element is s * (an E4M3
    value) with s a power of two, quantisation is exact and decode_fp8 / prefill_fp8 must
    equal decode / prefill on the dequantised bf16 pool;
  * a chunk with no prefix reads no pool element, so prefill_fp8 must equal the contiguous
    causal attention of its own bf16 rows.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth

HERE = os.path.dirname(os.path.abspath(__file__))
F8 = torch.float8_e4m3fn


def torch_values(codes: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(codes, dtype=np.uint8)).view(F8).to(torch.float64).numpy()


def torch_codes(x_f32: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x_f32, dtype=np.float32)).to(F8).view(torch.uint8).numpy()


def finite_codes():
    return np.array([c for c in range(256) if (c & 0x7F) != 0x7F], np.uint8)


# --------------------------------------------------------------------------- encoding
def test_e4m3_golden_values():
    n = 0
    with open(os.path.join(HERE, "golden", "e4m3_values.txt")) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            c, v = line.split()
            got = oracle.e4m3_value(int(c, 16))
            if v == "nan":
                assert math.isnan(got)
            else:
                assert got == float(v), (c, got, v)
            n += 1
    assert n >= 12


def test_e4m3_values_match_torch_all_codes():
    codes = np.arange(256, dtype=np.uint8)
    ours = oracle.e4m3_values(codes)
    ref = torch_values(codes)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan], ref[~nan])
    assert np.array_equal(np.signbit(ours[~nan]), np.signbit(ref[~nan]))  # -0 is 0x80


def test_e4m3_encode_matches_torch_in_range():
    rng = np.random.default_rng(31)
    mags = np.concatenate([rng.uniform(0, 448, 4000), 2.0 ** rng.uniform(-12, 8.8, 4000),
                           rng.uniform(0, 2 ** -6, 2000)]).astype(np.float32)
    mags = mags[mags <= 448]
    x = mags * np.where(rng.random(mags.size) < 0.5, -1, 1).astype(np.float32)
    ours = np.array([oracle.e4m3_encode(v) for v in x], np.uint8)
    assert np.array_equal(ours, torch_codes(x))


def test_e4m3_ties_round_to_even():
    # midpoints between consecutive finite non-negative values (exact in fp32)
    vals = torch_values(np.arange(0x7F, dtype=np.uint8))
    mids = ((vals[:-1] + vals[1:]) / 2).astype(np.float32)
    assert np.array_equal(mids.astype(np.float64), (vals[:-1] + vals[1:]) / 2)
    ours = np.array([oracle.e4m3_encode(v) for v in mids], np.uint8)
    assert np.array_equal(ours, torch_codes(mids))
    assert np.all(ours % 2 == 0)  # the even mantissa wins every tie
    neg = np.array([oracle.e4m3_encode(-v) for v in mids], np.uint8)
    assert np.array_equal(neg, ours | 0x80)


def test_e4m3_roundtrip_saturation_nan_zero():
    for c in finite_codes():
        assert oracle.e4m3_encode(oracle.e4m3_value(int(c))) == c
    for x in (448.0, 449.0, 463.9, 464.0, 480.0, 500.0, 1e30, float("inf")):
        assert oracle.e4m3_encode(x) == 0x7E, x        # satfinite
        assert oracle.e4m3_encode(-x) == 0xFE, x
    assert oracle.e4m3_encode(float("nan")) & 0x7F == 0x7F
    assert oracle.e4m3_encode(0.0) == 0x00 and oracle.e4m3_encode(-0.0) == 0x80
    assert oracle.e4m3_encode(2.0 ** -10) == 0x00      # tie between 0 and 2^-9 -> even (0)
    assert oracle.e4m3_encode(2.0 ** -10 * 1.01) == 0x01


def test_e4m3_encode_monotone():
    x = np.sort(np.random.default_rng(5).uniform(-600, 600, 3000).astype(np.float32))
    v = oracle.e4m3_values(np.array([oracle.e4m3_encode(t) for t in x], np.uint8))
    assert np.all(np.diff(v) >= 0)


def test_quantize_divides_in_fp32():
    g = synth.gen(77)
    x = synth.randn((4096,), g, torch.bfloat16) * 3
    for s in (0.0173, 0.5, 1.0, 3.3):
        xf = x.float() / torch.tensor(s, dtype=torch.float32)  # IEEE fp32 division
        keep = xf.abs() <= 448
        ours = oracle.e4m3_quantize(synth.bits(x), s)
        ref = torch_codes(xf.numpy())
        assert np.array_equal(ours[keep.numpy()], ref[keep.numpy()])
        assert np.all(ours[~keep.numpy()] & 0x7F == 0x7E)  # saturated, sign kept


# --------------------------------------------------------------------------- attention
def _repr_rows(g_np, n, H, d, s):
    """bf16 rows whose elements are s * (an E4M3 value), s a power of two: quantisation at
    scale s is exact, so the codes are known without the encoder."""
    codes = g_np.choice(finite_codes(), size=(n, H, d)).astype(np.uint8)
    vals = torch_values(codes) * s
    bf = torch.from_numpy(vals).to(torch.bfloat16)
    assert np.array_equal(bf.double().numpy(), vals)
    return codes, synth.bits(bf)


def _bf16_pool_of(codes, s):
    return synth.bits(torch.from_numpy(torch_values(codes) * s).to(torch.bfloat16))


@pytest.mark.parametrize("ctx", [[0, 5, 63, 64, 130], [200]])
def test_decode_fp8_reduces_to_bf16_oracle(ctx):
    rng = np.random.default_rng(11)
    Hq, Hkv, d, bs, MBR = 8, 2, 32, 16, 16
    ks, vs = 2.0 ** -4, 2.0 ** -2
    B = len(ctx)
    N_B = B * MBR
    bt = np.arange(N_B, dtype=np.int32).reshape(B, MBR)
    rng.shuffle(bt.reshape(-1))
    kc = rng.choice(finite_codes(), size=(N_B, Hkv, bs, d)).astype(np.uint8)
    vc = rng.choice(finite_codes(), size=(N_B, Hkv, bs, d)).astype(np.uint8)
    k_new_c, k_new = _repr_rows(rng, B, Hkv, d, ks)
    v_new_c, v_new = _repr_rows(rng, B, Hkv, d, vs)
    q = synth.bits(synth.randn((B, Hq, d), synth.gen(3), torch.bfloat16))
    scale = 1 / math.sqrt(d)
    kp8, vp8 = kc.copy(), vc.copy()
    out8 = oracle.decode_fp8(q, k_new, v_new, kp8, vp8, bt, np.arange(B), ctx, scale, ks, vs)
    kpb, vpb = _bf16_pool_of(kc, ks), _bf16_pool_of(vc, vs)
    outb = oracle.decode(q, k_new, v_new, kpb, vpb, bt, np.arange(B), ctx, scale)
    np.testing.assert_array_equal(out8, outb)
    for b, c in enumerate(ctx):  # the append stored the exact codes
        blk = bt[b, c // bs]
        assert np.array_equal(kp8[blk, :, c % bs], k_new_c[b])
        assert np.array_equal(vp8[blk, :, c % bs], v_new_c[b])


def test_decode_fp8_append_codes_match_torch():
    Hq, Hkv, d, bs = 4, 2, 64, 16
    g = synth.gen(19)
    k_new = synth.randn((3, Hkv, d), g, torch.bfloat16)
    v_new = synth.randn((3, Hkv, d), g, torch.bfloat16)
    q = synth.randn((3, Hq, d), g, torch.bfloat16)
    ks, vs = 0.037, 0.011
    kp = np.zeros((8, Hkv, bs, d), np.uint8)
    vp = np.zeros_like(kp)
    bt = np.array([[0, 1], [2, 3], [4, 5]], np.int32)
    ctx = [3, 16, 31]
    oracle.decode_fp8(synth.bits(q), synth.bits(k_new), synth.bits(v_new), kp, vp, bt,
                      np.arange(3), ctx, 0.125, ks, vs)
    for b, c in enumerate(ctx):
        blk = bt[b, c // bs]
        kf = (k_new[b].float() / torch.tensor(ks)).numpy()
        vf = (v_new[b].float() / torch.tensor(vs)).numpy()
        assert np.array_equal(kp[blk, :, c % bs], torch_codes(kf))
        assert np.array_equal(vp[blk, :, c % bs], torch_codes(vf))


def test_prefill_fp8_reduces_to_bf16_oracle():
    rng = np.random.default_rng(23)
    Hq, Hkv, d, bs, MBR = 4, 2, 32, 16, 8
    ks, vs = 2.0 ** -3, 2.0 ** -5
    chunks, prefix = [7, 20, 1], [0, 33, 16]
    n = len(chunks)
    T = sum(chunks)
    cu = np.concatenate([[0], np.cumsum(chunks)]).astype(np.int32)
    N_B = n * MBR
    bt = np.arange(N_B, dtype=np.int32).reshape(n, MBR)
    rng.shuffle(bt.reshape(-1))
    kc = rng.choice(finite_codes(), size=(N_B, Hkv, bs, d)).astype(np.uint8)
    vc = rng.choice(finite_codes(), size=(N_B, Hkv, bs, d)).astype(np.uint8)
    _, k_new = _repr_rows(rng, T, Hkv, d, ks)
    _, v_new = _repr_rows(rng, T, Hkv, d, vs)
    q = synth.bits(synth.randn((T, Hq, d), synth.gen(4), torch.bfloat16))
    scale = 1 / math.sqrt(d)
    kp8, vp8 = kc.copy(), vc.copy()
    out8 = oracle.prefill_fp8(q, k_new, v_new, kp8, vp8, bt, cu, np.arange(n), prefix, scale, ks, vs)
    kpb, vpb = _bf16_pool_of(kc, ks), _bf16_pool_of(vc, vs)
    outb = oracle.prefill(q, k_new, v_new, kpb, vpb, bt, cu, np.arange(n), prefix, scale)
    np.testing.assert_array_equal(out8, outb)
    # the chunk write left exactly the dequantised-pool image the bf16 oracle wrote
    np.testing.assert_array_equal(_bf16_pool_of(kp8, ks), kpb)
    np.testing.assert_array_equal(_bf16_pool_of(vp8, vs), vpb)


def test_prefill_fp8_chunk_reads_input_precision():
    # no prefix: no pool element is read, whatever the scale, so the result is the plain
    # causal attention of the chunk's own bf16 rows (not representable in E4M3)
    g = synth.gen(29)
    Hq, Hkv, d, T = 8, 2, 64, 40
    q = synth.randn((T, Hq, d), g, torch.bfloat16)
    k = synth.randn((T, Hkv, d), g, torch.bfloat16)
    v = synth.randn((T, Hkv, d), g, torch.bfloat16)
    kp = np.zeros((4, Hkv, 16, d), np.uint8)
    vp = np.zeros_like(kp)
    bt = np.array([[2, 0, 3, 1]], np.int32)
    out8 = oracle.prefill_fp8(synth.bits(q), synth.bits(k), synth.bits(v), kp, vp, bt, [0, T], [0],
                              [0], 0.125, 0.3, 0.7)
    ref = oracle.attention_contig(synth.bits(q), synth.bits(k), synth.bits(v), 0, 0.125)
    np.testing.assert_allclose(out8, ref, rtol=1e-13, atol=1e-13)
    assert np.any(kp != 0)  # the write still happened


def test_fp8_bad_block_and_invalid_scale():
    q = np.zeros((1, 2, 16), np.uint16)
    kn = np.zeros((1, 1, 16), np.uint16)
    kp = np.zeros((2, 1, 16, 16), np.uint8)
    with pytest.raises(ValueError, match="status 5"):
        oracle.decode_fp8(q, kn, kn, kp, kp.copy(), np.array([[-1]], np.int32), [0], [3], 1.0, 1.0, 1.0)
    with pytest.raises(ValueError, match="status 1"):
        oracle.decode_fp8(q, kn, kn, kp, kp.copy(), np.array([[0]], np.int32), [0], [3], 1.0, 0.0, 1.0)
