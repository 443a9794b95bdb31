"""Pins of the oracle's RoPE (oracle.rope / oracle.rope_inv_freq, PAPER
P:355 §6, DESIGN reading R27) against what mathematics fixes, not against a retyped formula:
a 2-D rotation in closed form, complex multiplication (an independent formulation of the
half-split pairs), norm preservation, the relative-position property of the dot product,
the geometric frequency ladder, and the shape of the Llama-3.1 rescaling (kept / stretched
bands, affine in 1/wavelength between them)."""
import math

import numpy as np
import pytest

import oracle

LLAMA31 = dict(theta=500000.0, factor=8.0, lf=1.0, hf=4.0, L0=8192.0)


def _x(T, H, d, seed):
    return np.random.default_rng(seed).standard_normal((T, H, d)).astype(np.float32)


def test_d2_is_the_rotation_matrix():
    x = np.array([[[1.0, 0.0]], [[0.0, 1.0]], [[0.5, -0.75]]], np.float32)
    for p in (0, 1, 7, 1000, 131071):
        out = oracle.rope(x, [p] * 3, theta=10000.0)
        c, s = math.cos(p), math.sin(p)  # f_0 = theta^0 = 1
        np.testing.assert_allclose(out[0, 0], [c, s], atol=1e-12)
        np.testing.assert_allclose(out[1, 0], [-s, c], atol=1e-12)
        np.testing.assert_allclose(out[2, 0], [0.5 * c + 0.75 * s, -0.75 * c + 0.5 * s], atol=1e-12)


def test_position_zero_is_identity():
    x = _x(3, 4, 64, 1)
    out = oracle.rope(x, [0, 0, 0], **LLAMA31)
    assert np.array_equal(out, x.astype(np.float64))


@pytest.mark.parametrize("cfg", [dict(theta=10000.0), LLAMA31])
def test_equals_complex_multiplication(cfg):
    T, H, d = 5, 3, 128
    x = _x(T, H, d, 2)
    pos = np.array([0, 1, 17, 4095, 100000])
    out = oracle.rope(x, pos, **cfg)
    f = oracle.rope_inv_freq(d, **cfg)
    z = x[..., : d // 2].astype(np.float64) + 1j * x[..., d // 2:].astype(np.float64)
    zr = z * np.exp(1j * pos[:, None, None] * f[None, None, :])
    np.testing.assert_allclose(out[..., : d // 2], zr.real, rtol=0, atol=1e-9)
    np.testing.assert_allclose(out[..., d // 2:], zr.imag, rtol=0, atol=1e-9)


def test_pair_norms_preserved():
    x = _x(4, 2, 64, 3)
    out = oracle.rope(x, [3, 99, 5000, 70000], **LLAMA31)
    n0 = x[..., :32].astype(np.float64) ** 2 + x[..., 32:].astype(np.float64) ** 2
    n1 = out[..., :32] ** 2 + out[..., 32:] ** 2
    np.testing.assert_allclose(n1, n0, rtol=1e-12)


@pytest.mark.parametrize("cfg", [dict(theta=10000.0), LLAMA31])
def test_dot_product_depends_only_on_relative_position(cfg):
    d = 128
    q, k = _x(1, 2, d, 4), _x(1, 2, d, 5)
    for m, n, c in [(10, 3, 0), (5000, 4000, 17), (2, 9, 30)]:
        a = (oracle.rope(q, [m], **cfg) * oracle.rope(k, [n], **cfg)).sum(-1)
        b = (oracle.rope(q, [m - n + c], **cfg) * oracle.rope(k, [c], **cfg)).sum(-1)
        np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-9)


def test_plain_frequencies_form_a_geometric_ladder():
    d, theta = 128, 10000.0
    f = oracle.rope_inv_freq(d, theta)
    assert f[0] == 1.0
    np.testing.assert_allclose(f[:-1] / f[1:], theta ** (2.0 / d), rtol=1e-12)
    # the lowest frequency closes the ladder: f_{d/2-1} = theta^(-(d-2)/d)
    np.testing.assert_allclose(f[-1], theta ** (-(d - 2) / d), rtol=1e-12)


def test_llama31_rescaling_shape():
    d = 128
    f0 = oracle.rope_inv_freq(d, 500000.0)
    f = oracle.rope_inv_freq(d, **LLAMA31)
    r = f / f0
    w = 2 * math.pi / f0
    hi = w < 8192.0 / 4.0
    lo = w > 8192.0 / 1.0
    mid = ~hi & ~lo
    assert hi.sum() > 0 and lo.sum() > 0 and mid.sum() >= 3
    np.testing.assert_array_equal(r[hi], 1.0)
    np.testing.assert_allclose(r[lo], 1.0 / 8.0, rtol=1e-15)
    assert np.all(np.diff(r) <= 1e-15)  # stretching grows monotonically toward low frequency
    assert np.all((r[mid] > 1 / 8) & (r[mid] < 1))
    # between the bands the ratio is affine in 1 / wavelength, reaching 1 at w = L0/hf and
    # 1/factor at w = L0/lf (continuity): fit on the band, extrapolate to both edges
    u = 1.0 / w[mid]
    A = np.vstack([u, np.ones_like(u)]).T
    coef, res, *_ = np.linalg.lstsq(A, r[mid], rcond=None)
    assert np.max(np.abs(A @ coef - r[mid])) < 1e-12
    np.testing.assert_allclose(coef[0] * (4.0 / 8192.0) + coef[1], 1.0, rtol=1e-9)
    np.testing.assert_allclose(coef[0] * (1.0 / 8192.0) + coef[1], 1.0 / 8.0, rtol=1e-9)


def test_interleaved_equals_complex_multiplication_on_adjacent_pairs():
    T, H, d = 4, 2, 64
    x = _x(T, H, d, 6)
    pos = np.array([0, 3, 900, 77777])
    out = oracle.rope(x, pos, theta=10000.0, interleaved=True)
    f = oracle.rope_inv_freq(d, 10000.0)
    z = x[..., 0::2].astype(np.float64) + 1j * x[..., 1::2].astype(np.float64)
    zr = z * np.exp(1j * pos[:, None, None] * f[None, None, :])
    np.testing.assert_allclose(out[..., 0::2], zr.real, rtol=0, atol=1e-9)
    np.testing.assert_allclose(out[..., 1::2], zr.imag, rtol=0, atol=1e-9)


@pytest.mark.parametrize("inter", [False, True])
def test_sub_range_rotates_only_its_columns(inter):
    """An MLA latent row: only the 64 rope columns at 512 rotate, exactly as a stand-alone
    64-wide rotation of those columns; the 512 latent columns pass through bit for bit."""
    x = _x(3, 2, 576, 7)
    pos = [5, 600, 40000]
    out = oracle.rope(x, pos, theta=10000.0, off=512, rd=64, interleaved=inter)
    assert np.array_equal(out[..., :512], x[..., :512].astype(np.float64))
    alone = oracle.rope(np.ascontiguousarray(x[..., 512:]), pos, theta=10000.0, interleaved=inter)
    np.testing.assert_array_equal(out[..., 512:], alone)
