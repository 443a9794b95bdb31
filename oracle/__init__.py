"""fp64 CPU oracle for the semi-PD co-run attention hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2504_19867_b200`` (neither imports the
other).  The arithmetic lives in ``semipd_oracle.c`` (plain C, fp64); this file
only marshals numpy arrays into it.  See that file's header for the passages
each function follows (§2.1, §4.2, §4.4, §6).

Parity pins: ``tests/test_oracle_pins.py`` (brute force, torch fp64 SDPA,
closed forms, invariants, SPEC allocator examples, exhaustive interleavings).
No oracle function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "semipd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

BF16, FP32 = 0, 1
OK, INVALID, OOM, UNKNOWN_REQ, TABLE_FULL, BAD_BLOCK = 0, 1, 2, 3, 4, 5


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -fopenmp, IEEE fp64: no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
             "-ffp-contract=off", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            vp, ip, dp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.c_void_p
            i, d = ctypes.c_int, ctypes.c_double
            L.semipd_ref_attention_contig.argtypes = [i, i, i, i, i, i, i, vp, vp, vp, i, d, dp]
            L.semipd_ref_prefill.argtypes = [i, vp, vp, vp, i, i, i, i, i, i, i, vp, vp, vp,
                                             vp, vp, i, vp, i, d, dp, vp]
            L.semipd_ref_decode.argtypes = [i, vp, vp, i, i, i, i, i, i, i, vp, vp, vp, vp, vp,
                                            i, vp, i, d, dp]
            L.semipd_ref_partial.argtypes = [vp, vp, vp, i, i, i, i, d, dp, dp, dp]
            L.semipd_ref_merge.argtypes = [i, i, dp, dp, dp, dp]
            L.semipd_ref_merge.restype = None
            L.semipd_ref_partial.restype = None
            L.semipd_ref_alloc_init.argtypes = [i, i, i, vp, vp, vp, vp, vp]
            L.semipd_ref_alloc_init.restype = None
            L.semipd_ref_alloc.argtypes = [i, i, i, vp, vp, vp, vp, vp, i, vp, vp]
            L.semipd_ref_free.argtypes = [i, i, i, vp, vp, vp, vp, i, vp]
            L.semipd_ref_sm_budget.argtypes = [i, d]
            L.semipd_ref_effective_shares.argtypes = [d, d, ctypes.POINTER(d), ctypes.POINTER(d)]
            L.semipd_ref_effective_shares.restype = None
            L.semipd_ref_blocks_for_tokens.argtypes = [i, i]
            L.semipd_ref_rope_inv_freq.argtypes = [i, d, d, d, d, d, dp]
            L.semipd_ref_rope_inv_freq.restype = None
            L.semipd_ref_rope.argtypes = [i, i, i, i, i, i, vp, i, vp, d, d, d, d, d, dp]
            L.semipd_ref_rope.restype = None
            f = ctypes.c_float
            L.semipd_ref_e4m3_value.argtypes = [i]
            L.semipd_ref_e4m3_value.restype = d
            L.semipd_ref_e4m3_encode.argtypes = [f]
            L.semipd_ref_e4m3_quantize.argtypes = [i, vp, f, vp]
            L.semipd_ref_e4m3_quantize.restype = None
            L.semipd_ref_e4m3_values.argtypes = [i, vp, dp]
            L.semipd_ref_e4m3_values.restype = None
            L.semipd_ref_decode_fp8.argtypes = [i, vp, vp, i, i, i, i, i, vp, vp, vp, vp, vp, i,
                                                vp, i, f, f, d, dp]
            L.semipd_ref_round_bf16.argtypes = [d]
            L.semipd_ref_round_bf16.restype = d
            L.semipd_ref_prefill_mla_expanded.argtypes = [i, vp, vp, vp, i, i, i, i, i, i, vp, vp, vp,
                                                          i, vp, i, vp, vp, d, dp, vp]
            L.semipd_ref_prefill_fp8.argtypes = [i, vp, vp, vp, i, i, i, i, i, vp, vp, vp, vp, vp,
                                                 i, vp, i, f, f, d, dp, vp]
            _ = ip
            _lib = L
    return _lib


def set_threads(n: int) -> None:
    """OpenMP thread count for the oracle (bench cpu_baseline reports it)."""
    os.environ["OMP_NUM_THREADS"] = str(n)
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(ctypes.c_int(n))
    except OSError:
        pass


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.uint16:
        return BF16
    if a.dtype == np.float32:
        return FP32
    raise TypeError(f"oracle inputs are bf16 bit patterns (uint16) or float32, got {a.dtype}")


def _c(a, dt=None):
    a = np.ascontiguousarray(np.asarray(a) if dt is None else np.asarray(a).astype(dt, copy=False))
    return a


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def to_f64(a: np.ndarray) -> np.ndarray:
    """Exact widening of stored elements (bf16 bits as uint16, or fp32) to fp64."""
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def attention_contig(q, k, v, causal_offset: int, scale: float) -> np.ndarray:
    """q [nq,Hq,dk], k [nk,Hkv,dk], v [nk,Hkv,dv]; row t sees keys j <= offset+t
    (offset < 0: all keys).  Returns fp64 [nq,Hq,dv]."""
    q, k, v = _c(q), _c(k), _c(v)
    dt = _dtype_code(q)
    assert k.dtype == q.dtype == v.dtype
    nq, Hq, dk = q.shape
    nk, Hkv, _ = k.shape
    dv = v.shape[2]
    out = np.zeros((nq, Hq, dv), np.float64)
    st = lib().semipd_ref_attention_contig(nq, nk, Hq, Hkv, dk, dv, dt, _p(q), _p(k), _p(v),
                                           int(causal_offset), float(scale), _p(out))
    if st != OK:
        raise ValueError(f"oracle attention_contig status {st}")
    return out


def prefill(q, k_new, v_new, k_pool, v_pool, block_tables, cu_seqlens, req_ids, prefix_lens,
            scale: float, kv_shared: bool = False, rows_mask=None, dv: int | None = None):
    """Chunked causal GQA prefill over the paged pool (see semipd_oracle.c).

    k_pool/v_pool are MODIFIED in place (the K/V write of P:184); pass copies.
    Pools: [N_B, Hkv, bs, dk] / [N_B, Hkv, bs, dv] in the storage dtype.
    Returns fp64 out [T, Hq, dv] (rows outside rows_mask are zero)."""
    q, k_new = _c(q), _c(k_new)
    v_new = _c(v_new) if v_new is not None else k_new
    assert k_pool.flags.c_contiguous and (v_pool is None or v_pool.flags.c_contiguous)
    dt = _dtype_code(q)
    T, Hq, dk = q.shape
    N_B, Hkv, bs, _ = k_pool.shape
    if dv is None:
        dv = v_new.shape[2]
    bt = _c(block_tables, np.int32)
    cu = _c(cu_seqlens, np.int32)
    rid = _c(req_ids, np.int32)
    pl = _c(prefix_lens, np.int32)
    n = len(rid)
    out = np.zeros((T, Hq, dv), np.float64)
    mask = None if rows_mask is None else _c(rows_mask, np.uint8)
    vp = k_pool if (kv_shared or v_pool is None) else v_pool
    st = lib().semipd_ref_prefill(n, _p(cu), _p(rid), _p(pl), Hq, Hkv, dk, dv, bs,
                                  int(kv_shared), dt, _p(q), _p(k_new), _p(v_new), _p(k_pool),
                                  _p(vp), N_B, _p(bt), bt.shape[1], float(scale), _p(out),
                                  None if mask is None else _p(mask))
    if st != OK:
        raise ValueError(f"oracle prefill status {st}")
    return out


def decode(q, k_new, v_new, k_pool, v_pool, block_tables, req_ids, ctx_lens, scale: float,
           kv_shared: bool = False, dv: int | None = None):
    """One decode step; pools MODIFIED in place (append at slot ctx).  Returns fp64
    out [B, Hq, dv]."""
    q, k_new = _c(q), _c(k_new)
    v_new = _c(v_new) if v_new is not None else k_new
    dt = _dtype_code(q)
    B, Hq, dk = q.shape
    N_B, Hkv, bs, _ = k_pool.shape
    if dv is None:
        dv = v_new.shape[2]
    bt = _c(block_tables, np.int32)
    rid = _c(req_ids, np.int32)
    cl = _c(ctx_lens, np.int32)
    out = np.zeros((B, Hq, dv), np.float64)
    vp = k_pool if (kv_shared or v_pool is None) else v_pool
    st = lib().semipd_ref_decode(B, _p(rid), _p(cl), Hq, Hkv, dk, dv, bs, int(kv_shared), dt,
                                 _p(q), _p(k_new), _p(v_new), _p(k_pool), _p(vp), N_B, _p(bt),
                                 bt.shape[1], float(scale), _p(out))
    if st != OK:
        raise ValueError(f"oracle decode status {st}")
    return out


def partial(q, k, v, j0: int, j1: int, scale: float):
    """Split-K partial (m, l, acc) of fp64 q[dk] against keys [j0, j1)."""
    q, k, v = _c(q, np.float64), _c(k, np.float64), _c(v, np.float64)
    m, l_ = ctypes.c_double(), ctypes.c_double()
    acc = np.zeros(v.shape[1], np.float64)
    lib().semipd_ref_partial(_p(q), _p(k), _p(v), j0, j1, k.shape[1], v.shape[1], scale,
                             ctypes.byref(m), ctypes.byref(l_), _p(acc))
    return m.value, l_.value, acc


def merge(ms, ls, accs) -> np.ndarray:
    ms, ls, accs = _c(ms, np.float64), _c(ls, np.float64), _c(accs, np.float64)
    out = np.zeros(accs.shape[1], np.float64)
    lib().semipd_ref_merge(len(ms), accs.shape[1], _p(ms), _p(ls), _p(accs), _p(out))
    return out


def sm_budget(num_sms: int, pct: float) -> int:
    return lib().semipd_ref_sm_budget(num_sms, float(pct))


def effective_shares(x: float, y: float):
    a, b = ctypes.c_double(), ctypes.c_double()
    lib().semipd_ref_effective_shares(x, y, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def blocks_for_tokens(tokens: int, bs: int) -> int:
    return lib().semipd_ref_blocks_for_tokens(tokens, bs)


class Allocator:
    """Sequential model of the atomic block allocator (§4.4)."""

    def __init__(self, num_blocks: int, max_reqs: int, max_blocks_per_req: int):
        self.N_B, self.R, self.MBR = num_blocks, max_reqs, max_blocks_per_req
        self.free_stack = np.zeros(num_blocks, np.int32)
        self.top = np.zeros(1, np.int32)
        self.bt = np.zeros((max_reqs, max_blocks_per_req), np.int32)
        self.nblk = np.zeros(max_reqs, np.int32)
        self.min_free = np.zeros(1, np.int32)
        lib().semipd_ref_alloc_init(self.N_B, self.R, self.MBR, _p(self.free_stack),
                                    _p(self.top), _p(self.bt), _p(self.nblk), _p(self.min_free))

    def _state(self):
        return (self.N_B, self.R, self.MBR, _p(self.free_stack), _p(self.top), _p(self.bt),
                _p(self.nblk))

    def alloc(self, ids, counts) -> int:
        ids = _c(np.asarray(ids, dtype=np.int32).reshape(-1))
        counts = _c(np.asarray(counts, dtype=np.int32).reshape(-1))
        assert len(ids) == len(counts)
        return lib().semipd_ref_alloc(*self._state(), _p(self.min_free), len(ids), _p(ids),
                                      _p(counts))

    def free(self, ids) -> int:
        ids = _c(np.asarray(ids, dtype=np.int32).reshape(-1))
        return lib().semipd_ref_free(*self._state(), len(ids), _p(ids))

    @property
    def free_blocks(self) -> int:
        return int(self.top[0])

    def snapshot(self):
        return (self.free_stack.copy(), int(self.top[0]), self.bt.copy(), self.nblk.copy())


def rope_inv_freq(d: int, theta: float, factor: float = 0.0, lf: float = 1.0, hf: float = 4.0,
                  L0: float = 8192.0) -> np.ndarray:
    """RoPE frequencies f_i, i < d/2 (Llama-3.1 rescaling if factor > 1; DESIGN R27)."""
    out = np.zeros(d // 2, np.float64)
    lib().semipd_ref_rope_inv_freq(d, theta, factor, lf, hf, L0, _p(out))
    return out


def rope(x, positions, theta: float, factor: float = 0.0, lf: float = 1.0, hf: float = 4.0,
         L0: float = 8192.0, off: int = 0, rd: int | None = None,
         interleaved: bool = False) -> np.ndarray:
    """Rotate columns [off, off + rd) of x [T, H, d] (bf16 bits as uint16, or float32) at
    positions [T]; returns fp64 [T, H, d] (half-split or interleaved pairs, DESIGN R27)."""
    x = _c(x)
    T, H, d = x.shape
    pos = np.ascontiguousarray(positions, dtype=np.int32)
    out = np.zeros((T, H, d), np.float64)
    rd = d - off if rd is None else rd
    lib().semipd_ref_rope(T, H, d, off, rd, int(bool(interleaved)), _p(x), _dtype_code(x), _p(pos),
                          theta, factor, lf, hf, L0, _p(out))
    return out


# ---- FP8 (E4M3) KV pages (semipd_oracle.c, reading R31) ----

def e4m3_value(code: int) -> float:
    """Exact value of one E4M3 code (NaN codes -> nan)."""
    return lib().semipd_ref_e4m3_value(int(code))


def e4m3_encode(x: float) -> int:
    """Round-to-nearest-even, satfinite E4M3 code of one fp32 value."""
    return lib().semipd_ref_e4m3_encode(float(x))


def e4m3_quantize(x_bf16: np.ndarray, scale: float) -> np.ndarray:
    """Codes (uint8) of bf16 elements (uint16 bits) under the write rule E4M3(fl32(x / s))."""
    x = _c(x_bf16)
    assert x.dtype == np.uint16
    out = np.zeros(x.shape, np.uint8)
    lib().semipd_ref_e4m3_quantize(x.size, _p(x), float(scale), _p(out))
    return out


def e4m3_values(codes: np.ndarray) -> np.ndarray:
    """fp64 values of E4M3 codes (uint8)."""
    c = _c(codes, np.uint8)
    out = np.zeros(c.shape, np.float64)
    lib().semipd_ref_e4m3_values(c.size, _p(c), _p(out))
    return out


def decode_fp8(q, k_new, v_new, k_pool, v_pool, block_tables, req_ids, ctx_lens, scale: float,
               k_scale: float, v_scale: float):
    """One decode step on an E4M3 pool (uint8 codes [N_B, Hkv, bs, d]); pools MODIFIED in
    place (quantised append at slot ctx).  q / k_new / v_new are bf16 bits (uint16).
    Returns fp64 out [B, Hq, dv]."""
    q, k_new, v_new = _c(q), _c(k_new), _c(v_new)
    assert q.dtype == k_new.dtype == v_new.dtype == np.uint16
    assert k_pool.dtype == v_pool.dtype == np.uint8
    assert k_pool.flags.c_contiguous and v_pool.flags.c_contiguous
    B, Hq, dk = q.shape
    N_B, Hkv, bs, _ = k_pool.shape
    dv = v_new.shape[2]
    bt = _c(block_tables, np.int32)
    rid = _c(req_ids, np.int32)
    cl = _c(ctx_lens, np.int32)
    out = np.zeros((B, Hq, dv), np.float64)
    st = lib().semipd_ref_decode_fp8(B, _p(rid), _p(cl), Hq, Hkv, dk, dv, bs, _p(q), _p(k_new),
                                     _p(v_new), _p(k_pool), _p(v_pool), N_B, _p(bt), bt.shape[1],
                                     float(k_scale), float(v_scale), float(scale), _p(out))
    if st != OK:
        raise ValueError(f"oracle decode_fp8 status {st}")
    return out


def prefill_fp8(q, k_new, v_new, k_pool, v_pool, block_tables, cu_seqlens, req_ids, prefix_lens,
                scale: float, k_scale: float, v_scale: float, rows_mask=None):
    """Chunked causal GQA prefill on an E4M3 pool; pools MODIFIED in place (quantised chunk
    write).  Prefix keys are read back from the pool, the chunk's own keys are its bf16 rows.
    Returns fp64 out [T, Hq, dv] (rows outside rows_mask are zero)."""
    q, k_new, v_new = _c(q), _c(k_new), _c(v_new)
    assert q.dtype == k_new.dtype == v_new.dtype == np.uint16
    assert k_pool.dtype == v_pool.dtype == np.uint8
    assert k_pool.flags.c_contiguous and v_pool.flags.c_contiguous
    T, Hq, dk = q.shape
    N_B, Hkv, bs, _ = k_pool.shape
    dv = v_new.shape[2]
    bt = _c(block_tables, np.int32)
    cu = _c(cu_seqlens, np.int32)
    rid = _c(req_ids, np.int32)
    pl = _c(prefix_lens, np.int32)
    out = np.zeros((T, Hq, dv), np.float64)
    mask = None if rows_mask is None else _c(rows_mask, np.uint8)
    st = lib().semipd_ref_prefill_fp8(len(rid), _p(cu), _p(rid), _p(pl), Hq, Hkv, dk, dv, bs,
                                      _p(q), _p(k_new), _p(v_new), _p(k_pool), _p(v_pool), N_B,
                                      _p(bt), bt.shape[1], float(k_scale), float(v_scale),
                                      float(scale), _p(out), None if mask is None else _p(mask))
    if st != OK:
        raise ValueError(f"oracle prefill_fp8 status {st}")
    return out


# ---- Expanded-form MLA prefill (semipd_oracle.c, reading R32) ----

def round_bf16(x: float) -> float:
    """One round-to-nearest-even of a double onto bf16."""
    return lib().semipd_ref_round_bf16(float(x))


def prefill_mla_expanded(q, kv_new, pool, block_tables, cu_seqlens, req_ids, prefix_lens,
                         w_uk, w_uv, scale: float, dn: int = 128, dr: int = 64, rows_mask=None):
    """Expanded-form MLA prefill.  q [T, H, dn + dr] (q_nope | q_pe), kv_new [T, dc + dr] latent
    rows of the chunk, pool [N_B, 1, bs, dc + dr] latent pages (MODIFIED: the chunk rows are
    written), w_uk [H, dn, dc], w_uv [H, dv, dc]; all bf16 bits (uint16).  Returns fp64
    out [T, H, dv] (rows outside rows_mask are zero)."""
    q, kv_new, w_uk, w_uv = _c(q), _c(kv_new), _c(w_uk), _c(w_uv)
    assert q.dtype == kv_new.dtype == w_uk.dtype == w_uv.dtype == pool.dtype == np.uint16
    assert pool.flags.c_contiguous
    T, H, dq = q.shape
    assert dq == dn + dr
    N_B, hk, bs, dl = pool.shape
    assert hk == 1
    dc = dl - dr
    dv = w_uv.shape[1]
    assert w_uk.shape == (H, dn, dc) and w_uv.shape == (H, dv, dc)
    bt = _c(block_tables, np.int32)
    cu = _c(cu_seqlens, np.int32)
    rid = _c(req_ids, np.int32)
    pl = _c(prefix_lens, np.int32)
    out = np.zeros((T, H, dv), np.float64)
    mask = None if rows_mask is None else _c(rows_mask, np.uint8)
    st = lib().semipd_ref_prefill_mla_expanded(
        len(rid), _p(cu), _p(rid), _p(pl), H, dn, dr, dv, dc, bs, _p(q), _p(kv_new), _p(pool), N_B,
        _p(bt), bt.shape[1], _p(w_uk), _p(w_uv), float(scale), _p(out),
        None if mask is None else _p(mask))
    if st != OK:
        raise ValueError(f"oracle prefill_mla_expanded status {st}")
    return out
