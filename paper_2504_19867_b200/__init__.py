"""semi-PD (arXiv 2504.19867) co-run prefill/decode attention hot path for B200.

Thin ctypes binding over ``libsemipd.so`` (C ABI declared in ``include/semipd.h``).
Argument marshalling only: every step of the path (allocation, K/V writes,
prefill attention, decode attention, split merge) runs in the library's CUDA
kernels.  PyTorch supplies device memory, streams and process groups.  There is
no CPU fallback: if the extension is missing or no CUDA device is present the
calls raise.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import torch

from . import _build

__all__ = ["SemipdError", "PoolConfig", "KVPool", "lib", "build", "blocks_for_tokens",
           "STATUS", "RopeConfig", "rope_"]

STATUS = {0: "OK", 1: "INVALID", 2: "OOM", 3: "UNKNOWN_REQ", 4: "TABLE_FULL", 5: "BAD_BLOCK",
          6: "CUDA", 7: "UNSUPPORTED"}
OK, INVALID, OOM, UNKNOWN_REQ, TABLE_FULL, BAD_BLOCK, CUDA_ERR, UNSUPPORTED = range(8)
BF16, FP32, FP8_E4M3 = 0, 1, 2

_lib = None
_lock = threading.Lock()


class SemipdError(RuntimeError):
    def __init__(self, fn: str, status: int):
        super().__init__(f"{fn} failed: {STATUS.get(status, status)}")
        self.status = status


class _Cfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "num_layers", "num_blocks", "block_size", "num_kv_heads", "head_dim_k", "head_dim_v",
        "kv_shared", "max_reqs", "max_blocks_per_req", "dtype", "device", "oplog_words")]


class _RopeCfg(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_double), ("factor", ctypes.c_double),
                ("low_freq_factor", ctypes.c_double), ("high_freq_factor", ctypes.c_double),
                ("original_max_pos", ctypes.c_int32), ("rot_offset", ctypes.c_int32),
                ("rot_dim", ctypes.c_int32), ("interleaved", ctypes.c_int32)]


def build(force: bool = False) -> str:
    return _build.build(force=force)


def lib():
    """Load libsemipd.so (built in-tree).  Raises if it cannot be built/loaded."""
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("SEMIPD_LIB")  # dev: a tagged variant (scripts/variants.py)
            if not path:
                path = _build.LIB
                if not os.path.exists(path) or not _build.up_to_date():
                    _build.build()
            L = ctypes.CDLL(path)
            vp, i32, i64, sz, f32, f64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                          ctypes.c_size_t, ctypes.c_float, ctypes.c_double)
            P = ctypes.POINTER
            sig = {
                "semipd_kv_pool_bytes": (sz, [P(_Cfg)]),
                "semipd_kv_pool_create": (i32, [P(_Cfg), vp, sz, vp, P(vp)]),
                "semipd_kv_pool_destroy": (i32, [vp]),
                "semipd_kv_pool_views": (i32, [vp, i32, P(vp), P(vp), P(vp), P(vp)]),
                "semipd_alloc_blocks": (i32, [vp, vp, vp, i32, vp, vp]),
                "semipd_free_blocks": (i32, [vp, vp, i32, vp, vp]),
                "semipd_blocks_for_tokens": (i32, [i32, i32]),
                "semipd_pool_stats": (i32, [vp, P(i32), P(i32), vp]),
                "semipd_pool_oplog": (i32, [vp, vp, sz, P(i64), P(i64), vp]),
                "semipd_set_partition": (i32, [vp, f64, f64]),
                "semipd_get_sm_budgets": (i32, [vp, P(i32), P(i32)]),
                "semipd_num_sms": (i32, [vp]),
                "semipd_prefill_attn": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32,
                                              f32, vp, i32, i32, vp, vp]),
                "semipd_decode_attn": (i32, [vp, i32, vp, vp, vp, vp, vp, i32, i32, i32, f32, vp,
                                             i32, vp, sz, i32, vp, vp]),
                "semipd_decode_workspace_bytes": (sz, [vp, i32, i32, i32]),
                "semipd_launch_count": (i64, [vp]),
                "semipd_set_trace": (i32, [vp, vp, i32, vp]),
                "semipd_set_spans": (i32, [vp, vp, i32]),
                "semipd_set_rope": (i32, [vp, P(_RopeCfg)]),
                "semipd_version": (ctypes.c_char_p, []),
                "semipd_set_kv_scales": (i32, [vp, P(f32), P(f32)]),
                "semipd_fp8_prefill_scratch_bytes": (sz, [vp, i32]),
                "semipd_set_fp8_prefill_scratch": (i32, [vp, vp, sz, i32]),
                "semipd_ipc_alloc": (i32, [sz, P(vp), vp]),
                "semipd_ipc_free": (i32, [vp]),
                "semipd_ipc_open": (i32, [vp, P(vp)]),
                "semipd_ipc_close": (i32, [vp]),
                "semipd_peer_gather": (i32, [vp, sz, P(vp), P(vp), vp, i32, i32, vp]),
                "semipd_set_decode_peers": (i32, [vp, P(vp), i32, i32]),
                "semipd_set_prefill_peers": (i32, [vp, P(vp), i32, i32]),
                "semipd_peer_handshake": (i32, [P(vp), vp, i32, i32, i32, vp]),
                "semipd_rope": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, f64,
                                      f64, f64, f64, i32, vp]),
                "semipd_prefill_mla_expanded_workspace_bytes": (sz, [vp, i32, i32, i32]),
                "semipd_prefill_mla_expanded": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, i32, i32,
                                                      i32, i32, i32, f32, vp, vp, sz, i32, vp, vp]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _check(fn: str, st: int):
    if st != OK:
        raise SemipdError(fn, st)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def blocks_for_tokens(tokens: int, block_size: int) -> int:
    return int(lib().semipd_blocks_for_tokens(tokens, block_size))


_TORCH_DT = {BF16: torch.bfloat16, FP32: torch.float32}


@dataclass
class RopeConfig:
    """RoPE parameters (Llama-3.1 defaults: theta 5e5, factor 8, low / high frequency factors
    1 / 4, original context 8192; factor <= 1 = plain RoPE)."""
    theta: float = 500000.0
    factor: float = 8.0
    low_freq_factor: float = 1.0
    high_freq_factor: float = 4.0
    original_max_pos: int = 8192


def rope_(q, k, positions, cfg: RopeConfig | None = None, stream=None, rot_offset: int = 0,
          rot_dim: int | None = None, interleaved: bool = False):
    """Rotate columns [rot_offset, rot_offset + rot_dim) of q [T, Hq, d] and k [T, Hkv, d] in
    place at int32 positions [T]; half-split pairs, or adjacent pairs if ``interleaved``
    (C ABI ``semipd_rope``; runs in the library's kernel)."""
    cfg = cfg or RopeConfig()
    t = q if q is not None else k
    dt = BF16 if t.dtype == torch.bfloat16 else FP32 if t.dtype == torch.float32 else None
    if dt is None:
        raise SemipdError("semipd_rope", UNSUPPORTED)
    for x in (q, k):
        if x is not None and (not x.is_contiguous() or x.dim() != 3 or x.dtype != t.dtype or
                              x.device != t.device or x.shape[0] != t.shape[0] or
                              x.shape[2] != t.shape[2]):
            raise SemipdError("semipd_rope", INVALID)
    # positions: int32, one per token, on the rows' device (torch.arange defaults to int64,
    # which the kernel would misread)
    if (positions is None or positions.dtype != torch.int32 or positions.device != t.device or
            positions.numel() < t.shape[0] or not positions.is_contiguous()):
        raise SemipdError("semipd_rope", INVALID)
    _check("semipd_rope", lib().semipd_rope(
        _ptr(q), _ptr(k), _ptr(positions), int(t.shape[0]), 0 if q is None else int(q.shape[1]),
        0 if k is None else int(k.shape[1]), int(t.shape[2]), int(rot_offset),
        int(t.shape[2] - rot_offset if rot_dim is None else rot_dim), int(bool(interleaved)), dt,
        float(cfg.theta),
        float(cfg.factor), float(cfg.low_freq_factor), float(cfg.high_freq_factor),
        int(cfg.original_max_pos), _stream(stream)))
    return q, k


@dataclass
class PoolConfig:
    num_layers: int
    num_blocks: int
    block_size: int
    num_kv_heads: int
    head_dim_k: int
    head_dim_v: int
    max_reqs: int
    max_blocks_per_req: int
    dtype: torch.dtype = torch.bfloat16  # bfloat16, float32, or float8_e4m3fn (E4M3 pages)
    kv_shared: bool = False
    oplog_words: int = 1 << 16

    def code(self) -> int:
        return {torch.bfloat16: BF16, torch.float32: FP32, torch.float8_e4m3fn: FP8_E4M3}[self.dtype]

    def c(self, device: int) -> _Cfg:
        return _Cfg(self.num_layers, self.num_blocks, self.block_size, self.num_kv_heads,
                    self.head_dim_k, self.head_dim_v, int(self.kv_shared), self.max_reqs,
                    self.max_blocks_per_req, self.code(), device, self.oplog_words)


class KVPool:
    """The unified paged KV-cache pool (§4.4) on one GPU.

    Device memory comes from PyTorch (one uint8 tensor); the library carves it.
    All methods are stream-ordered on ``stream`` (default: current stream)."""

    def __init__(self, cfg: PoolConfig, device: int | torch.device = 0, stream=None):
        if not torch.cuda.is_available():
            raise RuntimeError("semipd needs a CUDA device (no CPU fallback)")
        dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.cfg, self.device = cfg, dev
        L = lib()
        self._c = cfg.c(dev.index)
        nbytes = L.semipd_kv_pool_bytes(ctypes.byref(self._c))
        if nbytes == 0:
            raise SemipdError("semipd_kv_pool_bytes", INVALID)
        self.mem = torch.empty(nbytes + 1024, dtype=torch.uint8, device=dev)
        base = self.mem.data_ptr()
        self._off = (-base) % 1024
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _check("semipd_kv_pool_create",
                   L.semipd_kv_pool_create(ctypes.byref(self._c), ctypes.c_void_p(base + self._off),
                                           nbytes, _stream(stream), ctypes.byref(h)))
        self.h = h
        self.nbytes = nbytes
        self.num_sms = int(L.semipd_num_sms(h))
        self._status = torch.zeros(4, dtype=torch.int32, device=dev)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.semipd_kv_pool_destroy(h)
            self.h = None

    # ---------------------------------------------------------------- views
    def _view(self, ptr: int, numel: int, dtype: torch.dtype, shape):
        off = ptr - self.mem.data_ptr()
        esz = torch.tensor([], dtype=dtype).element_size()
        return self.mem[off:off + numel * esz].view(dtype).view(*shape)

    def views(self, layer: int):
        """(K [N_B,Hkv,bs,dk], V [N_B,Hkv,bs,dv] or None if kv_shared, block_tables
        [R,MBR], nblk [R]) as torch views of the pool memory (tests/harness).  FP8 pools: K / V
        are uint8 views of the E4M3 codes."""
        k, v, bt, nb = (ctypes.c_void_p() for _ in range(4))
        _check("semipd_kv_pool_views", lib().semipd_kv_pool_views(
            self.h, layer, ctypes.byref(k), ctypes.byref(v), ctypes.byref(bt), ctypes.byref(nb)))
        c = self.cfg
        dt = torch.uint8 if c.dtype == torch.float8_e4m3fn else c.dtype  # FP8: the raw codes
        K = self._view(k.value, c.num_blocks * c.num_kv_heads * c.block_size * c.head_dim_k, dt,
                       (c.num_blocks, c.num_kv_heads, c.block_size, c.head_dim_k))
        V = None
        if not c.kv_shared:
            V = self._view(v.value, c.num_blocks * c.num_kv_heads * c.block_size * c.head_dim_v,
                           dt, (c.num_blocks, c.num_kv_heads, c.block_size, c.head_dim_v))
        BT = self._view(bt.value, c.max_reqs * c.max_blocks_per_req, torch.int32,
                        (c.max_reqs, c.max_blocks_per_req))
        NB = self._view(nb.value, c.max_reqs, torch.int32, (c.max_reqs,))
        return K, V, BT, NB

    # ---------------------------------------------------------------- allocator
    def alloc_blocks(self, req_ids: torch.Tensor, n_blocks: torch.Tensor, status=None,
                     stream=None):
        n = int(req_ids.numel())
        _check("semipd_alloc_blocks", lib().semipd_alloc_blocks(
            self.h, _ptr(req_ids), _ptr(n_blocks), n, _ptr(status), _stream(stream)))

    def free_blocks(self, req_ids: torch.Tensor, status=None, stream=None):
        _check("semipd_free_blocks", lib().semipd_free_blocks(
            self.h, _ptr(req_ids), int(req_ids.numel()), _ptr(status), _stream(stream)))

    def stats(self, stream=None):
        f, m = ctypes.c_int32(), ctypes.c_int32()
        _check("semipd_pool_stats", lib().semipd_pool_stats(self.h, ctypes.byref(f),
                                                             ctypes.byref(m), _stream(stream)))
        return f.value, m.value

    def oplog(self, stream=None):
        """Op log words (int32 list) and dropped-op count."""
        n, d = ctypes.c_int64(), ctypes.c_int64()
        L = lib()
        _check("semipd_pool_oplog", L.semipd_pool_oplog(self.h, None, 0, ctypes.byref(n),
                                                        ctypes.byref(d), _stream(stream)))
        buf = (ctypes.c_int32 * max(1, n.value))()
        _check("semipd_pool_oplog", L.semipd_pool_oplog(self.h, ctypes.cast(buf, ctypes.c_void_p),
                                                        4 * n.value, ctypes.byref(n),
                                                        ctypes.byref(d), _stream(stream)))
        return list(buf[:n.value]), d.value

    # ---------------------------------------------------------------- partition
    def set_partition(self, x: float, y: float):
        _check("semipd_set_partition", lib().semipd_set_partition(self.h, float(x), float(y)))

    def sm_budgets(self):
        a, b = ctypes.c_int32(), ctypes.c_int32()
        _check("semipd_get_sm_budgets", lib().semipd_get_sm_budgets(self.h, ctypes.byref(a),
                                                                     ctypes.byref(b)))
        return a.value, b.value

    def set_decode_peers(self, peer_ptrs, tokens: int = 0):
        """Fuse the TP head all-gather into the decode epilogue: later decode calls also store
        each output vector at these device addresses (C ABI ``semipd_set_decode_peers``;
        ``tp.PeerGather.peer_shard_ptrs`` gives them).  ``tokens`` = the batch the gathered
        buffers hold; a decode call with another batch is refused.  [] clears."""
        arr = (ctypes.c_void_p * max(1, len(peer_ptrs)))(*[int(x) for x in peer_ptrs])
        _check("semipd_set_decode_peers", lib().semipd_set_decode_peers(
            self.h, arr, len(peer_ptrs), int(tokens)))

    def set_prefill_peers(self, peer_ptrs, tokens: int = 0):
        """Fuse the TP head all-gather into the prefill epilogue (C ABI
        ``semipd_set_prefill_peers``); ``tokens`` = the total_q the gathered buffers hold.
        [] clears."""
        arr = (ctypes.c_void_p * max(1, len(peer_ptrs)))(*[int(x) for x in peer_ptrs])
        _check("semipd_set_prefill_peers", lib().semipd_set_prefill_peers(
            self.h, arr, len(peer_ptrs), int(tokens)))

    # ---------------------------------------------------------------- FP8 pools (R31)
    def set_kv_scales(self, k_scales=None, v_scales=None):
        """Per-layer fp32 tensor scales of an FP8 pool (C ABI ``semipd_set_kv_scales``);
        a float applies to every layer, None leaves that tensor's scales unchanged."""
        L = self.cfg.num_layers

        def arr(x):
            if x is None:
                return None
            xs = [float(x)] * L if isinstance(x, (int, float)) else [float(v) for v in x]
            if len(xs) != L:
                raise ValueError(f"need {L} scales, got {len(xs)}")
            return (ctypes.c_float * L)(*xs)
        _check("semipd_set_kv_scales", lib().semipd_set_kv_scales(self.h, arr(k_scales), arr(v_scales)))

    def attach_fp8_prefill_scratch(self, max_reqs_per_call: int):
        """Allocate (torch, on the pool's device) and attach the bf16 staging scratch an FP8
        pool's prefill reads its prefix through (C ABI ``semipd_set_fp8_prefill_scratch``)."""
        L = lib()
        nb = int(L.semipd_fp8_prefill_scratch_bytes(self.h, int(max_reqs_per_call)))
        if nb == 0:
            raise SemipdError("semipd_fp8_prefill_scratch_bytes", INVALID)
        mem = torch.empty(nb + 1024, dtype=torch.uint8, device=self.device)
        off = (-mem.data_ptr()) % 1024
        with torch.cuda.device(self.device):
            _check("semipd_set_fp8_prefill_scratch", L.semipd_set_fp8_prefill_scratch(
                self.h, ctypes.c_void_p(mem.data_ptr() + off), nb, int(max_reqs_per_call)))
        self._f8_scratch = mem  # keep alive while attached
        return mem

    def launch_count(self) -> int:
        return int(lib().semipd_launch_count(self.h))

    def set_trace(self, buf: torch.Tensor | None, counter: torch.Tensor | None = None):
        cap = 0 if buf is None else buf.numel() // 4
        _check("semipd_set_trace", lib().semipd_set_trace(self.h, _ptr(buf), cap, _ptr(counter)))

    def set_spans(self, buf: torch.Tensor | None):
        """Device-side launch timing (C ABI ``semipd_set_spans``): ``buf`` is a zeroed int64
        tensor [cap, 8] on the pool's device; the i-th attention launch from now on folds its
        first-CTA-entry -> last-CTA-exit time into row i % cap (col 2: total ns, col 3:
        launches, cols 5 / 6: the last launch's start / end).  None disables."""
        cap = 0 if buf is None else buf.shape[0]
        _check("semipd_set_spans", lib().semipd_set_spans(self.h, _ptr(buf), cap))

    def set_rope(self, cfg: "RopeConfig | None", rot_offset: int = 0, rot_dim: int | None = None,
                 interleaved: bool = False):
        """Fuse RoPE into the attention calls' K/V write (C ABI ``semipd_set_rope``): from now
        on prefill_attn / decode_attn rotate q and k_new IN PLACE at the positions the call
        implies (prefix + t / ctx) and write the rotated rows into the pool in the same pass.
        None turns it off."""
        if cfg is None:
            _check("semipd_set_rope", lib().semipd_set_rope(self.h, None))
            return
        rd = self.cfg.head_dim_k - rot_offset if rot_dim is None else rot_dim
        c = _RopeCfg(float(cfg.theta), float(cfg.factor), float(cfg.low_freq_factor),
                     float(cfg.high_freq_factor), int(cfg.original_max_pos), int(rot_offset),
                     int(rd), int(bool(interleaved)))
        _check("semipd_set_rope", lib().semipd_set_rope(self.h, ctypes.byref(c)))

    # ---------------------------------------------------------------- attention
    def prefill_attn(self, layer: int, q, k_new, v_new, cu_seqlens, req_ids, prefix_lens,
                     total_q: int, max_chunk_len: int, scale: float, out, out_head_major=False,
                     sm_budget: int = 0, status=None, stream=None):
        n = int(req_ids.numel())
        _check("semipd_prefill_attn", lib().semipd_prefill_attn(
            self.h, layer, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(cu_seqlens), _ptr(req_ids),
            _ptr(prefix_lens), n, int(total_q), int(max_chunk_len), int(q.shape[1]),
            float(scale), _ptr(out), int(bool(out_head_major)), int(sm_budget), _ptr(status),
            _stream(stream)))
        return out

    def mla_expanded_workspace_bytes(self, max_reqs: int, max_total_keys: int, num_heads: int) -> int:
        return int(lib().semipd_prefill_mla_expanded_workspace_bytes(
            self.h, int(max_reqs), int(max_total_keys), int(num_heads)))

    def new_mla_expanded_workspace(self, max_reqs: int, max_total_keys: int, num_heads: int):
        nb = self.mla_expanded_workspace_bytes(max_reqs, max_total_keys, num_heads)
        if nb == 0:
            raise SemipdError("semipd_prefill_mla_expanded_workspace_bytes", UNSUPPORTED)
        return torch.empty(nb, dtype=torch.uint8, device=self.device)

    def prefill_mla_expanded(self, layer: int, q, kv_new, w_uk, w_uv, cu_seqlens, req_ids,
                             prefix_lens, total_q: int, max_chunk_len: int, max_total_keys: int,
                             scale: float, out, workspace, sm_budget: int = 0, status=None,
                             stream=None):
        """Expanded-form MLA prefill (include/semipd.h, reading R32)."""
        _check("semipd_prefill_mla_expanded", lib().semipd_prefill_mla_expanded(
            self.h, layer, _ptr(q), _ptr(kv_new), _ptr(w_uk), _ptr(w_uv), _ptr(cu_seqlens),
            _ptr(req_ids), _ptr(prefix_lens), int(req_ids.numel()), int(total_q),
            int(max_chunk_len), int(max_total_keys), int(q.shape[1]), float(scale), _ptr(out),
            _ptr(workspace), 0 if workspace is None else workspace.numel(), int(sm_budget),
            _ptr(status), _stream(stream)))
        return out

    def decode_workspace_bytes(self, max_batch: int, num_q_heads: int, max_ctx: int) -> int:
        return int(lib().semipd_decode_workspace_bytes(self.h, max_batch, num_q_heads, max_ctx))

    def new_decode_workspace(self, max_batch: int, num_q_heads: int, max_ctx: int):
        nb = self.decode_workspace_bytes(max_batch, num_q_heads, max_ctx)
        return torch.zeros(max(nb, 256), dtype=torch.uint8, device=self.device)

    def decode_attn(self, layer: int, q, k_new, v_new, req_ids, ctx_lens, max_ctx_len: int,
                    scale: float, out, workspace, out_head_major=False, sm_budget: int = 0,
                    status=None, stream=None):
        _check("semipd_decode_attn", lib().semipd_decode_attn(
            self.h, layer, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(req_ids), _ptr(ctx_lens),
            int(req_ids.numel()), int(max_ctx_len), int(q.shape[1]), float(scale), _ptr(out),
            int(bool(out_head_major)), _ptr(workspace),
            0 if workspace is None else workspace.numel(), int(sm_budget), _ptr(status),
            _stream(stream)))
        return out
