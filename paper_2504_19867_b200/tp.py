"""Tensor parallelism by KV head (§4.5).

Each rank owns KV heads [k·Hkv/TP, (k+1)·Hkv/TP) and, by the GQA map g(h) = h // G
(DESIGN R3), the contiguous q heads [k·Hq/TP, (k+1)·Hq/TP).  Each rank has its own
pool shard and allocator, so attention needs no communication.  The one exchange
step is an all-gather of the head-major outputs [Hq/TP, T, dv] -> [Hq, T, dv]: the
kernels write head-major output (``out_head_major=1``), so the gathered tensor needs
no transpose.  P:232 has the prefill workers talk only to each other and the decode
workers only to each other, so there is one process group (one NCCL communicator)
per phase; collectives of the two phases never share a communicator.

Plumbing only (torch.distributed): no attention arithmetic lives here.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def head_range(num_heads: int, tp: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of the heads rank `rank` owns when `num_heads` are split over `tp`."""
    if num_heads % tp:
        raise ValueError(f"{num_heads} heads do not split over tp={tp}")
    per = num_heads // tp
    return rank * per, (rank + 1) * per


def shard_qkv(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor | None, tp: int, rank: int):
    """Slice token-major [T, H, d] activations to this rank's heads (views)."""
    ql, qh = head_range(q.shape[1], tp, rank)
    kl, kh = head_range(k.shape[1], tp, rank)
    return q[:, ql:qh], k[:, kl:kh], (None if v is None else v[:, kl:kh])


@dataclass
class PhaseGroups:
    """One process group per phase over the same ranks (prefill workers, decode workers)."""
    prefill: object
    decode: object
    tp: int
    rank: int

    @staticmethod
    def create(backend: str | None = None, max_ctas: int | None = None) -> "PhaseGroups":
        """Two groups over all ranks.  With NCCL and ``max_ctas``, each communicator is
        capped to that many CTAs (ncclConfig_t.maxCTAs), so its collectives take a bounded
        number of SMs out of the phase partition."""
        ws, rank = dist.get_world_size(), dist.get_rank()
        ranks = list(range(ws))
        opts = nccl_options(max_ctas) if backend in (None, "nccl") and max_ctas else None
        pg_p = dist.new_group(ranks, backend=backend, pg_options=opts)
        pg_d = dist.new_group(ranks, backend=backend, pg_options=opts)
        return PhaseGroups(pg_p, pg_d, ws, rank)


def nccl_options(max_ctas: int):
    """ProcessGroupNCCL options whose communicator runs at most ``max_ctas`` CTAs per
    collective (and at least 1)."""
    if max_ctas < 1:
        raise ValueError("max_ctas must be >= 1")
    opts = dist.ProcessGroupNCCL.Options()
    opts.config.max_ctas = int(max_ctas)
    opts.config.min_ctas = 1
    return opts


def gather_heads(local_head_major: torch.Tensor, out: torch.Tensor, group) -> torch.Tensor:
    """All-gather head-major shards [Hq/TP, T, dv] into out [Hq, T, dv] (rank order =
    head order)."""
    local = local_head_major.contiguous()
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)
    else:  # gloo (CPU tests): list form
        parts = list(out.chunk(dist.get_world_size(group), dim=0))
        dist.all_gather(parts, local, group=group)
    return out


class _DevBuf:
    """A raw device allocation exposed to torch through __cuda_array_interface__ (bytes)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 2}


class PeerGather:
    """All-gather of head-major shards [Hq/TP, T, dv] -> [Hq, T, dv] with the copy engines
    over IPC-mapped peer memory (C ABI ``semipd_peer_gather``).

    Every rank owns one exportable region (``semipd_ipc_alloc``) holding ``n_bufs`` gathered
    buffers plus a 2·TP uint32 flag array; the regions' IPC handles are exchanged once over
    ``group`` (any backend) and mapped (``semipd_ipc_open``).  A gather pushes this rank's
    shard into slot ``rank`` of every peer's buffer, then signals and waits with stream
    memory operations: no kernel, no SM of the phase partition.  The operations carry no
    per-call value, so a gather can be captured in a CUDA graph and replayed.  All ranks
    must issue the same sequence of gathers on one PeerGather, from one stream at a time.  The attention kernel can
    write its head-major output straight into ``local_view(buf)`` (then the local copy is
    skipped).  Plumbing only: no attention arithmetic lives here."""

    def __init__(self, full_shape, dtype: torch.dtype, group, device, n_bufs: int = 1):
        import ctypes
        import math

        from . import _check, lib

        self._ct = ctypes
        self._lib = lib()
        self._check = _check
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > 8 or full_shape[0] % self.world:
            raise ValueError(f"{full_shape[0]} heads do not shard over {self.world} ranks")
        self.device = torch.device(device)
        self.full_shape = tuple(full_shape)
        self.dtype = dtype
        esz = torch.tensor([], dtype=dtype).element_size()
        self.full_bytes = math.prod(full_shape) * esz
        self.shard_bytes = self.full_bytes // self.world
        self.buf_stride = -(-self.full_bytes // 256) * 256
        self.n_bufs = n_bufs
        self.flag_off = n_bufs * self.buf_stride
        nbytes = self.flag_off + 2 * self.world * 4
        ptr = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        with torch.cuda.device(self.device):
            _check("semipd_ipc_alloc", self._lib.semipd_ipc_alloc(nbytes, ctypes.byref(ptr), handle))
        self.base = ptr.value
        self._mem = torch.as_tensor(_DevBuf(self.base, nbytes), device=self.device)
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=group)
        self.peer_base = []
        self._opened = []
        for k, h in enumerate(handles):
            if k == self.rank:
                self.peer_base.append(self.base)
                continue
            p = ctypes.c_void_p()
            with torch.cuda.device(self.device):
                _check("semipd_ipc_open", self._lib.semipd_ipc_open(ctypes.create_string_buffer(h, 64),
                                                                    ctypes.byref(p)))
            self.peer_base.append(p.value)
            self._opened.append(p.value)
        self.calls = 0
        vp = ctypes.c_void_p
        self._flags = (vp * self.world)(*[b + self.flag_off for b in self.peer_base])

    def out(self, buf: int = 0) -> torch.Tensor:
        """The gathered buffer ``buf`` as a [Hq, T, dv] tensor on this rank."""
        off = buf * self.buf_stride
        return self._mem[off:off + self.full_bytes].view(self.dtype).view(self.full_shape)

    def local_view(self, buf: int = 0) -> torch.Tensor:
        """This rank's head slice of ``out(buf)`` (write the shard here to skip the local copy)."""
        h = self.full_shape[0] // self.world
        return self.out(buf)[self.rank * h:(self.rank + 1) * h]

    def peer_shard_ptrs(self, buf: int = 0) -> list[int]:
        """Device addresses of this rank's head slice in every OTHER rank's gathered buffer
        ``buf`` (for ``KVPool.set_decode_peers``: the decode epilogue stores there)."""
        off = buf * self.buf_stride + self.rank * self.shard_bytes
        return [b + off for k, b in enumerate(self.peer_base) if k != self.rank]

    def handshake(self, which: int, stream=None):
        """``which`` 0 ("ready": every peer is done reading) before a fused-epilogue decode,
        1 ("landed": every peer's stores are here) after it (C ABI ``semipd_peer_handshake``)."""
        ct = self._ct
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.calls += which
        self._check("semipd_peer_handshake", self._lib.semipd_peer_handshake(
            self._flags, ct.c_void_p(self.base + self.flag_off), self.world, self.rank, int(which),
            ct.c_void_p(stream.cuda_stream)))

    def __call__(self, local: torch.Tensor, buf: int = 0, stream=None) -> torch.Tensor:
        ct = self._ct
        if local.dtype != self.dtype or local.numel() * local.element_size() != self.shard_bytes:
            raise ValueError("shard shape / dtype does not match the gather")
        local = local.contiguous()
        off = buf * self.buf_stride + self.rank * self.shard_bytes
        dsts = (ct.c_void_p * self.world)(*[b + off for b in self.peer_base])
        self.calls += 1
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self._check("semipd_peer_gather", self._lib.semipd_peer_gather(
            ct.c_void_p(local.data_ptr()), self.shard_bytes, dsts, self._flags,
            ct.c_void_p(self.base + self.flag_off), self.world, self.rank,
            ct.c_void_p(stream.cuda_stream)))
        return self.out(buf)

    def close(self):
        """Unmap the peers' regions and free this rank's (after a device sync / barrier)."""
        for p in self._opened:
            self._lib.semipd_ipc_close(self._ct.c_void_p(p))
        self._opened = []
        if self.base:
            self._mem = None
            self._lib.semipd_ipc_free(self._ct.c_void_p(self.base))
            self.base = 0
