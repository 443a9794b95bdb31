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
    def create(backend: str | None = None) -> "PhaseGroups":
        ws, rank = dist.get_world_size(), dist.get_rank()
        ranks = list(range(ws))
        pg_p = dist.new_group(ranks, backend=backend)
        pg_d = dist.new_group(ranks, backend=backend)
        return PhaseGroups(pg_p, pg_d, ws, rank)


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
