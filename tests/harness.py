"""Test harness: drives the CUDA path through the binding and the oracle on the
same seeded inputs, and compares.  (Test infrastructure: may import both.)"""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth

TOL = {torch.bfloat16: (2e-2, 1e-2), torch.float32: (1e-4, 1e-4)}  # (max_abs, fro_rel) S16


def np_bits(t: torch.Tensor) -> np.ndarray:
    return synth.bits(t.detach().cpu())


def to64(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().double().numpy()


def compare(gpu: np.ndarray, ref: np.ndarray, dtype, what: str = ""):
    max_abs_tol, rel_tol = TOL[dtype]
    diff = np.abs(gpu - ref)
    max_abs = float(diff.max()) if diff.size else 0.0
    den = float(np.linalg.norm(ref))
    fro = float(np.linalg.norm(gpu - ref) / den) if den > 0 else float(np.linalg.norm(gpu - ref))
    assert np.all(np.isfinite(gpu)), f"{what}: non-finite GPU output"
    assert max_abs <= max_abs_tol and fro <= rel_tol, \
        f"{what}: max_abs={max_abs:.3e} (tol {max_abs_tol}) fro_rel={fro:.3e} (tol {rel_tol})"
    return max_abs, fro


class Rig:
    """A GPU pool plus the oracle allocator mirror."""

    def __init__(self, shape: synth.AttnShape, num_blocks: int, max_reqs: int, mbr: int,
                 num_layers: int = 1, device: int = 0):
        from paper_2504_19867_b200 import KVPool, PoolConfig
        self.shape = shape
        self.cfg = PoolConfig(num_layers=num_layers, num_blocks=num_blocks,
                              block_size=shape.block_size, num_kv_heads=shape.num_kv_heads,
                              head_dim_k=shape.head_dim_k, head_dim_v=shape.head_dim_v,
                              max_reqs=max_reqs, max_blocks_per_req=mbr, dtype=shape.dtype,
                              kv_shared=shape.kv_shared)
        self.pool = KVPool(self.cfg, device)
        self.dev = self.pool.device
        self.ref_alloc = oracle.Allocator(num_blocks, max_reqs, mbr)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)

    def i32(self, xs):
        return torch.tensor(list(xs), dtype=torch.int32, device=self.dev)

    def alloc(self, ids, counts, expect_ok=True):
        self.pool.alloc_blocks(self.i32(ids), self.i32(counts), self.status)
        st = int(self.status.item())
        ref = self.ref_alloc.alloc(ids, counts)
        assert st == ref, f"alloc status gpu={st} oracle={ref}"
        if expect_ok:
            assert st == 0
        return st

    def free(self, ids):
        self.pool.free_blocks(self.i32(ids), self.status)
        st = int(self.status.item())
        ref = self.ref_alloc.free(ids)
        assert st == ref, f"free status gpu={st} oracle={ref}"
        return st

    def tables(self):
        _, _, BT, NB = self.pool.views(0)
        return BT.cpu().numpy(), NB.cpu().numpy()

    def assert_tables_match(self):
        bt, nb = self.tables()
        np.testing.assert_array_equal(bt, self.ref_alloc.bt)
        np.testing.assert_array_equal(nb, self.ref_alloc.nblk)
        free, _ = self.pool.stats()
        assert free == self.ref_alloc.free_blocks

    def scatter(self, layer: int, rid: int, k_tok: torch.Tensor, v_tok, start: int = 0):
        """Harness layout step: place cached K/V of request `rid` at positions
        start.. using the ORACLE's table (bit copies, no arithmetic)."""
        if k_tok.shape[0] == 0:
            return
        K, V, _, _ = self.pool.views(layer)
        bs = self.shape.block_size
        pos = torch.arange(start, start + k_tok.shape[0])
        blk = torch.from_numpy(self.ref_alloc.bt[rid]).long()[pos // bs]
        assert bool((blk >= 0).all())
        K[blk.to(self.dev), :, (pos % bs).to(self.dev)] = k_tok.to(self.dev)
        if V is not None and v_tok is not None:
            V[blk.to(self.dev), :, (pos % bs).to(self.dev)] = v_tok.to(self.dev)

    def host_pool(self, layer: int):
        K, V, _, _ = self.pool.views(layer)
        kp = np_bits(K).copy()
        vp = np_bits(V).copy() if V is not None else None
        return kp, vp
