#!/usr/bin/env python
"""bench.py — co-run prefill + decode attention on one unified paged KV pool.

Headline workload (BASELINE.json configs[1], "Llama-3-8B attention shapes bf16"): 32 layers,
32 q / 8 kv heads, d = 128, 64-token pages (R7; the 16-token setting is reported
as the `block16` field); per step (one co-run iteration):
  stream P (prefill worker): alloc the prefill request's blocks, then for each layer
    semipd_prefill_attn on one 2048-token chunk (P = 0; K/V write + causal GQA attention),
    then free the request's blocks;
  stream D (decode worker), concurrently: for each layer semipd_decode_attn on 64 requests
    at ctx 2048 (K/V append + split-K paged attention).
The two persistent grids are capped to the (x, y) SM partition.  The sweep
x = 10 .. 90 (+ refinement around the best) picks the split; the K timed steps run there.

metric: attention-stack tokens/s = (2048 prefill + 64 decode tokens) x steps / time (each
token through all 32 layers).  value = device time (CUDA events around K CUDA-graph
replays, max over ranks), inputs resident in HBM; e2e = the same through the public API with
pinned host inputs copied in and outputs copied out every step.

Kernel times come from the library's device-side launch spans (semipd_set_spans: first CTA
entry -> last CTA exit, %globaltimer) accumulated over the same timed replays, so the
roofline fractions describe the timed steps themselves.

Secondary fields (N = 1): block16 (same workload, 16-token pages), cfg3 (Llama-3-70B shapes,
TP 1), cfg4 (long-context mix), cfg5 (DeepSeek-V2-Lite MLA latent), each with per-phase
roofline fractions at its best split.

Multi-GPU (torchrun, N ranks): tensor parallel by KV head (Hq/N, Hkv/N per rank, own pool
shard), the head-major outputs all-gathered per layer on a per-phase process group
whose NCCL communicator is capped to --nccl-max-ctas CTAs; strong scaling; the step is
captured into a CUDA graph (collectives included) when NCCL allows it, else it runs eagerly
and the line says so.  --tp-mode pipelined runs each gather on a per-phase comm stream
overlapping the next layer (attention grid = budget - NCCL CTAs).  The DP-replica reference
(every rank runs the TP-1 workload, no collective) is reported as `dp_replicas`.
--impl reference times the fp64 oracle (oracle/, the reference arm of this tier) on the host
cores.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

MODELS = {"llama3-8b": synth.CFG2_LLAMA8B, "llama3-70b": synth.CFG3_LLAMA70B}
PREFILL_TOKENS = 2048
DECODE_BATCH = 64
DECODE_CTX = 2048
METRIC = "co-run prefill+decode attention tokens/s (32-layer stack)"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="semipd", choices=["semipd", "reference"])
    ap.add_argument("--model", default="llama3-8b", choices=list(MODELS))
    ap.add_argument("--split", type=float, default=None, help="prefill SM percent x (y = 100-x)")
    ap.add_argument("--sweep", default="10,20,30,40,50,60,70,80,90")
    ap.add_argument("--block-size", type=int, default=64,
                    help="KV page size in tokens (64: one 16 KiB TMA box per (block, head) "
                         "page on B200; 16 is reported as the block16 field)")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "peer", "fused"],
                    help="TP head all-gather: NCCL all_gather (CTAs); peer = copy-engine pushes "
                         "over IPC-mapped peer memory with stream-memop flags (no SMs); fused = "
                         "both kernels store their output into the peers' buffers from the "
                         "epilogue")
    ap.add_argument("--tp-mode", default="dependent", choices=["dependent", "pipelined"],
                    help="dependent: layer l's gather on the phase stream before layer l+1; "
                         "pipelined: on a per-phase comm stream overlapping layer l+1 (NCCL)")
    ap.add_argument("--nccl-max-ctas", type=int, default=4,
                    help="ncclConfig_t.maxCTAs of each phase communicator (counted inside the "
                         "phase budget in pipelined mode)")
    ap.add_argument("--tails", default="0:0",
                    help="tail_p:tail_d schedules swept with every split (R30: the last layers of "
                         "the worker that finishes second run on all SMs once the other is done); "
                         "0:0 = the pure split")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sustained", type=float, default=1.0,
                    help="seconds of back-to-back replays after all fields (the power-capped "
                         "rate; 0 = skip)")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every kernel from Python instead of replaying a CUDA graph")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the block16 / cfg3 / cfg4 / cfg5 fields")
    ap.add_argument("--no-dp", action="store_true", help="N > 1: skip the DP-replica reference")
    ap.add_argument("--extra", action="store_true", default=True,
                    help="serial / (100,100) baselines (default on: the paper's spatial-vs-temporal claim)")
    ap.add_argument("--no-extra", dest="extra", action="store_false")
    return ap.parse_args(argv)


# ----------------------------------------------------------------------------- helpers
def ncu_traffic(kernel: str):
    """dram read + write bytes per launch of `kernel` from the newest committed ncu capture
    (profiles/r*_ncu_traffic.json, written from an `ncu --set full` run of the same shapes)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_traffic.json")))
    for path in reversed(files):
        try:
            with open(path) as f:
                d = json.load(f)[kernel]
            return int(d["dram_read_bytes"]) + int(d["dram_write_bytes"])
        except Exception:
            continue
    return None


def peaks():
    """HBM GB/s and dense bf16 TFLOP/s (burst and sustained) from MEASURED_PEAKS.json, else
    the profiling guide's fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"hbm": float(d["hbm_gbs"]), "burst": float(d["bf16_tflops"]),
                "sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "kind": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm": 6650.0, "burst": 1590.0, "sustained": 1400.0,
                "kind": "fallback (B200_PROFILING.md)"}


def nvml_id(dev: torch.device):
    """The NVML handle key of a CUDA device: its PCI bus id (CUDA and NVML indices differ
    under CUDA_VISIBLE_DEVICES), else the CUDA index."""
    try:
        pr = torch.cuda.get_device_properties(dev)
        return "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
    except Exception:
        return dev.index or 0


def _clock_sampler_proc(index, period: float, stop, out):
    """Child process: poll NVML SM clock + clock-event reasons until `stop` is set."""
    import pynvml
    pynvml.nvmlInit()
    if isinstance(index, str):
        h = pynvml.nvmlDeviceGetHandleByPciBusId(index.encode())
    else:
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
    rows = []
    out.put(("max", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)))
    while not stop.is_set():
        rows.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                     pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
                     pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(period)
    out.put(("rows", rows))


class ClockSampler:
    """SM clocks + throttle reasons polled through NVML every ~5 ms while the timed region
    runs, from a child process (a thread would starve behind the launch loop's GIL)."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, index, period_s: float = 0.005):
        self.index, self.period, self.rows, self.max_mhz = index, period_s, [], None
        self.err = None

    def __enter__(self):
        try:
            import multiprocessing as mp
            ctx = mp.get_context("spawn")
            self.stop, self.q = ctx.Event(), ctx.Queue()
            self.p = ctx.Process(target=_clock_sampler_proc,
                                 args=(self.index, self.period, self.stop, self.q), daemon=True)
            self.p.start()
            kind, v = self.q.get(timeout=60)  # NVML is up before the timed region starts
            self.max_mhz = v
        except Exception as e:  # pragma: no cover
            self.err = repr(e)
        return self

    def __exit__(self, *a):
        try:
            self.stop.set()
            kind, rows = self.q.get(timeout=30)
            self.rows = rows
            self.p.join(timeout=10)
        except Exception as e:  # pragma: no cover
            self.err = repr(e)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "error": self.err}
        import pynvml as nv
        reasons = sorted({name for r in self.rows for name, attr in self.REASONS.items()
                          if r[1] & getattr(nv, attr)})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_median": round(statistics.median(r[2] for r in self.rows), 1),
                "source": f"nvml, {self.period * 1e3:g} ms, child process"}


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def gpu_local_cpus(dev: torch.device):
    """The host CPUs NVML reports as local to `dev` (its NUMA node), or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        idx = nvml_id(dev)
        h = (pynvml.nvmlDeviceGetHandleByPciBusId(idx.encode()) if isinstance(idx, str)
             else pynvml.nvmlDeviceGetHandleByIndex(idx))
        n = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1}
        cpus &= set(range(n))
        return cpus or None
    except Exception:
        return None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- algorithmic work
def decode_bytes(shape: synth.AttnShape, ctx_lens, kv_bytes: int = 2) -> float:
    """Algorithmic HBM bytes of one decode launch: every visible
    key's K and V once (V aliases K for the MLA latent: the 576-d row once), q in, o out.
    kv_bytes = 1 for an FP8 (E4M3) pool (reading R31); q / o stay bf16."""
    eb = 2
    row = shape.head_dim_k if shape.kv_shared else shape.head_dim_k + shape.head_dim_v
    kv = sum(c + 1 for c in ctx_lens) * shape.num_kv_heads * row * kv_bytes
    io = len(ctx_lens) * shape.num_q_heads * (shape.head_dim_k + shape.head_dim_v) * eb
    return float(kv + io)


def prefill_flops(shape: synth.AttnShape, C: int, P: int) -> float:
    """2 Hq (dk + dv) per unmasked (q, k) pair; pairs = C P + C (C + 1) / 2."""
    pairs = C * P + C * (C + 1) / 2
    return 2.0 * shape.num_q_heads * (shape.head_dim_k + shape.head_dim_v) * pairs


def mla_expanded_flops(H: int, C: int, P: int) -> float:
    """Expanded-form MLA prefill (reading R32): the up-projection of every key's latent
    (2 x 512 x 2 H 128 per key, P + C keys) plus causal MHA at dqk 192 / dv 128:
    2 H (192 + 128) per unmasked (q, k) pair."""
    pairs = C * P + C * (C + 1) / 2
    return 2.0 * (P + C) * 512 * 2 * H * 128 + 2.0 * H * (192 + 128) * pairs


def prefill_bytes(shape: synth.AttnShape, C: int) -> float:
    """HBM bytes a prefill launch must move at P = 0: q in, o out, k_new / v_new in and
    their copy into the pool pages (a3, fused)."""
    eb = 2
    qo = C * shape.num_q_heads * (shape.head_dim_k + shape.head_dim_v) * eb
    kvrow = shape.head_dim_k if shape.kv_shared else shape.head_dim_k + shape.head_dim_v
    return float(qo + 2 * C * shape.num_kv_heads * kvrow * eb)


# ----------------------------------------------------------------------------- workload
class Workload:
    """Pool + resident inputs for one rank (head shard under TP): `L` layers of one prefill
    chunk of C tokens at prefix P (one request) and a decode step of B requests."""

    def __init__(self, shape: synth.AttnShape, tp: int, dev: torch.device, seed: int = 1020,
                 gather: str = "nccl", B: int = DECODE_BATCH, ctx=DECODE_CTX,
                 C: int = PREFILL_TOKENS, P: int = 0, layers: int | None = None,
                 tp_mode: str = "dependent", nccl_max_ctas: int = 4, groups=None,
                 max_prefix: int | None = None, kv_fp8: bool = False, mla_expanded: bool = False):
        from paper_2504_19867_b200 import KVPool, PoolConfig
        self.full = shape
        self.shape = synth.shard_heads(shape, tp) if tp > 1 else shape
        self.tp, self.dev, self.gather_mode, self.tp_mode = tp, dev, gather, tp_mode
        self.nccl_ctas = nccl_max_ctas
        s = self.shape
        self.L = layers or s.num_layers
        self.B, self.C = B, C
        self.ctx_list = list(ctx) if isinstance(ctx, (list, tuple)) else [int(ctx)] * B
        self.ctx = max(self.ctx_list)
        bs = s.block_size
        nb_dec = [c // bs + 1 for c in self.ctx_list]   # slot ctx needs block ctx // bs
        nb_pre_max = -(-(C + max(P, max_prefix or 0)) // bs)
        n_blocks = sum(nb_dec) + nb_pre_max + 64
        self.cfg = PoolConfig(num_layers=self.L, num_blocks=n_blocks, block_size=bs,
                              num_kv_heads=s.num_kv_heads, head_dim_k=s.head_dim_k,
                              head_dim_v=s.head_dim_v, max_reqs=B + 2,
                              max_blocks_per_req=max(max(nb_dec), nb_pre_max) + 8,
                              dtype=torch.float8_e4m3fn if kv_fp8 else s.dtype,
                              kv_shared=s.kv_shared)
        self.pool = KVPool(self.cfg, dev)
        self.kv_fp8 = kv_fp8
        # expanded-form MLA prefill (reading R32): q [C, H, 192], the chunk's
        # latent rows [C, 576], per-layer up-projections W_UK / W_UV [H, 128, 512]; the call
        # runs 3 spanned kernels per layer (prep, up-projection GEMM, attention)
        self.mla_exp = mla_expanded
        assert not mla_expanded or s.kv_shared
        if kv_fp8:  # E4M3 pages (reading R31): per-tensor scales, prefix staging scratch
            self.pool.set_kv_scales(0.05, 0.02)
            self.pool.attach_fp8_prefill_scratch(1)
        i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
        self.i32 = i32
        self.rid_dec = i32(list(range(B)))
        self.ctx_lens = i32(self.ctx_list)
        self.pool.alloc_blocks(self.rid_dec, i32(nb_dec))
        self.rid_pre = i32([B])
        self.cu = i32([0, C])
        self.set_prefix(P)
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        # cached context: random bf16 in every layer's pool (distinct memory per layer, so the
        # per-step decode working set is far larger than L2)
        for l in range(self.L):
            K, V, _, _ = self.pool.views(l)
            if kv_fp8:  # random finite E4M3 codes (|value| < 2^7 before the scale)
                for T in (K, V):
                    T.copy_(torch.randint(0, 0x70, T.shape, generator=g, device=dev, dtype=torch.int32)
                            .to(torch.uint8))
            else:
                K.normal_(generator=g)
                if V is not None:
                    V.normal_(generator=g)
        Hq, Hkv, dk, dv = s.num_q_heads, s.num_kv_heads, s.head_dim_k, s.head_dim_v
        mk = lambda *shp: torch.randn(*shp, generator=g, device=dev, dtype=torch.float32).to(s.dtype)  # noqa: E731
        self.qp = [mk(C, Hq, 192 if mla_expanded else dk) for _ in range(self.L)]
        self.kp = [mk(C, Hkv, dk) for _ in range(self.L)]
        if mla_expanded:
            self.w_uk = [(mk(Hq, 128, dk - 64).float() / math.sqrt(dk - 64)).to(s.dtype) for _ in range(self.L)]
            self.w_uv = [(mk(Hq, 128, dk - 64).float() / math.sqrt(dk - 64)).to(s.dtype) for _ in range(self.L)]
            self.ws_exp = self.pool.new_mla_expanded_workspace(1, C + max(P, max_prefix or 0), Hq)
        self.vp = [None if s.kv_shared else mk(C, Hkv, dv) for _ in range(self.L)]
        self.qd = [mk(B, Hq, dk) for _ in range(self.L)]
        self.kd = [mk(B, Hkv, dk) for _ in range(self.L)]
        self.vd = [None if s.kv_shared else mk(B, Hkv, dv) for _ in range(self.L)]
        hm = tp > 1
        dvp = 128 if mla_expanded else dv
        self.op = [torch.empty((Hq, C, dvp) if hm else (C, Hq, dvp), dtype=s.dtype, device=dev)
                   for _ in range(self.L)]
        self.od = [torch.empty((Hq, B, dv) if hm else (B, Hq, dv), dtype=s.dtype, device=dev)
                   for _ in range(self.L)]
        self.ws = self.pool.new_decode_workspace(B, Hq, self.ctx)
        self.scale = s.softmax_scale
        self.sP = torch.cuda.Stream(device=dev)
        self.sD = torch.cuda.Stream(device=dev)
        self.pg_p = self.pg_d = None
        self.peer_p = self.peer_d = None
        self.fused = False
        self.gath_p = self.gath_d = None
        self.cP = self.cD = None
        if tp > 1:
            from paper_2504_19867_b200 import tp as tpmod
            self.pg_p, self.pg_d = groups.prefill, groups.decode
            n_g = self.L if tp_mode == "pipelined" else 1
            self.gath_p = [torch.empty((self.full.num_q_heads, C, dv), dtype=s.dtype, device=dev)
                           for _ in range(n_g)]
            self.gath_d = [torch.empty((self.full.num_q_heads, B, dv), dtype=s.dtype, device=dev)
                           for _ in range(n_g)]
            if tp_mode == "pipelined":
                self.cP = torch.cuda.Stream(device=dev)
                self.cD = torch.cuda.Stream(device=dev)
                self.ev_kp = [torch.cuda.Event() for _ in range(self.L)]
                self.ev_kd = [torch.cuda.Event() for _ in range(self.L)]
            if gather in ("peer", "fused"):  # copy engines + stream memops instead of NCCL CTAs
                nb = 2 if gather == "fused" else 1
                self.peer_p = tpmod.PeerGather((self.full.num_q_heads, C, dv), s.dtype, self.pg_p,
                                               dev, n_bufs=nb)
                self.peer_d = tpmod.PeerGather((self.full.num_q_heads, B, dv), s.dtype, self.pg_d,
                                               dev, n_bufs=nb)
            if gather == "fused":
                # both epilogues store straight into every rank's gathered buffer; layers
                # alternate between two buffers, so a layer's output stays readable (e2e D2H)
                # while the next layer is written (E2E waits before reusing a buffer)
                self.fused = True
                self.od = [self.peer_d.local_view(l % 2) for l in range(self.L)]
                self.op = [self.peer_p.local_view(l % 2) for l in range(self.L)]
        # device-side launch spans: slots in enqueue order (corun_step sets span_order)
        self.spans = torch.zeros(4 * self.L + 8, 8, dtype=torch.int64, device=dev)
        self.span_k = {"prefill": 3 if mla_expanded else 1, "decode": 1}  # spans per layer
        self.span_order = ("prefill", "decode")
        self.ev_p_done, self.ev_d_done = torch.cuda.Event(), torch.cuda.Event()

    def set_prefix(self, P: int):
        """The prefill request's prefix length (its chunk's blocks are allocated per step)."""
        self.P = P
        self.prefix = self.i32([P])
        self.nb_pre = -(-(self.C + P) // self.shape.block_size)
        self.nblk_pre = self.i32([self.nb_pre])

    # ---- algorithmic work of one launch
    def decode_bytes_per_launch(self) -> float:
        return decode_bytes(self.shape, self.ctx_list, 1 if getattr(self, "kv_fp8", False) else 2)

    def prefill_flops_per_launch(self) -> float:
        if getattr(self, "mla_exp", False):
            return mla_expanded_flops(self.shape.num_q_heads, self.C, self.P)
        return prefill_flops(self.shape, self.C, self.P)

    def prefill_bytes_per_launch(self) -> float:
        return prefill_bytes(self.shape, self.C)

    # ---- launch spans
    def arm_spans(self):
        self.pool.set_spans(self.spans)

    def kernel_stats(self, order=None):
        """Mean launch duration (ms) per phase over everything folded into the spans since
        the last zero, and the last launch sequence's per-stream spans."""
        order = order or self.span_order
        sp = self.spans.cpu().numpy().astype(np.float64)
        out = {}
        off = 0
        for ph in order:
            k = getattr(self, "span_k", {}).get(ph, 1)
            r = sp[off:off + k * self.L]
            off += k * self.L
            n = r[:, 3].sum()
            # ms: the phase's kernel time per layer (k spanned kernels per layer summed)
            out[ph] = {"ms": float(r[:, 2].sum() / (n / k) / 1e6) if n else None,
                       "launches": int(n),
                       "stream_ms": float((r[-1, 6] - r[0, 5]) / 1e6) if n else None}
            if k > 1 and n:
                out[ph]["parts_ms"] = [float(r[j::k, 2].sum() / r[j::k, 3].sum() / 1e6) for j in range(k)]
        return out

    # ---- TP exchange of layer l on phase stream s
    def _gather(self, phase, l, s):
        from paper_2504_19867_b200 import tp as tpmod
        peer = self.peer_p if phase == "p" else self.peer_d
        outs = self.op if phase == "p" else self.od
        if self.fused:  # the kernel already stored; wait until every peer's stores landed
            peer.handshake(1, stream=s)
            return
        if peer is not None:
            peer(outs[l], stream=s)
            return
        gath = self.gath_p if phase == "p" else self.gath_d
        pg = self.pg_p if phase == "p" else self.pg_d
        if self.tp_mode == "pipelined":
            cs, ev = (self.cP, self.ev_kp) if phase == "p" else (self.cD, self.ev_kd)
            ev[l].record(s)
            cs.wait_event(ev[l])
            with torch.cuda.stream(cs):
                tpmod.gather_heads(outs[l], gath[l], pg)
        else:
            with torch.cuda.stream(s):
                tpmod.gather_heads(outs[l], gath[0], pg)

    def _budget(self, budget, phase):
        """Pipelined TP: the NCCL CTAs of the overlapping gather come out of the phase budget."""
        if self.tp > 1 and self.tp_mode == "pipelined" and self.gather_mode == "nccl":
            n = budget if budget > 0 else self.pool.sm_budgets()[0 if phase == "p" else 1]
            return max(1, n - self.nccl_ctas)
        return budget

    def phase_prefill(self, budget=0, stream=None, tail=0):
        """The prefill worker's iteration.  tail > 0: the last `tail` layers wait until the
        decode worker has issued all of its launches and then run on every SM (the freed
        decode SMs are adopted at the next launch, R30)."""
        s = stream or self.sP
        p = self.pool
        b = self._budget(budget, "p")
        with torch.cuda.stream(s):
            p.alloc_blocks(self.rid_pre, self.nblk_pre, None, stream=s)
            for l in range(self.L):
                if tail and l == self.L - tail:
                    s.wait_event(self.ev_d_done)
                    b = p.num_sms
                if self.fused:
                    p.set_prefill_peers(self.peer_p.peer_shard_ptrs(l % 2), self.C)
                    self.peer_p.handshake(0, stream=s)  # every peer is done reading
                if self.mla_exp:
                    p.prefill_mla_expanded(l, self.qp[l], self.kp[l], self.w_uk[l], self.w_uv[l],
                                           self.cu, self.rid_pre, self.prefix, self.C, self.C,
                                           self.C + self.P, 1 / math.sqrt(192), self.op[l],
                                           self.ws_exp, sm_budget=b, stream=s)
                else:
                    p.prefill_attn(l, self.qp[l], self.kp[l], self.vp[l], self.cu, self.rid_pre,
                                   self.prefix, self.C, self.C, self.scale, self.op[l],
                                   out_head_major=self.tp > 1, sm_budget=b, stream=s)
                if self.tp > 1:
                    self._gather("p", l, s)
            p.free_blocks(self.rid_pre, None, stream=s)
            if self.cP is not None:
                s.wait_stream(self.cP)
            self.ev_p_done.record(s)

    def phase_decode(self, budget=0, stream=None, tail=0):
        """The decode worker's iteration; tail as for phase_prefill (waits for the prefill
        worker's last launch, then runs its last `tail` layers on every SM)."""
        s = stream or self.sD
        p = self.pool
        b = self._budget(budget, "d")
        with torch.cuda.stream(s):
            for l in range(self.L):
                if tail and l == self.L - tail:
                    s.wait_event(self.ev_p_done)
                    b = p.num_sms
                if self.fused:
                    p.set_decode_peers(self.peer_d.peer_shard_ptrs(l % 2), self.B)
                    self.peer_d.handshake(0, stream=s)
                p.decode_attn(l, self.qd[l], self.kd[l], self.vd[l], self.rid_dec, self.ctx_lens,
                              self.ctx, self.scale, self.od[l], self.ws,
                              out_head_major=self.tp > 1, sm_budget=b, stream=s)
                if self.tp > 1:
                    self._gather("d", l, s)
            if self.cD is not None:
                s.wait_stream(self.cD)
            self.ev_d_done.record(s)

    def corun_step(self, x, y, tail_p=0, tail_d=0):
        """One co-run iteration: both workers concurrently at budgets from (x, y).  With
        tail_d (tail_p) > 0 the decode (prefill) worker's last layers run on all SMs once the
        other worker is done (R30); at most one of the two is non-zero.  The worker that
        waits is enqueued second, so its event wait sees this iteration's record."""
        assert not (tail_p and tail_d)
        main = torch.cuda.current_stream(self.dev)
        self.pool.set_partition(x, y)
        self.sP.wait_stream(main)
        self.sD.wait_stream(main)
        if tail_p:
            self.span_order = ("decode", "prefill")
            self.phase_decode(0)
            self.phase_prefill(0, tail=tail_p)
        else:
            self.span_order = ("prefill", "decode")
            self.phase_prefill(0)
            self.phase_decode(0, tail=tail_d)
        main.wait_stream(self.sP)
        main.wait_stream(self.sD)

    def serial_step(self):
        """Time-sliced baseline (unified system): each phase on all SMs in turn."""
        main = torch.cuda.current_stream(self.dev)
        n = self.pool.num_sms
        self.phase_prefill(n, stream=main)
        self.phase_decode(n, stream=main)

    def uncontrolled_step(self):
        """(100,100): non-persistent grids on both streams, hardware arbitrates."""
        main = torch.cuda.current_stream(self.dev)
        self.sP.wait_stream(main)
        self.sD.wait_stream(main)
        self.phase_prefill(-1)
        self.phase_decode(-1)
        main.wait_stream(self.sP)
        main.wait_stream(self.sD)

    def tokens_per_step(self) -> int:
        return self.C + self.B


def time_steps(fn, steps, dev, barrier=None):
    torch.cuda.synchronize(dev)
    if barrier:
        barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize(dev)
    if barrier:
        barrier()
    return e0.elapsed_time(e1) / 1e3  # seconds


def max_over_ranks(t: float, ws: int, dev) -> float:
    if ws > 1:
        tt = torch.tensor([t], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
    return t


class Runner:
    """Graph capture + timing of one workload's steps with the launch spans armed."""

    def __init__(self, w: Workload, dev, barrier=None, use_graph=True, ws=1):
        self.w, self.dev, self.barrier, self.use_graph, self.ws = w, dev, barrier, use_graph, ws
        self.graph_error = None

    def capture(self, fn):
        """Capture fn into a CUDA graph (spans armed first, so slot i = launch i of fn);
        returns a replay callable, or an eager callable that re-arms the spans each step if
        capture is off or fails."""
        w = self.w
        if self.use_graph:
            try:
                w.arm_spans()
                fn()
                torch.cuda.synchronize(self.dev)
                w.arm_spans()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    fn()
                g.replay()
                torch.cuda.synchronize(self.dev)
                return g.replay
            except Exception as e:  # NCCL without graph support etc.: eager, said in the line
                self.graph_error = repr(e)[:200]
                self.use_graph = False
                torch.cuda.synchronize(self.dev)

        def eager():
            w.arm_spans()
            fn()
        eager()
        torch.cuda.synchronize(self.dev)
        return eager

    def time(self, step, reps):
        """Seconds per step over `reps` calls (max over ranks) + the spans' kernel stats."""
        self.w.spans.zero_()
        t = time_steps(step, reps, self.dev, self.barrier) / reps
        return max_over_ranks(t, self.ws, self.dev), self.w.kernel_stats()


def phase_record(w: Workload, n_p: int, n_d: int, t_step: float, ks: dict, pk: dict) -> dict:
    """Per-split record: both phases' rates and roofline fractions
    from the spans of the timed replays.  tokens_per_s is for the workload's L-layer stack."""
    N = w.pool.num_sms
    dec_ms, pre_ms = ks["decode"]["ms"], ks["prefill"]["ms"]
    rec = {"n_p": n_p, "n_d": n_d, "ms": t_step * 1e3,
           "tokens_per_s": w.tokens_per_step() / t_step}
    if dec_ms:
        gbs = w.decode_bytes_per_launch() / (dec_ms / 1e3) / 1e9
        rec.update(decode_ms=dec_ms, decode_gbs=gbs, decode_frac=gbs / pk["hbm"])
    if pre_ms:
        tfs = w.prefill_flops_per_launch() / (pre_ms / 1e3) / 1e12
        share = n_p / N
        rec.update(prefill_ms=pre_ms, prefill_tflops=tfs, prefill_frac=tfs / pk["burst"],
                   prefill_frac_share_burst=tfs / (pk["burst"] * share),
                   prefill_frac_share_sustained=tfs / (pk["sustained"] * share))
    if dec_ms and pre_ms:
        rec["target_score"] = min(rec["decode_frac"] / 0.70, rec["prefill_frac_share_burst"] / 0.50)
        sp, sd = ks["prefill"]["stream_ms"], ks["decode"]["stream_ms"]
        rec["overlap"] = min(sp, sd) / max(sp, sd)
    return rec


def sweep_splits(w: Workload, run: Runner, xs, pk, reps=3, refine=True, tails=((0, 0),)):
    """Co-run at every x in xs (y = 100 - x) and every (tail_p, tail_d) schedule in `tails`,
    graph-replayed; refine +-2.5 / 5 around the best tokens/s with its tail.  Returns the
    records (pure splits have tail_p = tail_d = 0)."""
    out = []

    def measure(x, tp=0, td=0):
        step = run.capture(lambda: w.corun_step(x, 100 - x, tp, td))
        t, ks = run.time(step, reps)
        n_p, n_d = w.pool.sm_budgets()
        out.append({"x": x, "y": 100 - x, "tail_p": tp, "tail_d": td,
                    **phase_record(w, n_p, n_d, t, ks, pk)})

    for x in xs:
        for tp, td in tails:
            measure(x, tp, td)
    if refine and len(xs) > 1:
        b = max(out, key=lambda r: r["tokens_per_s"])
        for x in (b["x"] - 5, b["x"] - 2.5, b["x"] + 2.5, b["x"] + 5):
            if 0 < x < 100 and all(abs(r["x"] - x) > 1e-6 or (r["tail_p"], r["tail_d"]) !=
                                   (b["tail_p"], b["tail_d"]) for r in out):
                measure(x, b["tail_p"], b["tail_d"])
    out.sort(key=lambda r: (r["x"], r["tail_p"], r["tail_d"]))
    return out


def calibrated_corun(w: Workload, x, y, pk, step_p_ms, step_d_ms, target_ms=50.0, tries=3):
    """both workers loop on their own stream for >= target_ms, with the
    iteration counts calibrated so the two streams end within 5 % of each other; each phase's
    rate = its work / its own stream's elapsed time.  Eager launches (the host runs far
    ahead of the GPU here), events on each stream."""
    dev = w.dev
    kp = max(1, round(target_ms / step_p_ms))
    kd = max(1, round(target_ms / step_d_ms))
    rec = None
    for _ in range(tries):
        main = torch.cuda.current_stream(dev)
        w.pool.set_partition(x, y)
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        ep, ed = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        w.sP.wait_stream(main)
        w.sD.wait_stream(main)
        # interleave the two workers' submissions so neither stream starts long after the other
        for i in range(max(kp, kd)):
            if i < kp:
                w.phase_prefill(0)
            if i < kd:
                w.phase_decode(0)
        ep.record(w.sP)
        ed.record(w.sD)
        torch.cuda.synchronize(dev)
        tp_ms, td_ms = e0.elapsed_time(ep), e0.elapsed_time(ed)
        n_p, n_d = w.pool.sm_budgets()
        pre = kp * w.L * w.prefill_flops_per_launch() / (tp_ms / 1e3) / 1e12
        dec = kd * w.L * w.decode_bytes_per_launch() / (td_ms / 1e3) / 1e9
        rec = {"x": x, "y": y, "n_p": n_p, "n_d": n_d, "k_prefill_steps": kp, "k_decode_steps": kd,
               "prefill_stream_ms": tp_ms, "decode_stream_ms": td_ms,
               "overlap": min(tp_ms, td_ms) / max(tp_ms, td_ms),
               "prefill_tflops": pre, "prefill_frac_share_burst": pre / (pk["burst"] * n_p / w.pool.num_sms),
               "decode_gbs": dec, "decode_frac": dec / pk["hbm"],
               "note": "per-phase rates over the phase's own stream time (incl. alloc/free and "
                       "launch gaps), eager launches"}
        if rec["overlap"] >= 0.95:
            break
        # rescale the shorter stream's count toward the longer one
        if tp_ms < td_ms:
            kp = max(1, round(kp * td_ms / tp_ms))
        else:
            kd = max(1, round(kd * tp_ms / td_ms))
    return rec


def best_of(recs):
    best = max(recs, key=lambda r: r["tokens_per_s"])
    tgt = max((r for r in recs if "target_score" in r), key=lambda r: r["target_score"],
              default=None)
    return best, tgt


# ----------------------------------------------------------------------------- e2e
class E2E:
    """Same step through the public API with pinned host inputs/outputs: every step copies
    its inputs host -> device and its outputs device -> host inside the timed region.
    The copies run on their own streams, per layer, so the PCIe transfers pipeline with
    the attention kernels and H2D overlaps D2H (the copy engines are independent):
      H2D stream: layer l's prefill q / k / v and decode q / k / v, then an event each;
      stream P / D: wait for layer l's inputs, run the kernel, record an event;
      D2H stream: wait for layer l's outputs, copy them out, record an event.
    Device buffers are per layer (fused TP gather: two alternating buffers, and a phase
    waits for the D2H of layer l - 2 before writing its buffer again) and the step ends with
    the main stream joining all four streams, so nothing is overwritten while in use."""

    def __init__(self, w: Workload):
        self.w = w
        pin = lambda t: None if t is None else t.cpu().pin_memory()  # noqa: E731
        # device tensors the step's kernels use (the workload's own, or the packed views below)
        self.qp, self.kp, self.vp = list(w.qp), list(w.kp), list(w.vp)
        self.qd, self.kd, self.vd = list(w.qd), list(w.kd), list(w.vd)
        self.op, self.od = list(w.op), list(w.od)
        # (TP > 1 gathers the workload's own output buffers, so it keeps the per-tensor copies)
        self.packed = not w.fused and w.tp == 1
        if self.packed:
            # one pinned buffer and one device buffer per layer holding all six inputs (and one
            # pair for the two outputs): one H2D and one D2H copy per layer instead of six and
            # two (measured: pieces run H2D + D2H at 72 GB/s, per-layer copies at 80)
            def pack(ts, empty):
                offs, o = [], 0
                for t in ts:
                    offs.append(o)
                    if t is not None:
                        o += -(-t.numel() * t.element_size() // 4096) * 4096
                h = torch.empty(o, dtype=torch.uint8).pin_memory()
                d = torch.empty(o, dtype=torch.uint8, device=w.dev)
                hv, dv = [], []
                for t, off in zip(ts, offs):
                    if t is None:
                        hv.append(None)
                        dv.append(None)
                        continue
                    n = t.numel() * t.element_size()
                    hv.append(h[off:off + n].view(t.dtype).view(t.shape))
                    dv.append(d[off:off + n].view(t.dtype).view(t.shape))
                    if not empty:
                        hv[-1].copy_(t.cpu())
                        dv[-1].copy_(t)
                return h, d, hv, dv

            self.h_in, self.d_in, self.h_out, self.d_out = [], [], [], []
            self.h_qp, self.h_kp, self.h_vp, self.h_qd, self.h_kd, self.h_vd = ([] for _ in range(6))
            self.h_op, self.h_od = [], []
            for l in range(w.L):
                h, d, hv, dv = pack([w.qp[l], w.kp[l], w.vp[l], w.qd[l], w.kd[l], w.vd[l]], False)
                self.h_in.append(h)
                self.d_in.append(d)
                for lst, v in zip((self.h_qp, self.h_kp, self.h_vp, self.h_qd, self.h_kd, self.h_vd), hv):
                    lst.append(v)
                self.qp[l], self.kp[l], self.vp[l], self.qd[l], self.kd[l], self.vd[l] = dv
                h, d, hv, dv = pack([w.op[l], w.od[l]], True)
                self.h_out.append(h)
                self.d_out.append(d)
                self.h_op.append(hv[0])
                self.h_od.append(hv[1])
                self.op[l], self.od[l] = dv
        else:
            self.h_qp = [pin(t) for t in w.qp]
            self.h_kp = [pin(t) for t in w.kp]
            self.h_vp = [pin(t) for t in w.vp]
            self.h_qd = [pin(t) for t in w.qd]
            self.h_kd = [pin(t) for t in w.kd]
            self.h_vd = [pin(t) for t in w.vd]
            self.h_op = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in w.op]
            self.h_od = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in w.od]
        # bytes the step's copies move (packed: the whole per-layer buffers, alignment included)
        if self.packed:
            self.h2d = sum(h.numel() for h in self.h_in)
            self.d2h = sum(h.numel() for h in self.h_out)
        else:
            self.h2d = sum(t.numel() * t.element_size() for lst in
                           (self.h_qp, self.h_kp, self.h_vp, self.h_qd, self.h_kd, self.h_vd)
                           for t in lst if t is not None)
            self.d2h = sum(t.numel() * t.element_size() for lst in (self.h_op, self.h_od) for t in lst)
        self.s_in = torch.cuda.Stream(w.dev)
        self.s_out = torch.cuda.Stream(w.dev)
        ev = lambda: [torch.cuda.Event() for _ in range(w.L)]  # noqa: E731
        self.in_p, self.in_d, self.out_p, self.out_d = ev(), ev(), ev(), ev()
        self.done_p, self.done_d = ev(), ev()

    def step(self, x, y, tail_p=0, tail_d=0):
        w = self.w
        assert not (tail_p and tail_d)
        main = torch.cuda.current_stream(w.dev)
        w.pool.set_partition(x, y)
        for s in (self.s_in, self.s_out, w.sP, w.sD):
            s.wait_stream(main)

        def cp(d, h):
            if h is not None:
                d.copy_(h, non_blocking=True)

        with torch.cuda.stream(self.s_in):
            for l in range(w.L):
                if self.packed:
                    self.d_in[l].copy_(self.h_in[l], non_blocking=True)
                    self.in_d[l].record(self.s_in)
                    self.in_p[l].record(self.s_in)
                    continue
                cp(w.qd[l], self.h_qd[l])
                cp(w.kd[l], self.h_kd[l])
                cp(w.vd[l], self.h_vd[l])
                self.in_d[l].record(self.s_in)
                cp(w.qp[l], self.h_qp[l])
                cp(w.kp[l], self.h_kp[l])
                cp(w.vp[l], self.h_vp[l])
                self.in_p[l].record(self.s_in)
        tp = w.tp > 1
        nsm = w.pool.num_sms

        def prefill_phase():
            with torch.cuda.stream(w.sP):
                w.pool.alloc_blocks(w.rid_pre, w.nblk_pre, None, stream=w.sP)
                for l in range(w.L):
                    w.sP.wait_event(self.in_p[l])
                    b = 0
                    if tail_p and l >= w.L - tail_p:
                        if l == w.L - tail_p:
                            w.sP.wait_event(w.ev_d_done)
                        b = nsm
                    if w.fused:
                        if l >= 2:
                            w.sP.wait_event(self.done_p[l - 2])  # buffer l % 2 read out
                        w.pool.set_prefill_peers(w.peer_p.peer_shard_ptrs(l % 2), w.C)
                        w.peer_p.handshake(0, stream=w.sP)
                    w.pool.prefill_attn(l, self.qp[l], self.kp[l], self.vp[l], w.cu, w.rid_pre, w.prefix,
                                        w.C, w.C, w.scale, self.op[l], out_head_major=tp,
                                        sm_budget=b, stream=w.sP)
                    if tp:
                        w._gather("p", l, w.sP)  # same exchange step as the device-timed path
                    self.out_p[l].record(w.sP)
                w.pool.free_blocks(w.rid_pre, None, stream=w.sP)
                if w.cP is not None:
                    w.sP.wait_stream(w.cP)
                w.ev_p_done.record(w.sP)

        def decode_phase():
            with torch.cuda.stream(w.sD):
                for l in range(w.L):
                    w.sD.wait_event(self.in_d[l])
                    b = 0
                    if tail_d and l >= w.L - tail_d:
                        if l == w.L - tail_d:
                            w.sD.wait_event(w.ev_p_done)
                        b = nsm
                    if w.fused:
                        if l >= 2:
                            w.sD.wait_event(self.done_d[l - 2])
                        w.pool.set_decode_peers(w.peer_d.peer_shard_ptrs(l % 2), w.B)
                        w.peer_d.handshake(0, stream=w.sD)
                    w.pool.decode_attn(l, self.qd[l], self.kd[l], self.vd[l], w.rid_dec, w.ctx_lens, w.ctx,
                                       w.scale, self.od[l], w.ws, out_head_major=tp, sm_budget=b,
                                       stream=w.sD)
                    if tp:
                        w._gather("d", l, w.sD)
                    self.out_d[l].record(w.sD)
                if w.cD is not None:
                    w.sD.wait_stream(w.cD)
                w.ev_d_done.record(w.sD)

        if tail_p:
            decode_phase()
            prefill_phase()
        else:
            prefill_phase()
            decode_phase()
        with torch.cuda.stream(self.s_out):
            for l in range(w.L):
                if self.packed:
                    self.s_out.wait_event(self.out_d[l])
                    self.s_out.wait_event(self.out_p[l])
                    self.h_out[l].copy_(self.d_out[l], non_blocking=True)
                    self.done_d[l].record(self.s_out)
                    self.done_p[l].record(self.s_out)
                    continue
                self.s_out.wait_event(self.out_d[l])
                self.h_od[l].copy_(self.od[l], non_blocking=True)
                self.done_d[l].record(self.s_out)
                self.s_out.wait_event(self.out_p[l])
                self.h_op[l].copy_(self.op[l], non_blocking=True)
                self.done_p[l].record(self.s_out)
        for s in (self.s_in, self.s_out, w.sP, w.sD):
            main.wait_stream(s)


# ----------------------------------------------------------------------------- oracle arm
def oracle_sample_rate(shape: synth.AttnShape, threads: int, budget_s: float = 15.0):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload and
    extrapolate to attention-stack tokens/s for the full step.  About budget_s of CPU
    work, split evenly: decode = whole layer-steps of the B=64 ctx-2048 batch (all
    heads), repeated; prefill = evenly spaced rows of the 2048 chunk (all heads), the
    row count calibrated so the rows take ~budget_s/2 (causal cost averages out)."""
    import oracle
    oracle.set_threads(threads)
    s = shape
    bs = s.block_size
    rng = np.random.default_rng(0)
    to_bits = lambda a: (a.view(np.uint32) >> 16).astype(np.uint16)  # noqa: E731 (bf16 bit patterns)
    bf = lambda *sh: to_bits(rng.standard_normal(sh).astype(np.float32))  # noqa: E731
    # decode sample: the whole B-request batch of one layer, repeated
    B = DECODE_BATCH
    nb = DECODE_CTX // bs + 1
    kpool, vpool = bf(B * nb, s.num_kv_heads, bs, s.head_dim_k), bf(B * nb, s.num_kv_heads, bs, s.head_dim_v)
    bt = np.arange(B * nb, dtype=np.int32).reshape(B, nb)
    q, kn, vn = bf(B, s.num_q_heads, s.head_dim_k), bf(B, s.num_kv_heads, s.head_dim_k), bf(B, s.num_kv_heads, s.head_dim_v)
    reps, t_dec = 0, 0.0
    t0 = time.perf_counter()
    while reps == 0 or t_dec < budget_s / 2:
        oracle.decode(q, kn, vn, kpool, vpool, bt, list(range(B)), [DECODE_CTX] * B, s.softmax_scale)
        reps += 1
        t_dec = time.perf_counter() - t0
    t_dec_layer = t_dec / reps
    del kpool, vpool
    # prefill sample: evenly spaced rows of the 2048 chunk
    C = PREFILL_TOKENS
    nbp = -(-C // bs)
    kpp = np.zeros((nbp, s.num_kv_heads, bs, s.head_dim_k), np.uint16)
    vpp = np.zeros((nbp, s.num_kv_heads, bs, s.head_dim_v), np.uint16)
    btp = np.arange(nbp, dtype=np.int32).reshape(1, nbp)
    qp, kp, vp = bf(C, s.num_q_heads, s.head_dim_k), bf(C, s.num_kv_heads, s.head_dim_k), bf(C, s.num_kv_heads, s.head_dim_v)

    def rows(stride):
        mask = np.zeros(C, np.uint8)
        mask[stride // 2::stride] = 1
        t = time.perf_counter()
        oracle.prefill(qp, kp, vp, kpp, vpp, btp, [0, C], [0], [0], s.softmax_scale, rows_mask=mask)
        return time.perf_counter() - t, int(mask.sum())

    t_cal, n_cal = rows(256)
    per_row = t_cal / n_cal
    n_rows = int(min(C, max(n_cal, (budget_s / 2) / per_row)))
    stride = max(1, C // n_rows)
    t_pre, n_rows = rows(stride)
    t_pre_chunk = t_pre * C / n_rows
    t_step = s.num_layers * (t_dec_layer + t_pre_chunk)
    tokens = PREFILL_TOKENS + DECODE_BATCH
    sample = (f"{reps}x one decode layer-step (B={B}, ctx {DECODE_CTX}, all {s.num_q_heads} heads) "
              f"in {t_dec:.1f} s + {n_rows} of {C} prefill rows (every {stride}th, all heads, 1 layer) "
              f"in {t_pre:.1f} s; extrapolated x{s.num_layers} layers, x{C / n_rows:.0f} rows")
    return tokens / t_step, sample, time.perf_counter()


def cpu_baseline(shape, budget_nproc: float = 12.0, budget_1: float = 8.0) -> dict:
    """The oracle at nproc threads (the reported value) and at 1 thread, with the CPU model."""
    import oracle
    threads = os.cpu_count() or 1
    v, sample, _ = oracle_sample_rate(shape, threads, budget_nproc)
    v1, sample1, _ = oracle_sample_rate(shape, 1, budget_1)
    oracle.set_threads(threads)
    return {"value": v, "unit": "tokens/s", "cores": threads, "kind": "oracle", "sample": sample,
            "nproc": threads, "cpu_model": cpu_model(),
            "one_thread": {"value": v1, "unit": "tokens/s", "sample": sample1},
            "parallel_speedup": v / v1 if v1 else None}


def workload_config(shape: synth.AttnShape, ws: int, gather: str = "nccl",
                    tp_mode: str = "dependent") -> dict:
    """The `config` both arms print (the reference arm runs the same workload)."""
    decode_gb = shape.num_layers * (DECODE_BATCH * (DECODE_CTX + 1) * shape.num_kv_heads * 2 * 128 * 2) / 1e9
    return {"workload": f"{shape.name} attention (Hq {shape.num_q_heads}, Hkv {shape.num_kv_heads}, "
                        f"d 128, bs {shape.block_size}, {shape.num_layers} layers): decode B={DECODE_BATCH} "
                        f"ctx={DECODE_CTX} + prefill chunk {PREFILL_TOKENS} (P=0), co-run",
            "parallelism": (f"tp{ws} (KV-head shards, "
                            + {"peer": "copy-engine peer all-gather)",
                               "fused": "peer stores from the decode / prefill epilogues)"}
                            .get(gather, f"NCCL all-gather, {tp_mode})")
                            if ws > 1 else "tp1"),
            "l2": f"no flush: per-step decode working set {decode_gb:.1f} GB >> 126 MB L2"}


def run_reference(args):
    ws, rank, _ = dist_info()
    if rank != 0:
        return 0
    shape = dataclasses.replace(MODELS[args.model], block_size=args.block_size)
    threads = os.cpu_count() or 1
    # each step is a bounded sample; the whole --steps/--warmup run stays within ~3 min
    budget = max(2.0, min(15.0, 180.0 / (args.steps + args.warmup)))
    vals = []
    t_start = time.perf_counter()
    for i in range(args.warmup + args.steps):
        v, sample, _ = oracle_sample_rate(shape, threads, budget)
        if i >= args.warmup:
            vals.append(v)
    elapsed = time.perf_counter() - t_start
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * (PREFILL_TOKENS + DECODE_BATCH) / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(shape, 1),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle",
                         "sample": sample, "cpu_model": cpu_model(),
                         "step_time": "extrapolated from the sample (per-row / per-layer rates)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": elapsed,
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- secondary fields
def _sweep_field(w: Workload, dev, pk, xs, **info):
    run = Runner(w, dev)
    recs = sweep_splits(w, run, xs, pk, reps=3, refine=False)
    best, tgt = best_of(recs)
    return {**info, "layers": w.L, "best": best, "best_target": tgt, "sweep": recs}


def secondary_block16(args, dev, pk):
    """The headline workload with 16-token pages (SURVEY S7's reading)."""
    shape = dataclasses.replace(MODELS[args.model], block_size=16)
    return _sweep_field(Workload(shape, 1, dev, seed=1016), dev, pk, [20, 25, 30, 40, 50],
                        block_size=16)


def secondary_cfg3(args, dev, pk):
    """BASELINE configs[2] shapes on one GPU (TP 1): Llama-3-70B attention (Hq 64, Hkv 8,
    G = 8), 80 layers, same per-step workload."""
    shape = dataclasses.replace(synth.CFG3_LLAMA70B, block_size=args.block_size)
    return _sweep_field(Workload(shape, 1, dev, seed=1030), dev, pk, [30, 35, 40, 45, 50, 55, 60],
                        model="llama3-70b (TP 1)")


def secondary_cfg4(args, dev, pk, layers: int = 8):
    """BASELINE configs[3]: 16 decode requests at ctx 32768 + 8192-token chunks of a 32k
    prompt at P = 0, 8192, 16384, 24576, under the partition schedule (30,70) -> (50,50) ->
    (70,30).  `layers` distinct layers (working set 17 GB >> L2); rates are per launch;
    tokens_per_s is for the `layers`-layer stack.  Also the partition-switch cost (eager: the
    first step after set_partition vs the next two) with zero KV bytes moved."""
    shape = dataclasses.replace(synth.CFG2_LLAMA8B, block_size=64)
    w = Workload(shape, 1, dev, seed=1040, B=16, ctx=32768, C=8192, P=0, layers=layers,
                 max_prefix=24576)
    out = {"layers": layers, "decode": "B=16 ctx 32768 (S=9 splits)",
           "prefill": "C=8192 at P = 0 / 8192 / 16384 / 24576", "splits": []}
    for x, y in [(30, 70), (50, 50), (70, 30)]:
        per_p = []
        for P in (0, 8192, 16384, 24576):
            w.set_prefix(P)
            run = Runner(w, dev)
            step = run.capture(lambda: w.corun_step(x, y))
            t, ks = run.time(step, 2)
            n_p, n_d = w.pool.sm_budgets()
            per_p.append({"P": P, **phase_record(w, n_p, n_d, t, ks, pk)})
        out["splits"].append({
            "x": x, "y": y, "n_p": per_p[0]["n_p"], "n_d": per_p[0]["n_d"], "per_prefix": per_p,
            "decode_frac_mean": statistics.mean(r["decode_frac"] for r in per_p),
            "prefill_frac_share_burst_mean": statistics.mean(r["prefill_frac_share_burst"]
                                                             for r in per_p),
            "tokens_per_s_cycle": 4 * w.tokens_per_step() / sum(r["ms"] for r in per_p) * 1e3})
    w.set_prefix(0)
    ptr0 = w.pool.mem.data_ptr()
    sw = []
    for _ in range(2):  # eager warm-up at the last split, so the first switch is not a cold step
        w.corun_step(70, 30)
    torch.cuda.synchronize(dev)
    for x, y in [(30, 70), (50, 50), (70, 30), (30, 70)]:
        ts = [time_steps(lambda: w.corun_step(x, y), 1, dev) * 1e3 for _ in range(3)]
        sw.append({"x": x, "first_ms": ts[0], "steady_ms": statistics.mean(ts[1:]),
                   "switch_cost_ms": ts[0] - statistics.mean(ts[1:])})
    out["switch"] = sw
    out["kv_moved_bytes"] = 0 if w.pool.mem.data_ptr() == ptr0 else None
    out["best_target"] = max(out["splits"], key=lambda r: min(
        r["decode_frac_mean"] / 0.7, r["prefill_frac_share_burst_mean"] / 0.5))
    return out


def secondary_fp8(args, dev, pk):
    """The headline workload over an FP8 (E4M3) pool (reading R31): decode
    reads 1-byte codes (half the bytes: the decode fraction is against the FP8 byte count),
    prefill attends its chunk at bf16 with P = 0 (the quantised K/V write is a separate pass)."""
    shape = dataclasses.replace(MODELS[args.model], block_size=64)
    return _sweep_field(Workload(shape, 1, dev, seed=1080, kv_fp8=True), dev, pk,
                        [30, 35, 40, 45, 50, 55, 60], kv_dtype="e4m3 (scales 0.05 / 0.02)")


def secondary_cfg5(args, dev, pk):
    """BASELINE configs[4] kernels at trace-like scale: DeepSeek-V2-Lite absorbed MLA (16 q
    heads over the 576-d latent, V = K[:, :512], 64-token pages, 27 layers); decode B = 256
    at lognormal contexts (mean ~350, seed 5005) co-running with a 2048-token prefill chunk."""
    rng = np.random.default_rng(5005)
    ctx = [int(c) for c in np.clip(rng.lognormal(math.log(350.0) - 0.125, 0.5, 256), 64, 4096)]
    ctx.sort(reverse=True)  # the engine's decode batch order: longest first (LPT, engine.py)
    w = Workload(synth.CFG5_MLA, 1, dev, seed=1050, B=256, ctx=ctx, C=2048)
    return _sweep_field(w, dev, pk, [15, 20, 25, 30, 40, 50, 60, 70], model="deepseek-v2-lite-mla",
                        decode_ctx_mean=statistics.mean(ctx))


def secondary_cfg5_expanded(args, dev, pk):
    """cfg5_mla with the expanded-form MLA prefill (reading R32): the same
    decode batch (absorbed decode over the latent) co-running with the 2048-token chunk's
    prefill as prep + up-projection GEMM + causal MHA at dqk 192 / dv 128 (3 kernels per layer); the
    prefill rate and fraction are against the expanded form's own flops (mla_expanded_flops)."""
    rng = np.random.default_rng(5005)
    ctx = [int(c) for c in np.clip(rng.lognormal(math.log(350.0) - 0.125, 0.5, 256), 64, 4096)]
    ctx.sort(reverse=True)
    w = Workload(synth.CFG5_MLA, 1, dev, seed=1050, B=256, ctx=ctx, C=2048, mla_expanded=True)
    return _sweep_field(w, dev, pk, [15, 25, 40, 50, 60, 70, 80, 90], model="deepseek-v2-lite-mla",
                        prefill_form="expanded (R32)", decode_ctx_mean=statistics.mean(ctx))


# ----------------------------------------------------------------------------- main
def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        return run_reference(args)
    ws, rank, local = dist_info()
    # dev-only overrides to exercise the N > 1 plumbing on a one-GPU box: every rank on
    # cuda:0 and the gloo backend (NCCL refuses two ranks on one device). Never set by the driver.
    one_gpu = os.environ.get("SPD_BENCH_ONE_GPU") == "1"
    backend = os.environ.get("SPD_BENCH_BACKEND", "nccl")
    dev = torch.device("cuda", 0 if one_gpu else local)
    torch.cuda.set_device(dev)
    barrier = None
    groups = None
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")       # communicator rank counts in the log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        barrier = lambda: dist.barrier()  # noqa: E731
        from paper_2504_19867_b200 import tp as tpmod
        groups = tpmod.PhaseGroups.create(backend=backend, max_ctas=args.nccl_max_ctas)
    shape = dataclasses.replace(MODELS[args.model], block_size=args.block_size)
    w = Workload(shape, ws, dev, gather=args.gather, tp_mode=args.tp_mode,
                 nccl_max_ctas=args.nccl_max_ctas, groups=groups)
    pk = peaks()
    W = max(3, args.warmup)
    run = Runner(w, dev, barrier, not args.no_graph, ws)
    for _ in range(2):
        w.corun_step(50, 50)
    # ---- split sweep (graph-replayed, per-split roofline record; not part of the value)
    xs = [float(x) for x in args.sweep.split(",")] if args.split is None else [args.split]
    tails = tuple(tuple(int(v) for v in t.split(":")) for t in args.tails.split(","))
    sweep = sweep_splits(w, run, xs, pk, reps=3, refine=args.split is None, tails=tails)
    best, tgt = best_of(sweep)
    pure = [r for r in sweep if r["tail_p"] == 0 and r["tail_d"] == 0]
    best_pure = max(pure, key=lambda r: r["tokens_per_s"]) if pure else None
    x, y, tp, td = best["x"], best["y"], best["tail_p"], best["tail_d"]
    # the sweep's 3 replays per split can misorder splits within ~2 %: re-time the three best
    # schedules exactly as the timed region will run them (W warm-up replays, then K timed) and
    # run the timed region at the fastest of those.  Back-to-back replays reach the board's
    # power cap within ~0.2 s, and the splits do not slow alike under it (power)
    reselect = []
    if args.split is None and len(sweep) > 1:
        top = sorted(sweep, key=lambda r: -r["tokens_per_s"])[:3]
        for r in top:
            st_ = run.capture(lambda r=r: w.corun_step(r["x"], r["y"], r["tail_p"], r["tail_d"]))
            for _ in range(W):
                st_()
            t_, _ = run.time(st_, args.steps)
            reselect.append({"x": r["x"], "tail_p": r["tail_p"], "tail_d": r["tail_d"],
                             "sweep_ms": r["ms"], "ms_timed_protocol": t_ * 1e3})
        pick = min(reselect, key=lambda r: r["ms_timed_protocol"])
        x, y, tp, td = pick["x"], 100 - pick["x"], pick["tail_p"], pick["tail_d"]
    # library launches of one step (an eager step; graph replays launch the same kernels)
    c0 = w.pool.launch_count()
    w.corun_step(x, y, tp, td)
    torch.cuda.synchronize(dev)
    per_step = w.pool.launch_count() - c0
    # ---- the timed region: K replays of the captured co-run step at the best schedule
    step = run.capture(lambda: w.corun_step(x, y, tp, td))
    for _ in range(W):
        step()
    w.spans.zero_()
    with ClockSampler(nvml_id(dev)) as clk:
        t = time_steps(step, args.steps, dev, barrier)
    t = max_over_ranks(t, ws, dev)
    ks = w.kernel_stats()
    launches = per_step * args.steps
    value = w.tokens_per_step() * args.steps / t
    ms_step = t / args.steps * 1e3
    n_p, n_d = w.pool.sm_budgets()
    if args.tp_mode == "pipelined" and ws > 1 and args.gather == "nccl":
        n_p, n_d = w._budget(0, "p"), w._budget(0, "d")
    rec = phase_record(w, n_p, n_d, t / args.steps, ks, pk)
    dec_ms, pre_ms = ks["decode"]["ms"], ks["prefill"]["ms"]
    roof_dec = {"kernel": "decode_bf16_kernel / decode_pair_kernel (split-K paged decode)",
                "bound": "hbm", "achieved": rec["decode_gbs"], "peak": pk["hbm"], "unit": "GB/s",
                "frac": rec["decode_frac"], "peak_kind": pk["kind"],
                "traffic": ncu_traffic("decode_bf16_kernel"),
                "traffic_unit": "DRAM bytes per launch (ncu --set full)",
                "algorithmic_bytes_per_launch": w.decode_bytes_per_launch(),
                "avg_launch_ms": dec_ms, "launches_timed": ks["decode"]["launches"],
                "timing": "device launch spans (first CTA entry -> last CTA exit) over the K "
                          "timed graph replays", "sm_budget": n_d}
    roof_pre = {"kernel": "prefill_tc_kernel tcgen05 causal GQA (K/V pool write fused)",
                "bound": "tensor", "achieved": rec["prefill_tflops"],
                "peak": pk["burst"] * n_p / w.pool.num_sms, "unit": "TFLOP/s",
                "frac": rec["prefill_frac_share_burst"],
                "frac_whole_gpu_burst": rec["prefill_frac"],
                "frac_share_scaled_burst": rec["prefill_frac_share_burst"],
                "frac_share_scaled_sustained": rec["prefill_frac_share_sustained"],
                "peak_kind": f"{pk['kind']} burst x n_p/148 (the kernel runs at full clocks on "
                             f"its partition; sustained {pk['sustained']} is a power-limited "
                             f"full-chip rate)",
                "traffic": ncu_traffic("prefill_tc_kernel"),
                "traffic_unit": "DRAM bytes per launch (ncu --set full)",
                "algorithmic_flops_per_launch": w.prefill_flops_per_launch(),
                "avg_launch_ms": pre_ms, "launches_timed": ks["prefill"]["launches"],
                "sm_budget": n_p}
    dominant = "decode" if dec_ms >= pre_ms else "prefill"
    consistency = {"decode_kernels_ms_per_step": dec_ms * w.L,
                   "prefill_kernels_ms_per_step": pre_ms * w.L, "ms_per_step": ms_step,
                   "ok": max(dec_ms, pre_ms) * w.L <= ms_step * 1.001}
    step_bytes = w.L * (w.decode_bytes_per_launch() + w.prefill_bytes_per_launch())
    step_gbs = step_bytes / (t / args.steps) / 1e9
    roof_step = {"bound": "hbm", "achieved": step_gbs, "peak": pk["hbm"], "unit": "GB/s",
                 "frac": step_gbs / pk["hbm"], "peak_kind": pk["kind"],
                 "algorithmic_bytes_per_step": step_bytes}
    corun_streams = {"prefill_stream_ms": ks["prefill"]["stream_ms"],
                     "decode_stream_ms": ks["decode"]["stream_ms"],
                     "overlap": rec.get("overlap"),
                     "note": "first-kernel start to last-kernel end per stream, last replay"}
    # ---- each phase alone on all SMs (graph replay) and the time-sliced / (100,100) baselines
    nsm = w.pool.num_sms
    iso = {"sm_budget": nsm}
    for ph, fn in (("prefill", lambda: w.phase_prefill(nsm, stream=torch.cuda.current_stream(dev))),
                   ("decode", lambda: w.phase_decode(nsm, stream=torch.cuda.current_stream(dev)))):
        ti, kk = run.time(run.capture(fn), 3)
        kk = w.kernel_stats(order=(ph,))[ph]
        if ph == "prefill":
            a = w.prefill_flops_per_launch() / (kk["ms"] / 1e3) / 1e12
            iso[ph] = {"achieved": a, "unit": "TFLOP/s", "peak": pk["burst"], "frac": a / pk["burst"],
                       "frac_sustained": a / pk["sustained"], "ms_per_launch": kk["ms"],
                       "ms_per_phase_step": ti * 1e3}
        else:
            a = w.decode_bytes_per_launch() / (kk["ms"] / 1e3) / 1e9
            iso[ph] = {"achieved": a, "unit": "GB/s", "peak": pk["hbm"], "frac": a / pk["hbm"],
                       "ms_per_launch": kk["ms"], "ms_per_phase_step": ti * 1e3}
    extra = {}
    if args.extra:
        ts = run.time(run.capture(w.serial_step), 3)[0]
        tu = run.time(run.capture(w.uncontrolled_step), 3)[0]
        extra = {"serial_ms": ts * 1e3, "uncontrolled_100_100_ms": tu * 1e3, "corun_ms": ms_step,
                 "speedup_vs_serial": ts / (t / args.steps),
                 "speedup_vs_100_100": tu / (t / args.steps)}
    # the calibrated co-run keeps the GPU busy for ~120 ms: after the short graph-replayed
    # baselines above, so its sustained load does not lower their clocks
    cal = None
    if ws == 1:
        cal = calibrated_corun(w, x, y, pk, ks["prefill"]["stream_ms"], ks["decode"]["stream_ms"])
    w.pool.set_spans(None)
    e2e = None
    if not args.no_e2e:
        # pinned host buffers on the GPU's own NUMA node (first touch by a local CPU) and the
        # launching thread there too: a remote node would cap the host <-> device copies
        local = gpu_local_cpus(dev)
        saved = os.sched_getaffinity(0)
        if local:
            try:
                os.sched_setaffinity(0, local)
            except OSError:
                local = None
        ee = E2E(w)
        for _ in range(2):
            ee.step(x, y, tp, td)
        ne = max(2, min(args.steps, 5))
        te = max_over_ranks(time_steps(lambda: ee.step(x, y, tp, td), ne, dev, barrier) / ne, ws, dev)
        e2e = {"value": w.tokens_per_step() / te, "unit": "tokens/s",
               "h2d_bytes_per_step": ee.h2d, "d2h_bytes_per_step": ee.d2h,
               "ms_per_step": te * 1e3,
               "pcie_gbs_effective": (ee.h2d + ee.d2h) / te / 1e9,
               "host_cpus_gpu_local": len(local) if local else None}
        del ee
        try:
            os.sched_setaffinity(0, saved)
        except OSError:
            pass
    dp = None
    if ws > 1 and not args.no_dp:
        # DP-replica reference (SURVEY §8(e) "Replicas"): every rank runs the TP-1 workload
        # on its own GPU, no collective; ideal weak scaling
        full = Workload(shape, 1, dev, seed=1020 + rank)
        rr = Runner(full, dev, barrier, not args.no_graph, ws)
        t_dp = rr.time(rr.capture(lambda: full.corun_step(x, y, tp, td)), 5)[0]
        dp = {"value": ws * full.tokens_per_step() / t_dp, "unit": "tokens/s",
              "ms_per_step": t_dp * 1e3, "scaling": "weak", "replicas": ws,
              "split": {"x": x, "y": y}, "cuda_graph": rr.use_graph}
        del rr, full
    graph_used, graph_error = run.use_graph, run.graph_error
    secondary = {}
    if ws == 1 and not args.no_secondary:
        del run, step
        for name, fn in (("block16", secondary_block16), ("cfg3_llama70b", secondary_cfg3),
                         ("cfg4_longctx", secondary_cfg4), ("cfg5_mla", secondary_cfg5),
                         ("cfg5_mla_expanded", secondary_cfg5_expanded),
                         ("fp8_kv", secondary_fp8)):
            try:
                secondary[name] = fn(args, dev, pk)
            except Exception as e:  # a secondary field never voids the headline
                secondary[name] = {"error": repr(e)[:300]}
            torch.cuda.synchronize(dev)
            torch.cuda.empty_cache()
    sustained = None
    if ws == 1 and args.sustained > 0:
        # the same step replayed back to back for ~args.sustained seconds, after everything
        # else: a B200 at this load reaches its 1000 W cap within ~0.2 s and lowers the SM
        # clock (sw_power_cap), so this is the power-capped rate a long-running job sees; the
        # headline's K steps mostly run before the cap engages (their clocks say which)
        rs = Runner(w, dev, None, not args.no_graph, 1)
        st_ = rs.capture(lambda: w.corun_step(x, y, tp, td))
        n_win = 10
        per_win = max(1, int(round(args.sustained / n_win / (ms_step / 1e3))))
        wins = []
        with ClockSampler(nvml_id(dev), period_s=0.02) as ck:
            for _ in range(n_win):
                wins.append(time_steps(st_, per_win, dev) / per_win * 1e3)
        late = wins[n_win // 2:]
        sustained = {"seconds": round(sum(wins) * per_win / 1e3, 3), "steps": n_win * per_win,
                     "ms_per_step_windows": [round(v, 4) for v in wins],
                     "ms_per_step_last_half": statistics.mean(late),
                     "tokens_per_s_last_half": w.tokens_per_step() / (statistics.mean(late) / 1e3),
                     "split": {"x": x, "y": y}, "clocks": ck.summary(),
                     "note": "not the headline: the same captured step, back to back after all "
                             "other fields; shows the power-capped steady state"}
        # the other re-timed schedules under the same (capped) load: the split that is best
        # at full clocks need not be best at the capped clock (power)
        others = []
        for r in reselect:
            if (r["x"], r["tail_p"], r["tail_d"]) == (x, tp, td):
                continue
            so = rs.capture(lambda r=r: w.corun_step(r["x"], 100 - r["x"], r["tail_p"], r["tail_d"]))
            n_o = max(1, int(round(0.3 / (ms_step / 1e3))))
            t_o = time_steps(so, n_o, dev) / n_o
            others.append({"x": r["x"], "tail_p": r["tail_p"], "tail_d": r["tail_d"],
                           "ms_per_step": t_o * 1e3, "tokens_per_s": w.tokens_per_step() / t_o})
            del so
        sustained["other_splits"] = others
        del rs, st_
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(shape)
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": W,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {**workload_config(shape, ws, args.gather, args.tp_mode),
                       "split": {"x": x, "y": y, "n_prefill_sms": n_p, "n_decode_sms": n_d,
                                 "tail_p": tp, "tail_d": td,
                                 "schedule": "pure split" if not (tp or td) else
                                 f"split, then the last {tp or td} {'prefill' if tp else 'decode'} "
                                 f"layers on all {w.pool.num_sms} SMs once the other worker is "
                                 f"done (R30)"}},
            "best_pure_split": best_pure,
            "split_reselect": reselect,
            "roofline": roof_dec if dominant == "decode" else roof_pre,
            "roofline_decode": roof_dec, "roofline_prefill": roof_pre, "roofline_step": roof_step,
            "kernel_time_check": consistency,
            "corun_streams": corun_streams, "corun_calibrated": cal, "isolated_full_chip": iso,
            "decode_tokens_per_s": w.B * args.steps / t,
            "prefill_tokens_per_s": w.C * args.steps / t,
            "best_target_split": tgt,
            "target_met": bool(tgt and tgt["target_score"] >= 1.0),
            "sweep": sweep, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
            "gpu_launches": launches, "cuda_graph": graph_used, "graph_error": graph_error,
            "dp_replicas": dp, "extra": extra or None, "sustained": sustained, **secondary,
        }
        if ws > 1:
            line["tp"] = {"mode": args.tp_mode, "gather": args.gather,
                          "nccl_max_ctas": args.nccl_max_ctas}
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
