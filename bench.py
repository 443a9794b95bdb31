#!/usr/bin/env python
"""bench.py — co-run prefill + decode attention on one unified paged KV pool.

Workload (BASELINE.json configs[1], "Llama-3-8B attention shapes bf16"): 32 layers,
32 q / 8 kv heads, d = 128, block 16; per step (one co-run iteration, SURVEY §8(a)
rows a1-a9):
  stream P (prefill worker): alloc 128 blocks for the prefill request, then for each
    layer semipd_prefill_attn on one 2048-token chunk (P = 0; K/V write + causal GQA
    attention), then free the request's blocks;
  stream D (decode worker), concurrently: for each layer semipd_decode_attn on 64
    requests at ctx 2048 (K/V append + split-K paged attention).
The two persistent grids are capped to the (x, y) SM partition.  A short
sweep over x picks the best split during warm-up; the K timed steps run at it.

metric: attention-stack tokens/s = (2048 prefill + 64 decode tokens) x steps / time
(each token through all 32 layers).  value = device time (CUDA events, max over
ranks), inputs resident in HBM; e2e = the same through the public API with pinned
host inputs copied in and outputs copied out every step.

Multi-GPU (torchrun, N ranks): tensor parallel by KV head (Hq/N, Hkv/N per rank,
own pool shard), NCCL all-gather of head-major outputs per layer on a per-phase
process group, strong scaling.  --impl reference times the fp64 oracle
(oracle/, the reference arm of this tier) on the host cores.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import statistics
import subprocess
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="semipd", choices=["semipd", "reference"])
    ap.add_argument("--model", default="llama3-8b", choices=list(MODELS))
    ap.add_argument("--split", type=float, default=None, help="prefill SM percent x (y = 100-x)")
    ap.add_argument("--sweep", default="25,30,35,40,45,50,60")
    ap.add_argument("--block-size", type=int, default=64,
                    help="KV page size in tokens (64: one 16 KiB TMA box per (block, head) "
                         "page on B200; 16 is supported but TMA-per-box bound)")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "peer", "fused"],
                    help="TP head all-gather: NCCL all_gather (CTAs); peer = copy-engine pushes "
                         "over IPC-mapped peer memory with stream-memop flags (no SMs); fused = "
                         "both kernels store their output into the peers' buffers from the "
                         "epilogue")
    ap.add_argument("--peer-graph", action="store_true",
                    help="N > 1 with --gather peer: replay the co-run step as a CUDA graph")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every kernel from Python instead of replaying a CUDA graph")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--extra", action="store_true", default=True,
                    help="serial / (100,100) baselines (default on: the paper's spatial-vs-temporal claim)")
    ap.add_argument("--no-extra", dest="extra", action="store_false")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def ncu_traffic(kernel: str):
    """dram read + write bytes per launch of `kernel` from the newest committed ncu capture
    (profiles/r*_ncu_traffic.json, written from an `ncu --set full` run of the same shapes)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_traffic.json")))
    if not files:
        return None
    try:
        with open(files[-1]) as f:
            d = json.load(f)[kernel]
        return int(d["dram_read_bytes"]) + int(d["dram_write_bytes"])
    except Exception:
        return None


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(
            d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


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
                     pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
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
        reasons = sorted({name for _, rs in self.rows for name, attr in self.REASONS.items()
                          if rs & getattr(nv, attr)})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml, 5 ms, child process"}


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- workload
class Workload:
    """Pool + resident inputs for one rank (head shard under TP)."""

    def __init__(self, shape: synth.AttnShape, tp: int, dev: torch.device, seed: int = 1020,
                 gather: str = "nccl"):
        from paper_2504_19867_b200 import KVPool, PoolConfig
        self.full = shape
        self.shape = synth.shard_heads(shape, tp) if tp > 1 else shape
        self.tp, self.dev = tp, dev
        s = self.shape
        self.L = s.num_layers
        self.B, self.ctx, self.C = DECODE_BATCH, DECODE_CTX, PREFILL_TOKENS
        bs = s.block_size
        self.nb_dec = self.ctx // bs + 1                 # slot ctx needs block ctx // bs
        self.nb_pre = -(-self.C // bs)
        n_blocks = self.B * self.nb_dec + self.nb_pre + 64
        self.cfg = PoolConfig(num_layers=self.L, num_blocks=n_blocks, block_size=bs,
                              num_kv_heads=s.num_kv_heads, head_dim_k=s.head_dim_k,
                              head_dim_v=s.head_dim_v, max_reqs=self.B + 2,
                              max_blocks_per_req=self.nb_dec + 8, dtype=s.dtype)
        self.pool = KVPool(self.cfg, dev)
        i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
        self.rid_dec = i32(list(range(self.B)))
        self.ctx_lens = i32([self.ctx] * self.B)
        self.pool.alloc_blocks(self.rid_dec, i32([self.nb_dec] * self.B))
        self.rid_pre = i32([self.B])
        self.nblk_pre = i32([self.nb_pre])
        self.cu = i32([0, self.C])
        self.prefix = i32([0])
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        # cached context: random bf16 in every layer's pool (distinct memory per layer,
        # so the per-step decode working set (L x 537 MB) is far larger than L2)
        for l in range(self.L):
            K, V, _, _ = self.pool.views(l)
            K.normal_(generator=g)
            V.normal_(generator=g)
        Hq, Hkv, d = s.num_q_heads, s.num_kv_heads, s.head_dim_k
        mk = lambda *shp: torch.randn(*shp, generator=g, device=dev, dtype=torch.float32).to(s.dtype)  # noqa: E731
        self.qp = [mk(self.C, Hq, d) for _ in range(self.L)]
        self.kp = [mk(self.C, Hkv, d) for _ in range(self.L)]
        self.vp = [mk(self.C, Hkv, d) for _ in range(self.L)]
        self.qd = [mk(self.B, Hq, d) for _ in range(self.L)]
        self.kd = [mk(self.B, Hkv, d) for _ in range(self.L)]
        self.vd = [mk(self.B, Hkv, d) for _ in range(self.L)]
        hm = tp > 1
        self.op = [torch.empty((Hq, self.C, d) if hm else (self.C, Hq, d), dtype=s.dtype,
                               device=dev) for _ in range(self.L)]
        self.od = [torch.empty((Hq, self.B, d) if hm else (self.B, Hq, d), dtype=s.dtype,
                               device=dev) for _ in range(self.L)]
        self.ws = self.pool.new_decode_workspace(self.B, Hq, self.ctx)
        self.scale = s.softmax_scale
        self.sP = torch.cuda.Stream(device=dev)
        self.sD = torch.cuda.Stream(device=dev)
        self.pg_p = self.pg_d = None
        self.peer_p = self.peer_d = None
        self.fused_d = self.fused_p = False
        self.gath_p = self.gath_d = None
        if tp > 1:
            from paper_2504_19867_b200 import tp as tpmod
            groups = tpmod.PhaseGroups.create(  # one communicator per phase
                backend=os.environ.get("SPD_BENCH_BACKEND", "nccl"))
            self.pg_p, self.pg_d = groups.prefill, groups.decode
            self.gath_p = torch.empty((self.full.num_q_heads, self.C, d), dtype=s.dtype, device=dev)
            self.gath_d = torch.empty((self.full.num_q_heads, self.B, d), dtype=s.dtype, device=dev)
            if gather in ("peer", "fused"):  # copy engines + stream memops instead of NCCL CTAs
                self.peer_p = tpmod.PeerGather(self.gath_p.shape, s.dtype, self.pg_p, dev)
                self.peer_d = tpmod.PeerGather(self.gath_d.shape, s.dtype, self.pg_d, dev)
            if gather == "fused":  # both epilogues store straight into every rank's buffer
                self.fused_d = self.fused_p = True
                self.pool.set_decode_peers(self.peer_d.peer_shard_ptrs())
                self.od = [self.peer_d.local_view() for _ in range(self.L)]
                self.pool.set_prefill_peers(self.peer_p.peer_shard_ptrs())
                self.op = [self.peer_p.local_view() for _ in range(self.L)]
        # per-launch timing events (decode kernel on stream D, prefill call on stream P)
        self.ev_d = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                     for _ in range(self.L)]
        self.ev_p = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                     for _ in range(self.L)]

    # algorithmic work: count unmasked pairs and K/V bytes once
    def decode_bytes_per_launch(self) -> float:
        s = self.shape
        eb = 2
        kv = self.B * (self.ctx + 1) * s.num_kv_heads * (s.head_dim_k + s.head_dim_v) * eb
        io = self.B * s.num_q_heads * (s.head_dim_k + s.head_dim_v) * eb  # q in, o out
        return float(kv + io)

    def prefill_bytes_per_launch(self) -> float:
        # HBM bytes the prefill launch must move at P = 0: q in, o out, k_new / v_new in and
        # their copy into the pool pages (a3, fused)
        s = self.shape
        eb = 2
        qo = self.C * s.num_q_heads * (s.head_dim_k + s.head_dim_v) * eb
        kv = self.C * s.num_kv_heads * (s.head_dim_k + s.head_dim_v) * eb
        return float(qo + 2 * kv)

    def prefill_flops_per_launch(self) -> float:
        s = self.shape
        pairs = self.C * (self.C + 1) / 2
        return 2.0 * s.num_q_heads * (s.head_dim_k + s.head_dim_v) * pairs

    # TP > 1: the head all-gather of layer l's head-major output on the phase stream s
    # (one communicator per phase); a no-op at TP = 1
    def pre_p(self, l, s):  # fused gather: every peer is done reading before the stores
        if self.fused_p:
            self.peer_p.handshake(0, stream=s)

    def gather_p(self, l, s):
        if self.fused_p:  # the kernel already stored; wait until every peer's stores landed
            self.peer_p.handshake(1, stream=s)
        elif self.tp > 1:
            from paper_2504_19867_b200 import tp as tpmod
            if self.peer_p is not None:
                self.peer_p(self.op[l], stream=s)
            else:
                tpmod.gather_heads(self.op[l], self.gath_p, self.pg_p)

    def pre_d(self, l, s):  # fused gather: every peer is done reading before the stores
        if self.fused_d:
            self.peer_d.handshake(0, stream=s)

    def gather_d(self, l, s):
        if self.fused_d:  # the kernel already stored; wait until every peer's stores landed
            self.peer_d.handshake(1, stream=s)
        elif self.tp > 1:
            from paper_2504_19867_b200 import tp as tpmod
            if self.peer_d is not None:
                self.peer_d(self.od[l], stream=s)
            else:
                tpmod.gather_heads(self.od[l], self.gath_d, self.pg_d)

    def phase_prefill(self, budget, timed=False, stream=None):
        s = stream or self.sP
        p = self.pool
        with torch.cuda.stream(s):
            p.alloc_blocks(self.rid_pre, self.nblk_pre, None, stream=s)
            for l in range(self.L):
                self.pre_p(l, s)
                if timed:
                    self.ev_p[l][0].record(s)
                p.prefill_attn(l, self.qp[l], self.kp[l], self.vp[l], self.cu, self.rid_pre,
                               self.prefix, self.C, self.C, self.scale, self.op[l],
                               out_head_major=self.tp > 1, sm_budget=budget, stream=s)
                if timed:
                    self.ev_p[l][1].record(s)
                self.gather_p(l, s)
            p.free_blocks(self.rid_pre, None, stream=s)

    def phase_decode(self, budget, timed=False, stream=None):
        s = stream or self.sD
        p = self.pool
        with torch.cuda.stream(s):
            for l in range(self.L):
                self.pre_d(l, s)
                if timed:
                    self.ev_d[l][0].record(s)
                p.decode_attn(l, self.qd[l], self.kd[l], self.vd[l], self.rid_dec, self.ctx_lens,
                              self.ctx, self.scale, self.od[l], self.ws,
                              out_head_major=self.tp > 1, sm_budget=budget, stream=s)
                if timed:
                    self.ev_d[l][1].record(s)
                self.gather_d(l, s)

    def corun_step(self, x, y, timed=False):
        """One co-run iteration: both workers concurrently at budgets from (x, y)."""
        main = torch.cuda.current_stream(self.dev)
        self.pool.set_partition(x, y)
        self.sP.wait_stream(main)
        self.sD.wait_stream(main)
        self.phase_prefill(0, timed)
        self.phase_decode(0, timed)
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


# ----------------------------------------------------------------------------- e2e
class E2E:
    """Same step through the public API with pinned host inputs/outputs: every step copies
    its inputs host -> device and its outputs device -> host inside the timed region.
    The copies run on their own streams, per layer, so the PCIe transfers pipeline with
    the attention kernels and H2D overlaps D2H (the copy engines are independent):
      H2D stream: layer l's prefill q / k / v and decode q / k / v, then an event each;
      stream P / D: wait for layer l's inputs, run the kernel, record an event;
      D2H stream: wait for layer l's outputs, copy them out.
    Device buffers are per layer and the step ends with the main stream joining all four
    streams, so nothing is overwritten while still in use."""

    def __init__(self, w: Workload):
        self.w = w
        pin = lambda t: t.cpu().pin_memory()  # noqa: E731
        self.h_qp = [pin(t) for t in w.qp]
        self.h_kp = [pin(t) for t in w.kp]
        self.h_vp = [pin(t) for t in w.vp]
        self.h_qd = [pin(t) for t in w.qd]
        self.h_kd = [pin(t) for t in w.kd]
        self.h_vd = [pin(t) for t in w.vd]
        self.h_op = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in w.op]
        self.h_od = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in w.od]
        self.h2d = sum(t.numel() * t.element_size() for lst in
                       (self.h_qp, self.h_kp, self.h_vp, self.h_qd, self.h_kd, self.h_vd) for t in lst)
        self.d2h = sum(t.numel() * t.element_size() for lst in (self.h_op, self.h_od) for t in lst)
        self.s_in = torch.cuda.Stream(w.dev)
        self.s_out = torch.cuda.Stream(w.dev)
        ev = lambda: [torch.cuda.Event() for _ in range(w.L)]  # noqa: E731
        self.in_p, self.in_d, self.out_p, self.out_d = ev(), ev(), ev(), ev()

    def step(self, x, y):
        w = self.w
        main = torch.cuda.current_stream(w.dev)
        w.pool.set_partition(x, y)
        for s in (self.s_in, self.s_out, w.sP, w.sD):
            s.wait_stream(main)
        with torch.cuda.stream(self.s_in):
            for l in range(w.L):
                w.qd[l].copy_(self.h_qd[l], non_blocking=True)
                w.kd[l].copy_(self.h_kd[l], non_blocking=True)
                w.vd[l].copy_(self.h_vd[l], non_blocking=True)
                self.in_d[l].record(self.s_in)
                w.qp[l].copy_(self.h_qp[l], non_blocking=True)
                w.kp[l].copy_(self.h_kp[l], non_blocking=True)
                w.vp[l].copy_(self.h_vp[l], non_blocking=True)
                self.in_p[l].record(self.s_in)
        with torch.cuda.stream(w.sP):
            w.pool.alloc_blocks(w.rid_pre, w.nblk_pre, None, stream=w.sP)
            for l in range(w.L):
                w.sP.wait_event(self.in_p[l])
                w.pre_p(l, w.sP)
                w.pool.prefill_attn(l, w.qp[l], w.kp[l], w.vp[l], w.cu, w.rid_pre, w.prefix, w.C,
                                    w.C, w.scale, w.op[l], out_head_major=w.tp > 1, stream=w.sP)
                w.gather_p(l, w.sP)  # TP > 1: same exchange step as the device-timed path
                self.out_p[l].record(w.sP)
            w.pool.free_blocks(w.rid_pre, None, stream=w.sP)
        with torch.cuda.stream(w.sD):
            for l in range(w.L):
                w.sD.wait_event(self.in_d[l])
                w.pre_d(l, w.sD)
                w.pool.decode_attn(l, w.qd[l], w.kd[l], w.vd[l], w.rid_dec, w.ctx_lens, w.ctx,
                                   w.scale, w.od[l], w.ws, out_head_major=w.tp > 1, stream=w.sD)
                w.gather_d(l, w.sD)
                self.out_d[l].record(w.sD)
        with torch.cuda.stream(self.s_out):
            for l in range(w.L):
                self.s_out.wait_event(self.out_d[l])
                self.h_od[l].copy_(w.od[l], non_blocking=True)
                self.s_out.wait_event(self.out_p[l])
                self.h_op[l].copy_(w.op[l], non_blocking=True)
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


def workload_config(shape: synth.AttnShape, ws: int, gather: str = "nccl") -> dict:
    """The `config` both arms print (the reference arm runs the same workload)."""
    decode_gb = shape.num_layers * (DECODE_BATCH * (DECODE_CTX + 1) * shape.num_kv_heads * 2 * 128 * 2) / 1e9
    return {"workload": f"{shape.name} attention (Hq {shape.num_q_heads}, Hkv {shape.num_kv_heads}, "
                        f"d 128, bs {shape.block_size}, {shape.num_layers} layers): decode B={DECODE_BATCH} "
                        f"ctx={DECODE_CTX} + prefill chunk {PREFILL_TOKENS} (P=0), co-run",
            "parallelism": (f"tp{ws} (KV-head shards, "
                            + {"peer": "copy-engine peer all-gather)",
                               "fused": "peer stores from the decode / prefill epilogues)"}
                            .get(gather, "NCCL all-gather)")
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
        "impl": "reference", "metric": "co-run prefill+decode attention tokens/s (32-layer stack)",
        "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * (PREFILL_TOKENS + DECODE_BATCH) / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(shape, 1),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": elapsed,
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- main
def main():
    args = parse()
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
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        barrier = lambda: dist.barrier()  # noqa: E731
    shape = dataclasses.replace(MODELS[args.model], block_size=args.block_size)
    w = Workload(shape, ws, dev, gather=args.gather)
    hbm_peak, bf16_peak, bf16_sus, peak_kind = peaks()
    W = max(3, args.warmup)
    splits = [float(x) for x in args.sweep.split(",")] if args.split is None else [args.split]
    # warm-up + split sweep (1 timed step per split, not part of the reported number)
    for _ in range(2):
        w.corun_step(50, 50)
    sweep = []

    # N > 1 runs eagerly.  The peer gather is graph-safe (tests/test_gpu_peer_gather.py replays
    # a captured gather), but with two ranks time-slicing one GPU the replayed step was 7x
    # slower than eager (138 vs 19 ms), so graph replay for N > 1 stays opt-in (--peer-graph)
    use_graph = not args.no_graph and (ws == 1 or (args.gather == "peer" and args.peer_graph))

    def capture(x):
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            w.corun_step(x, 100 - x)
        g.replay()
        torch.cuda.synchronize(dev)
        return g

    def measure(x):
        if use_graph:
            g = capture(x)
            t = time_steps(g.replay, 3, dev, barrier) / 3
        else:
            t = time_steps(lambda: w.corun_step(x, 100 - x), 2, dev, barrier) / 2
        if ws > 1:
            tt = torch.tensor([t], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            t = float(tt.item())
        sweep.append({"x": x, "y": 100 - x, "n_p": w.pool.sm_budgets()[0],
                      "n_d": w.pool.sm_budgets()[1],
                      "tokens_per_s": (PREFILL_TOKENS + DECODE_BATCH) / t, "ms": t * 1e3})

    for x in splits:
        measure(x)
    if args.split is None:  # refine around the best coarse split (+-2.5 % = ~4 SMs)
        x0 = max(sweep, key=lambda r: r["tokens_per_s"])["x"]
        for x in (x0 - 2.5, x0 + 2.5):
            if 0 < x < 100 and all(abs(r["x"] - x) > 1e-6 for r in sweep):
                measure(x)
    best = max(sweep, key=lambda r: r["tokens_per_s"])
    x, y = best["x"], best["y"]
    for _ in range(W):
        w.corun_step(x, y)
    # the co-run step (both streams, alloc -> 32 layers x 2 kernels -> free) is captured once
    # into a CUDA graph and replayed: no per-kernel launch gaps from the Python loop
    graph = capture(x) if use_graph else None
    if graph is not None:
        graph.replay()
        torch.cuda.synchronize(dev)
    # ---- timed region
    per_step = [0]
    with ClockSampler(nvml_id(dev)) as clk:
        # the last timed step runs eagerly with per-launch CUDA events (the roofline's kernel
        # times; an event pair between back-to-back kernels costs ~3 us, so only one step)
        k_step = [0]

        def step():
            k_step[0] += 1
            if k_step[0] == args.steps or graph is None:
                c0 = w.pool.launch_count()
                w.corun_step(x, y, timed=k_step[0] == args.steps)
                per_step[0] = w.pool.launch_count() - c0
            else:
                graph.replay()

        t = time_steps(step, args.steps, dev, barrier)
    launches = per_step[0] * args.steps  # the graph replays the same launches
    if ws > 1:
        tt = torch.tensor([t], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
    tokens = (PREFILL_TOKENS + DECODE_BATCH) * args.steps
    value = tokens / t
    # per-launch kernel times (last timed step's events)
    dec_ms = statistics.mean(a.elapsed_time(b) for a, b in w.ev_d)
    pre_ms = statistics.mean(a.elapsed_time(b) for a, b in w.ev_p)
    # co-run overlap of the two streams in that step: each stream's span
    # from its first kernel start to its last kernel end; overlap = min / max span
    span_p = w.ev_p[0][0].elapsed_time(w.ev_p[-1][1])
    span_d = w.ev_d[0][0].elapsed_time(w.ev_d[-1][1])
    corun_overlap = {"prefill_stream_ms": span_p, "decode_stream_ms": span_d,
                     "overlap": min(span_p, span_d) / max(span_p, span_d)}
    dec_gbs = w.decode_bytes_per_launch() / (dec_ms / 1e3) / 1e9
    pre_tfs = w.prefill_flops_per_launch() / (pre_ms / 1e3) / 1e12
    n_p, n_d = w.pool.sm_budgets()
    dec_total, pre_total = dec_ms * w.L, pre_ms * w.L
    dominant = "decode" if dec_total >= pre_total else "prefill"
    roof_dec = {"kernel": "decode_bf16_kernel (split-K paged decode)", "bound": "hbm",
                "achieved": dec_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": dec_gbs / hbm_peak,
                "peak_kind": peak_kind, "traffic": ncu_traffic("decode_bf16_kernel"),
                "traffic_unit": "DRAM bytes per launch (ncu)",
                "algorithmic_bytes_per_launch": w.decode_bytes_per_launch(),
                "avg_launch_ms": dec_ms, "sm_budget": n_d}
    share = n_p / w.pool.num_sms
    roof_pre = {"kernel": "prefill_tc_kernel tcgen05 causal GQA (K/V pool write fused)", "bound": "tensor",
                "achieved": pre_tfs, "peak": bf16_sus, "unit": "TFLOP/s",
                "frac": pre_tfs / bf16_sus, "frac_share_scaled": pre_tfs / (bf16_sus * share),
                "peak_kind": f"{peak_kind} sustained", "traffic": ncu_traffic("prefill_tc_kernel"),
                "traffic_unit": "DRAM bytes per launch (ncu)",
                "algorithmic_flops_per_launch": w.prefill_flops_per_launch(),
                "avg_launch_ms": pre_ms, "sm_budget": n_p}
    # whole co-run step against HBM: both phases' algorithmic bytes per step / step time.
    # Decode streams the KV cache and the prefill moves q / o / chunk K/V, all through the one
    # shared HBM, so this bounds the step however the SMs are split
    step_bytes = w.L * (w.decode_bytes_per_launch() + w.prefill_bytes_per_launch())
    step_gbs = step_bytes / (t / args.steps) / 1e9
    roof_step = {"bound": "hbm", "achieved": step_gbs, "peak": hbm_peak, "unit": "GB/s",
                 "frac": step_gbs / hbm_peak, "peak_kind": peak_kind,
                 "algorithmic_bytes_per_step": step_bytes}
    def graphed(fn):  # the baselines get the same CUDA-graph replay as the co-run step
        if not use_graph:
            return fn
        fn()
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize(dev)
        return g.replay

    # each phase alone on the whole GPU (148 SMs): the kernels' full-chip roofline fractions,
    # next to the co-run ones above (32 launches + the phase's alloc / free, graph replay)
    # (the stream is looked up at call time: under graph capture it is the capture stream)
    nsm = w.pool.num_sms
    t_pi = time_steps(graphed(lambda: w.phase_prefill(nsm, stream=torch.cuda.current_stream(dev))),
                      3, dev, barrier) / 3
    t_di = time_steps(graphed(lambda: w.phase_decode(nsm, stream=torch.cuda.current_stream(dev))),
                      3, dev, barrier) / 3
    pre_iso = w.prefill_flops_per_launch() * w.L / t_pi / 1e12
    dec_iso = w.decode_bytes_per_launch() * w.L / t_di / 1e9
    isolated = {"sm_budget": nsm,
                "prefill": {"achieved": pre_iso, "unit": "TFLOP/s", "peak": bf16_sus,
                            "frac": pre_iso / bf16_sus, "ms_per_launch": t_pi / w.L * 1e3},
                "decode": {"achieved": dec_iso, "unit": "GB/s", "peak": hbm_peak,
                           "frac": dec_iso / hbm_peak, "ms_per_launch": t_di / w.L * 1e3},
                "note": "per phase, all SMs, 32-layer graph replay incl. the phase's alloc/free"}
    extra = {}
    if args.extra:

        ts = time_steps(graphed(w.serial_step), 3, dev, barrier) / 3
        tu = time_steps(graphed(w.uncontrolled_step), 3, dev, barrier) / 3
        extra = {"serial_ms": ts * 1e3, "uncontrolled_100_100_ms": tu * 1e3,
                 "corun_ms": t / args.steps * 1e3,
                 "speedup_vs_serial": ts / (t / args.steps),
                 "speedup_vs_100_100": tu / (t / args.steps)}
    e2e = None
    if not args.no_e2e:
        ee = E2E(w)
        for _ in range(2):
            ee.step(x, y)
        te = time_steps(lambda: ee.step(x, y), max(2, min(args.steps, 5)), dev, barrier)
        te /= max(2, min(args.steps, 5))
        if ws > 1:
            tt = torch.tensor([te], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": (PREFILL_TOKENS + DECODE_BATCH) / te, "unit": "tokens/s",
               "h2d_bytes_per_step": ee.h2d, "d2h_bytes_per_step": ee.d2h,
               "ms_per_step": te * 1e3}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        v, sample, _ = oracle_sample_rate(shape, threads)
        cpu = {"value": v, "unit": "tokens/s", "cores": threads, "kind": "oracle",
               "sample": sample}
    if rank == 0:
        line = {
            "metric": "co-run prefill+decode attention tokens/s (32-layer stack)",
            "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": W,
            "ms_per_step": t / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {**workload_config(shape, ws, args.gather),
                       "split": {"x": x, "y": y, "n_prefill_sms": n_p, "n_decode_sms": n_d}},
            "roofline": roof_dec if dominant == "decode" else roof_pre,
            "roofline_decode": roof_dec, "roofline_prefill": roof_pre, "roofline_step": roof_step,
            "corun_streams": corun_overlap, "isolated_full_chip": isolated,
            "decode_tokens_per_s": DECODE_BATCH * args.steps / t,
            "prefill_tokens_per_s": PREFILL_TOKENS * args.steps / t,
            "sweep": sweep, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
            "gpu_launches": launches, "cuda_graph": graph is not None, "extra": extra or None,
        }
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
