"""One-GPU emulation of the copy-engine peer all-gather at TP = 2/4/8 (semipd_peer_gather).

Every emulated rank is a stream of this process; its gathered buffer and flag array are
plain device allocations, so the C ABI call is exactly the multi-GPU one with local
pointers (the copies move HBM -> HBM on the copy engines instead of over NVLink).  Checks
the gathered bytes, then times one gather round (all ranks) for the cfg3 decode (B = 64)
and prefill (C = 2048) head-output sizes.  Prints one JSON line per (TP, phase)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_19867_b200 as spd  # noqa: E402


def run(tp, full_shape, iters=20, check=True):
    L = spd.lib()
    dev = torch.device("cuda", 0)
    vp = ctypes.c_void_p
    outs = [torch.zeros(full_shape, dtype=torch.bfloat16, device=dev) for _ in range(tp)]
    flags = [torch.zeros(2 * tp, dtype=torch.int32, device=dev) for _ in range(tp)]
    h = full_shape[0] // tp
    shards = [torch.randn((h,) + tuple(full_shape[1:]), device=dev).to(torch.bfloat16) for _ in range(tp)]
    streams = [torch.cuda.Stream(dev) for _ in range(tp)]
    shard_bytes = shards[0].numel() * 2
    fl = (vp * tp)(*[f.data_ptr() for f in flags])

    def round_():
        main = torch.cuda.current_stream(dev)
        for r in range(tp):
            streams[r].wait_stream(main)
        for r in range(tp):
            dsts = (vp * tp)(*[o.data_ptr() + r * shard_bytes for o in outs])
            st = L.semipd_peer_gather(vp(shards[r].data_ptr()), shard_bytes, dsts, fl,
                                      vp(flags[r].data_ptr()), tp, r, vp(streams[r].cuda_stream))
            assert st == 0, st
        for r in range(tp):
            main.wait_stream(streams[r])

    round_()
    torch.cuda.synchronize()
    if check:
        want = torch.cat(shards)
        for r in range(tp):
            assert torch.equal(outs[r].view(torch.int16), want.view(torch.int16)), r
        assert all(int(f.abs().sum()) == 0 for f in flags)  # every flag reset
    for _ in range(3):
        round_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        round_()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    # the same round captured once as a CUDA graph: GPU-side cost without the host submission
    # of the emulated ranks (which one host thread issues one after another)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        round_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us_g = e0.elapsed_time(e1) * 1e3 / iters
    if check:
        for r in range(tp):
            assert torch.equal(outs[r].view(torch.int16), torch.cat(shards).view(torch.int16)), r
        assert all(int(f.abs().sum()) == 0 for f in flags)
    moved = shard_bytes * tp * (tp - 1)  # bytes crossing between ranks per round
    return {"tp": tp, "full_shape": list(full_shape), "shard_bytes": shard_bytes,
            "us_per_round_eager": us, "us_per_round_graph": us_g, "moved_bytes": moved,
            "GB_s_moved_graph": moved / us_g / 1e3}


if __name__ == "__main__":
    for tp in (2, 4, 8):
        for phase, shp in (("decode", (64, 64, 128)), ("prefill", (64, 2048, 128))):
            r = run(tp, shp)
            r["phase"] = phase
            print(json.dumps(r), flush=True)


def memop_latency(n=200):
    """One stream: write 1 -> wait >= 1 -> write 0 on a local flag, n times (no other
    stream involved): the floor of one signal/wait pair."""
    from cuda.bindings import driver as drv
    dev = torch.device("cuda", 0)
    f = torch.zeros(4, dtype=torch.int32, device=dev)
    s = torch.cuda.Stream(dev)
    cs = drv.CUstream(s.cuda_stream)
    ptr = drv.CUdeviceptr(f.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(2):
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(n):
            drv.cuStreamWriteValue32(cs, ptr, 1, 0)
            drv.cuStreamWaitValue32(cs, ptr, 1, 0)
            drv.cuStreamWriteValue32(cs, ptr, 0, 0)
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


def memop_pingpong(n=200):
    """Two streams ping-pong through flags (A sets a, waits b; B waits a, sets b)."""
    from cuda.bindings import driver as drv
    dev = torch.device("cuda", 0)
    f = torch.zeros(2, dtype=torch.int32, device=dev)
    sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ca, cb = drv.CUstream(sa.cuda_stream), drv.CUstream(sb.cuda_stream)
    pa, pb = drv.CUdeviceptr(f.data_ptr()), drv.CUdeviceptr(f.data_ptr() + 4)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(sa)
    for i in range(1, n + 1):
        drv.cuStreamWriteValue32(ca, pa, i, 0)
        drv.cuStreamWaitValue32(cb, pa, i, 0)
        drv.cuStreamWriteValue32(cb, pb, i, 0)
        drv.cuStreamWaitValue32(ca, pb, i, 0)
    e1.record(sa)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


if __name__ == "__main__" and os.environ.get("SPD_MEMOP_PROBE") == "1":
    print(json.dumps({"memop_write_wait_reset_us": memop_latency(),
                      "memop_pingpong_round_trip_us": memop_pingpong(),
                      "CUDA_DEVICE_MAX_CONNECTIONS": os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS")}))
