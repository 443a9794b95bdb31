#!/usr/bin/env python
"""Dev probe: per-window step times of the bench's cfg2 co-run step at one split, replayed
back to back (is there a warm-up transient or a sustained-load slowdown?).  Prints one line
per window of R replays."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses
import torch
import bench


def _sampler(stop, out):
    import time
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    rows = []
    t0 = time.perf_counter()
    while not stop.is_set():
        try:
            mt = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_MEMORY_TEMP])[0].value.uiVal
        except Exception:
            mt = -1
        rows.append((round(time.perf_counter() - t0, 3), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                     nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM), nv.nvmlDeviceGetPowerUsage(h) // 1000,
                     nv.nvmlDeviceGetTemperature(h, nv.NVML_TEMPERATURE_GPU), mt,
                     hex(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
        time.sleep(0.05)
    out.put(rows)


def main():
    x = float(sys.argv[1]) if len(sys.argv) > 1 else 30.0
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    shape = dataclasses.replace(bench.MODELS["llama3-8b"], block_size=64)
    w = bench.Workload(shape, 1, dev)
    run = bench.Runner(w, dev)
    for _ in range(2):
        w.corun_step(50, 50)
    step = run.capture(lambda: w.corun_step(x, 100 - x, 0, 0))
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    stop, q = ctx.Event(), ctx.Queue()
    pr = ctx.Process(target=_sampler, args=(stop, q), daemon=True)
    pr.start()
    import time
    time.sleep(3.0)
    ts = []
    for i in range(n):
        t = bench.time_steps(step, R, dev) / R * 1e3
        ts.append(t)
        print(f"window {i:3d} ms/step {t:.4f}", flush=True)
    stop.set()
    for r in q.get(timeout=30)[::4]:
        print("nvml t,sm,mem,W,T,Tmem,reasons", *r)
    print("first3", [round(v, 4) for v in ts[:3]], "median", round(sorted(ts)[len(ts) // 2], 4),
          "min", round(min(ts), 4), "max", round(max(ts), 4))


if __name__ == "__main__":
    main()
