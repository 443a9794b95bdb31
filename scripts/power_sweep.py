#!/usr/bin/env python
"""Dev probe: the cfg-2 co-run step per split under sustained (power-capped) load: after ~0.6 s
of back-to-back replays at that split, time ~0.6 s more and read the board's energy counter
(NVML total energy, mJ) and SM clock around it.  One JSON line per split."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses
import torch
import bench


def main():
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    xs = [float(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "25,30,35,40,45,50").split(",")]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    shape = dataclasses.replace(bench.MODELS["llama3-8b"], block_size=64)
    w = bench.Workload(shape, 1, dev)
    run = bench.Runner(w, dev)
    for _ in range(2):
        w.corun_step(50, 50)
    for x in xs:
        step = run.capture(lambda: w.corun_step(x, 100 - x, 0, 0))
        bench.time_steps(step, 180, dev)  # ~0.6 s: reach the power cap
        n = 180
        e0 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
        c0 = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        t = bench.time_steps(step, n, dev)
        e1 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
        c1 = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        rec = {"x": x, "ms_per_step": t / n * 1e3, "tokens_per_s": w.tokens_per_step() * n / t,
               "joules_per_step": (e1 - e0) / 1e3 / n, "avg_power_w": (e1 - e0) / 1e3 / t,
               "sm_mhz_start_end": [c0, c1], "sw_power_cap": bool(reasons & nv.nvmlClocksEventReasonSwPowerCap)}
        print(json.dumps(rec), flush=True)
        time.sleep(1.0)  # let the board cool a little between splits


if __name__ == "__main__":
    main()
