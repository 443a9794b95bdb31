import time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for name, f in [("clock", lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                ("reasons", lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)),
                ("both", lambda: (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))]:
    t = time.perf_counter(); n = 0
    while time.perf_counter() - t < 1.0:
        f(); n += 1
    print(name, "calls/s", n, "ms/call", 1000.0 / n)
