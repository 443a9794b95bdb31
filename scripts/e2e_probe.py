"""Dev probe: where the e2e step's time goes (full step vs copies only vs kernels only)."""
import os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench


def main():
    x = 30.0
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    local = bench.gpu_local_cpus(dev)
    if local:
        os.sched_setaffinity(0, local)
    shape = dataclasses.replace(bench.MODELS["llama3-8b"], block_size=64)
    w = bench.Workload(shape, 1, dev)
    ee = bench.E2E(w)
    f = lambda: ee.step(x, 100 - x)  # noqa: E731
    for _ in range(2):
        f()
    t = bench.time_steps(f, 5, dev) / 5
    print(f"full e2e step {t * 1e3:.2f} ms")
    pa, da = w.pool.prefill_attn, w.pool.decode_attn
    w.pool.prefill_attn = lambda *a, **k: None
    w.pool.decode_attn = lambda *a, **k: None
    t = bench.time_steps(f, 5, dev) / 5
    print(f"copies only {t * 1e3:.2f} ms")
    w.pool.prefill_attn, w.pool.decode_attn = pa, da
    h2d_only = ee.h_op, ee.h_od
    import time
    tt = time.perf_counter()
    for _ in range(5):
        f()
    th = (time.perf_counter() - tt) / 5
    torch.cuda.synchronize()
    print(f"host enqueue time per step {th * 1e3:.2f} ms")


if __name__ == "__main__":
    main()
