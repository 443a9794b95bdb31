"""Dev probe: how many NVML samples bench.ClockSampler takes over a ~70 ms busy region."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench


def main():
  dev = torch.device("cuda", 0)
  a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
  for label, fn in [("sleep", lambda: time.sleep(0.07)),
                    ("gemm", lambda: [a @ a for _ in range(40)] and torch.cuda.synchronize())]:
    with bench.ClockSampler(bench.nvml_id(dev)) as clk:
        t = time.perf_counter(); fn(); dt = time.perf_counter() - t
    print(label, round(dt * 1e3, 1), "ms", clk.summary())


if __name__ == "__main__":
    main()
