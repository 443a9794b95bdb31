"""RoPE kernel bandwidth (semipd_rope, bf16 in place): algorithmic bytes = read + write of q
and k = 2 * T * (Hq + Hkv) * d * 2 B per launch.  Rotates through buffer sets larger than
the 126 MB L2 so every launch streams from HBM.  One JSON line per case."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_19867_b200 import RopeConfig, rope_  # noqa: E402

dev = torch.device("cuda", 0)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))
for T, Hq, Hkv in [(2048, 32, 8), (8192, 32, 8), (32768, 32, 8), (64, 32, 8)]:
    d = 128
    per = 2 * T * (Hq + Hkv) * d * 2
    nset = max(1, min(16, (512 << 20) // (per // 2) + 1))
    sets = [(torch.randn(T, Hq, d, device=dev).to(torch.bfloat16),
             torch.randn(T, Hkv, d, device=dev).to(torch.bfloat16)) for _ in range(nset)]
    pos = torch.arange(T, dtype=torch.int32, device=dev) + 1000
    cfg = RopeConfig()
    for q, k in sets:
        rope_(q, k, pos, cfg)
    iters = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(iters):
        q, k = sets[i % nset]
        rope_(q, k, pos, cfg)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    print(json.dumps({"kernel": "rope_kernel<bf16>", "T": T, "Hq": Hq, "Hkv": Hkv, "d": d,
                      "bytes_per_launch": per, "us": us, "GB_s": per / us / 1e3,
                      "buffer_sets": nset}), flush=True)
