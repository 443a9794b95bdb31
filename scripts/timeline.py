#!/usr/bin/env python
"""Build a SPD_TIMELINE variant of the library and dump the prefill pipeline timeline of
CTA 0 (clock64 stamps per softmax tile / MMA issue) for one cfg2 prefill launch."""
import ctypes, json, math, os, subprocess, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_19867_b200 import _build
lib_tl = os.path.join(_build.PKG, "libsemipd_tl.so")
objs = []
for src in _build.sources():
    obj = os.path.join(_build.BUILD, "tl_" + os.path.basename(src)[:-3] + ".o")
    extra = os.environ.get("TL_FLAGS", "").split()
    subprocess.check_call([_build.nvcc(), *_build.NVCC_FLAGS, "-DSPD_TIMELINE", *extra, "-c", src, "-o", obj],
                          stderr=subprocess.DEVNULL)
    objs.append(obj)
subprocess.check_call([_build.nvcc(), *_build.ARCH, "-shared", "-o", lib_tl, *objs])
import paper_2504_19867_b200 as spd
spd._build.LIB = lib_tl
spd._build.up_to_date = lambda: True
L = spd.lib()
budget = int(sys.argv[1]) if len(sys.argv) > 1 else 74
dev = torch.device("cuda", 0)
C, Hq, Hkv, d = 2048, 32, 8, 128
cfg = spd.PoolConfig(1, 40, 64, Hkv, d, d, 2, 34)
pool = spd.KVPool(cfg, dev)
i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)
pool.alloc_blocks(i32([0]), i32([32]))
q = torch.randn(C, Hq, d, device=dev).bfloat16(); k = torch.randn(C, Hkv, d, device=dev).bfloat16()
v = torch.randn(C, Hkv, d, device=dev).bfloat16(); out = torch.empty_like(q)
buf = torch.zeros(32 * 1024 * 8, dtype=torch.int64, device=dev); ctr = torch.zeros(1, dtype=torch.int32, device=dev)
for it in range(3):
    ctr.zero_()
    buf.zero_()
    L.semipd_debug_set_timeline(pool.h, ctypes.c_void_p(buf.data_ptr()), ctypes.c_void_p(ctr.data_ptr()))
    pool.prefill_attn(0, q, k, v, i32([0, C]), i32([0]), i32([0]), C, C, 1 / math.sqrt(d), out, sm_budget=budget)
    torch.cuda.synchronize()
rec = [r for r in buf.view(-1, 8).cpu().tolist() if r[2] != 0]
n = len(rec)
t0 = min(r[2] for r in rec)
for r in rec:
    r[2:4] = [x - t0 if x else 0 for x in r[2:4]]
    if r[0] < 20:
        r[4] = r[4] - t0 if r[4] else 0
rec.sort(key=lambda r: r[2])
json.dump(rec, open(os.path.join(ROOT, "gpurun_out", os.environ.get("TL_OUT", "timeline.json")), "w"))
print("records", n)
