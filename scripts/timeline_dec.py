#!/usr/bin/env python
"""SPD_TIMELINE build of the library; per-stage pipeline stamps of CTA 0 of the cfg2 decode
kernel (B=64, ctx 2048, bs 64) at budget argv[1]: kind 1 = producer (before empty wait, after
it, after the TMA issue), kind 2 = consumer (before full wait, after it, after release)."""
import ctypes, json, math, os, subprocess, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_19867_b200 import _build
lib_tl = os.path.join(_build.PKG, "libsemipd_tl.so")
objs = []
for src in _build.sources():
    obj = os.path.join(_build.BUILD, "tl_" + os.path.basename(src)[:-3] + ".o")
    subprocess.check_call([_build.nvcc(), *_build.NVCC_FLAGS, "-DSPD_TIMELINE", "-c", src, "-o", obj],
                          stderr=subprocess.DEVNULL)
    objs.append(obj)
subprocess.check_call([_build.nvcc(), *_build.ARCH, "-shared", "-o", lib_tl, *objs])
import paper_2504_19867_b200 as spd
spd._build.LIB = lib_tl
spd._build.up_to_date = lambda: True
L = spd.lib()
budget = int(sys.argv[1]) if len(sys.argv) > 1 else 89
B, ctx, bs = 64, 2048, 64
dev = torch.device("cuda", 0)
nb = ctx // bs + 1
pool = spd.KVPool(spd.PoolConfig(2, B * nb + 4, bs, 8, 128, 128, B + 1, nb + 1), dev)
i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)
pool.alloc_blocks(i32(list(range(B))), i32([nb] * B))
for l in range(2):
    K, V, _, _ = pool.views(l)
    K.normal_(); V.normal_()
q = torch.randn(B, 32, 128, device=dev).bfloat16(); kn = torch.randn(B, 8, 128, device=dev).bfloat16()
vn = torch.randn(B, 8, 128, device=dev).bfloat16(); out = torch.empty(B, 32, 128, dtype=torch.bfloat16, device=dev)
ws = pool.new_decode_workspace(B, 32, ctx)
buf = torch.zeros(4 * 2048 * 8, dtype=torch.int64, device=dev)
ctr = torch.zeros(1, dtype=torch.int32, device=dev)
for it in range(3):
    buf.zero_()
    L.semipd_debug_set_timeline(pool.h, ctypes.c_void_p(buf.data_ptr()), ctypes.c_void_p(ctr.data_ptr()))
    pool.decode_attn(it % 2, q, kn, vn, i32(list(range(B))), i32([ctx] * B), ctx, 1 / math.sqrt(128), out, ws,
                     sm_budget=budget)
    torch.cuda.synchronize()
rec = [r[:5] for r in buf.view(-1, 8).cpu().tolist() if r[0] != 0]
t0 = min(r[2] for r in rec)
for r in rec:
    r[2:5] = [x - t0 if x else 0 for x in r[2:5]]
json.dump(rec, open(os.path.join(ROOT, "gpurun_out", "timeline_dec.json"), "w"))
print("records", len(rec))
