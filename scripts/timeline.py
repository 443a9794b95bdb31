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
buf = torch.zeros(48 * 1024 * 8, dtype=torch.int64, device=dev); ctr = torch.zeros(1, dtype=torch.int32, device=dev)
for it in range(3):
    ctr.zero_()
    buf.zero_()
    L.semipd_debug_set_timeline(pool.h, ctypes.c_void_p(buf.data_ptr()), ctypes.c_void_p(ctr.data_ptr()))
    pool.prefill_attn(0, q, k, v, i32([0, C]), i32([0]), i32([0]), C, C, 1 / math.sqrt(d), out, sm_budget=budget)
    torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
pool.prefill_attn(0, q, k, v, i32([0, C]), i32([0]), i32([0]), C, C, 1 / math.sqrt(d), out, sm_budget=budget)
ev[1].record()
torch.cuda.synchronize()
print("kernel_us", ev[0].elapsed_time(ev[1]) * 1e3)
allr = buf.view(-1, 8).cpu().tolist()
cta = [r for r in allr if r[0] == 40]
if cta:
    g0 = min(r[2] for r in cta)
    ends = sorted(((r[3] - g0) / 1e3, (r[2] - g0) / 1e3, r[4], r[1]) for r in cta)
    print("cta_end_us min/med/max", ends[0][0], ends[len(ends) // 2][0], ends[-1][0],
          "start_us max", max(e[1] for e in ends))
    print("slowest CTAs (end_us, start_us, pair_steps, cta):", ends[-6:])
    print("pair steps per CTA: max", max(e[2] for e in ends), "min", min(e[2] for e in ends))
    json.dump(ends, open(os.path.join(ROOT, "gpurun_out", "tl_cta_%d.json" % budget), "w"))
rec = [r for r in allr if r[2] != 0 and r[0] != 40]
n = len(rec)
t0 = min(r[2] for r in rec)
for r in rec:
    r[2:4] = [x - t0 if x else 0 for x in r[2:4]]
    if r[0] < 20:
        r[4] = r[4] - t0 if r[4] else 0
        r[5:8] = [x - t0 if x > 0 else 0 for x in r[5:8]]
rec.sort(key=lambda r: r[2])
json.dump(rec, open(os.path.join(ROOT, "gpurun_out", os.environ.get("TL_OUT", "timeline.json")), "w"))
print("records", n)
