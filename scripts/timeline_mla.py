#!/usr/bin/env python
"""Build a SPD_TIMELINE variant of the library and dump the MLA tcgen05 decode pipeline of
CTA 0 (clock64 stamps: producer half-page issues, MMA QK/PV issues, softmax waits) for one
B=256 ctx=1000 launch.  Records (kind, tile, a, b, c):
  1 producer: before empty wait, after wait, after both TMA issued
  2 QK issued   3 PV issued
  4 softmax: s_full wait start, s_full done, o_done wait start   5: o_done done, p_full arrive"""
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
budget = int(sys.argv[1]) if len(sys.argv) > 1 else 148
B, ctx = int(os.environ.get("TL_B", "256")), int(os.environ.get("TL_CTX", "1000"))
if os.environ.get("TL_LOGN"):  # the bench's cfg-5 batch: lognormal around ctx, longest first
    import numpy as np
    rng = np.random.default_rng(5005)
    ctxs = sorted((int(c) for c in np.clip(rng.lognormal(math.log(ctx) - 0.125, 0.5, B), 64, 4096)), reverse=True)
else:
    ctxs = [ctx] * B
ctx = max(ctxs)
dev = torch.device("cuda", 0)
nb = ctx // 64 + 1
pool = spd.KVPool(spd.PoolConfig(1, B * nb + 4, 64, 1, 576, 512, B + 1, nb + 1, kv_shared=True), dev)
i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)
pool.alloc_blocks(i32(list(range(B))), i32([c // 64 + 1 for c in ctxs]))
K, _, _, _ = pool.views(0)
K.normal_()
q = torch.randn(B, 16, 576, device=dev).bfloat16()
kn = torch.randn(B, 1, 576, device=dev).bfloat16()
out = torch.empty(B, 16, 512, dtype=torch.bfloat16, device=dev)
ws = pool.new_decode_workspace(B, 16, ctx)
buf = torch.zeros(9 * 512 * 8, dtype=torch.int64, device=dev)
ctr = torch.zeros(1, dtype=torch.int32, device=dev)
tl_cta = int(os.environ.get("TL_CTA", "0"))
for it in range(3):
    ctr.fill_(tl_cta)
    buf.zero_()
    L.semipd_debug_set_timeline(pool.h, ctypes.c_void_p(buf.data_ptr()), ctypes.c_void_p(ctr.data_ptr()))
    pool.decode_attn(0, q, kn, None, i32(list(range(B))), i32(ctxs), ctx, 1 / math.sqrt(192), out, ws,
                     sm_budget=budget)
    torch.cuda.synchronize()
rec = [r for r in buf.view(-1, 8)[:, :5].cpu().tolist() if r[0] != 0]
n = len(rec)
cta = [r for r in rec if r[0] == 8]
rec = [r for r in rec if r[0] != 8]
if cta:
    g0 = min(r[2] for r in cta)
    for r in cta:
        r[2] -= g0
        r[3] -= g0
    ends = sorted(r[3] for r in cta)
    starts = sorted(r[2] for r in cta)
    print("CTA start ns: min %d max %d; end ns: min %d median %d max %d" % (starts[0], starts[-1], ends[0], ends[len(ends)//2], ends[-1]))
    print("CTA end ns deciles:", [ends[int(len(ends) * k / 10)] for k in range(10)] + [ends[-1]])
    json.dump(cta, open(os.path.join(ROOT, "gpurun_out", "cta_times.json"), "w"))
t0 = min(r[2] for r in rec)
for r in rec:
    r[2:5] = [x - t0 if x else 0 for x in r[2:5]]
rec.sort(key=lambda r: (r[1], r[0]))
json.dump(rec, open(os.path.join(ROOT, "gpurun_out", os.environ.get("TL_OUT", "timeline_mla.json")), "w"))
print("records", n)
