import sys, os, numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', 'tests'))
import synth, oracle
from harness import Rig, np_bits
import test_gpu_parity as T
chunks, prefixes = [int(x) for x in sys.argv[1].split(',')], [int(x) for x in sys.argv[2].split(',')]
dist = int(sys.argv[3]) if len(sys.argv) > 3 else 2
shape = T.small(T.SHAPE_8B)
try:
    T.run_prefill(shape, chunks, prefixes, seed=31, dist=dist)
    print("PASS")
except AssertionError as e:
    print("FAIL", str(e)[:200])
# re-run to get arrays
bs = 16
nblk = [-(-(c + p) // bs) for c, p in zip(chunks, prefixes)]
rig = Rig(shape, num_blocks=sum(nblk) + 5, max_reqs=len(chunks) + 2, mbr=max(nblk) + 2)
rids = list(range(len(chunks)))
for i in np.random.default_rng(32).permutation(len(chunks)):
    rig.alloc([rids[i]], [nblk[i]])
case = synth.prefill_case(shape, chunks, prefixes, 31, dist, rids)
for i in range(len(chunks)):
    rig.scatter(0, rids[i], case.k_prefix[i], case.v_prefix[i])
kp, vp = rig.host_pool(0)
dev = rig.dev
T_ = sum(chunks)
out = torch.zeros(T_, 32, 128, dtype=torch.bfloat16, device=dev)
rig.pool.prefill_attn(0, case.q.to(dev), case.k_new.to(dev), case.v_new.to(dev), rig.i32(case.cu_seqlens), rig.i32(rids), rig.i32(prefixes), T_, max(chunks), shape.softmax_scale, out, status=rig.status)
torch.cuda.synchronize()
ref = oracle.prefill(np_bits(case.q), np_bits(case.k_new), np_bits(case.v_new), kp, vp, rig.ref_alloc.bt, case.cu_seqlens, rids, prefixes, shape.softmax_scale)
err = np.abs(out.float().cpu().double().numpy() - ref).max(axis=2)
bad = np.argwhere(err > 2e-2)
print("status", int(rig.status.item()), "n bad (row,head):", len(bad))
cu = case.cu_seqlens
for t, h in bad[:40]:
    i = max(k for k in range(len(chunks)) if cu[k] <= t)
    print("row", t, "req", i, "trel", t - cu[i], "head", h, "err", round(float(err[t, h]), 4))
