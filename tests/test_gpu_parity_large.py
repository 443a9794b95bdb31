"""GPU parity at the BASELINE.json configurations' full sizes ("Parity on the
large configs uses the same sample, with all heads and all decode requests"), plus the
device error path (§8(b) BAD_BLOCK) and the host INVALID branches of the attention calls.

- cfg 4 (long-context mix): decode B = 16 at ctx 32768, all rows and heads: S = 9 splits of
  <= 4096 keys, merged in split order (a7); an 8192-token prefill chunk at every prefix
  P in {0, 8192, 16384, 24576} of a 32k prompt (every 64th row + the last row, all heads).
- cfg 2 as bench.py runs it: the pool layout of bench.Workload (64 decode requests at
  ctx 2048 allocated first, then the prefill request), 64-token pages, both phases co-running
  on two streams at the bench's split (40, 60) -> 59 / 89 SMs; decode all rows, prefill every
  16th row + the last.

Tolerances (R16): bf16 max_abs <= 2e-2 and fro_rel <= 1e-2; K/V pool writes and
block tables bit-exact."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth
from harness import Rig, compare, np_bits

pytestmark = pytest.mark.gpu

SHAPE_8B = synth.CFG2_LLAMA8B


def one_layer(shape, **kw):
    d = dict(name=shape.name, num_q_heads=shape.num_q_heads, num_kv_heads=shape.num_kv_heads,
             head_dim_k=shape.head_dim_k, head_dim_v=shape.head_dim_v,
             block_size=shape.block_size, dtype=shape.dtype, num_layers=1,
             kv_shared=shape.kv_shared, scale=shape.scale)
    d.update(kw)
    return synth.AttnShape(**d)


def sample_rows(T: int, stride: int) -> np.ndarray:
    m = np.zeros(T, np.uint8)
    m[::stride] = 1
    m[-1] = 1
    return m


# ----------------------------------------------------------------------------- cfg 4
@pytest.mark.parametrize("bs,dist", [(64, synth.FLAT), (16, synth.NEEDLE)])
def test_decode_cfg4_ctx32k_nine_splits(bs, dist):
    """cfg 4 decode at full size: 16 requests at ctx 32768 (32769 keys with the appended
    row): ceil(32769 / 4096) = 9 splits per (request, kv head), 1152 units, fp32 partials
    merged by the last CTA in split order.  Every output row against the oracle; the
    appended rows bit-exact in the pool."""
    from test_gpu_parity import run_decode
    shape = one_layer(SHAPE_8B, block_size=bs)
    run_decode(shape, [32768] * 16, seed=1040 + dist, dist=dist)


@pytest.mark.parametrize("P", [0, 8192, 16384, 24576])
def test_prefill_cfg4_chunk8k_at_prefix(P):
    """cfg 4 prefill at full size: one 8192-token chunk of a 32k prompt over a paged prefix
    of P tokens (64-token pages): up to 256 kv tiles per q tile, lazy rescale over the whole
    row.  Every 64th row + the last row, all 32 heads; the chunk's K/V pool writes
    bit-exact."""
    from test_gpu_parity import run_prefill
    run_prefill(one_layer(SHAPE_8B, block_size=64), [8192], [P], seed=1041 + P // 8192,
                dist=synth.NEEDLE if P == 24576 else synth.FLAT,
                rows_mask=sample_rows(8192, 64))


# ----------------------------------------------------------------------------- cfg 2 (bench)
def test_bench_config_corun_full_size():
    """The bench's own step at full size, one layer: bench.Workload's pool (64 decode
    requests x 33 pages at ctx 2048, then the prefill request's 32 pages; 64-token pages),
    prefill (C = 2048, P = 0) on stream P at 59 SMs co-running with decode (B = 64) on
    stream D at 89 SMs (split (40, 60), the bench's best).  Decode: all rows; prefill:
    every 16th row + the last; the appended and the chunk's K/V bit-exact."""
    shape = one_layer(SHAPE_8B, block_size=64)
    B, ctx, C, bs = 64, 2048, 2048, 64
    nb_dec, nb_pre = ctx // bs + 1, -(-C // bs)
    rig = Rig(shape, num_blocks=B * nb_dec + nb_pre + 64, max_reqs=B + 2, mbr=nb_dec + 8)
    rig.alloc(list(range(B)), [nb_dec] * B)  # bench.Workload: decode requests first, one call
    rig.alloc([B], [nb_pre])
    rig.assert_tables_match()
    dc = synth.decode_case(shape, [ctx] * B, seed=1020, dist=synth.FLAT, req_ids=list(range(B)))
    for b in range(B):
        rig.scatter(0, b, dc.k_ctx[b], dc.v_ctx[b])
    pc = synth.prefill_case(shape, [C], [0], seed=1220, dist=synth.VSHIFT, req_ids=[B])
    kp, vp = rig.host_pool(0)
    dev = rig.dev
    Hq, dv = shape.num_q_heads, shape.head_dim_v
    out_d = torch.empty(B, Hq, dv, dtype=shape.dtype, device=dev)
    out_p = torch.empty(C, Hq, dv, dtype=shape.dtype, device=dev)
    ws = rig.pool.new_decode_workspace(B, Hq, ctx)
    st_p = torch.zeros(1, dtype=torch.int32, device=dev)
    st_d = torch.zeros(1, dtype=torch.int32, device=dev)
    ins = [t.to(dev) for t in (dc.q, dc.k_new, dc.v_new, pc.q, pc.k_new, pc.v_new)]
    sP, sD = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    rig.pool.set_partition(40, 60)
    assert rig.pool.sm_budgets() == (59, 89)
    torch.cuda.synchronize()
    with torch.cuda.stream(sP):
        rig.pool.prefill_attn(0, ins[3], ins[4], ins[5], rig.i32([0, C]), rig.i32([B]),
                              rig.i32([0]), C, C, shape.softmax_scale, out_p, status=st_p,
                              stream=sP)
    with torch.cuda.stream(sD):
        rig.pool.decode_attn(0, ins[0], ins[1], ins[2], rig.i32(range(B)), rig.i32([ctx] * B), ctx,
                             shape.softmax_scale, out_d, ws, status=st_d, stream=sD)
    torch.cuda.synchronize()
    assert int(st_p.item()) == 0 and int(st_d.item()) == 0
    ref_d = oracle.decode(np_bits(dc.q), np_bits(dc.k_new), np_bits(dc.v_new), kp, vp,
                          rig.ref_alloc.bt, list(range(B)), [ctx] * B, shape.softmax_scale)
    mask = sample_rows(C, 16)
    ref_p = oracle.prefill(np_bits(pc.q), np_bits(pc.k_new), np_bits(pc.v_new), kp, vp,
                           rig.ref_alloc.bt, [0, C], [B], [0], shape.softmax_scale,
                           rows_mask=mask)
    compare(out_d.float().cpu().double().numpy(), ref_d, shape.dtype, "bench decode")
    sel = mask.astype(bool)
    compare(out_p.float().cpu().double().numpy()[sel], ref_p[sel], shape.dtype, "bench prefill")
    K, V = rig.host_pool(0)
    np.testing.assert_array_equal(K, kp)  # decode appends + the chunk's K/V, bit-exact
    np.testing.assert_array_equal(V, vp)


# ----------------------------------------------------------------------------- BAD_BLOCK
def _bad_decode(shape, ctx, bad_req, bad_page, bad_value, seed=7):
    """Decode where request `bad_req`'s table entry `bad_page` is replaced by `bad_value`
    (-1 = unallocated, or an id >= N_B).  Expect status BAD_BLOCK, no fault, and every other
    request still equal to the oracle."""
    bs = shape.block_size
    nblk = [c // bs + 1 for c in ctx]
    rig = Rig(shape, num_blocks=sum(nblk) + 4, max_reqs=len(ctx) + 1, mbr=max(nblk) + 1)
    for b, n in enumerate(nblk):
        rig.alloc([b], [n])
    case = synth.decode_case(shape, ctx, seed, synth.FLAT)
    for b in range(len(ctx)):
        rig.scatter(0, b, case.k_ctx[b], case.v_ctx[b])
    kp, vp = rig.host_pool(0)
    _, _, BT, _ = rig.pool.views(0)
    BT[bad_req, bad_page] = bad_value
    dev = rig.dev
    B, Hq, dv = len(ctx), shape.num_q_heads, shape.head_dim_v
    out = torch.zeros(B, Hq, dv, dtype=shape.dtype, device=dev)
    ws = rig.pool.new_decode_workspace(B, Hq, max(ctx))
    rig.pool.decode_attn(0, case.q.to(dev), case.k_new.to(dev),
                         None if case.v_new is None else case.v_new.to(dev),
                         rig.i32(range(B)), rig.i32(ctx), max(ctx), shape.softmax_scale, out, ws,
                         status=rig.status)
    torch.cuda.synchronize()  # raises if the kernel faulted
    assert int(rig.status.item()) == 5, "expected SEMIPD_ERR_BAD_BLOCK"
    good = [b for b in range(B) if b != bad_req]
    ref = oracle.decode(np_bits(case.q[good]), np_bits(case.k_new[good]),
                        None if case.v_new is None else np_bits(case.v_new[good]), kp, vp,
                        rig.ref_alloc.bt, good, [ctx[b] for b in good], shape.softmax_scale,
                        kv_shared=shape.kv_shared, dv=dv)
    compare(out.float().cpu().double().numpy()[good], ref, shape.dtype, "decode beside a bad table")
    # the pool is usable afterwards: restore the entry, rerun, status OK
    BT[bad_req, bad_page] = int(rig.ref_alloc.bt[bad_req, bad_page])
    rig.pool.decode_attn(0, case.q.to(dev), case.k_new.to(dev),
                         None if case.v_new is None else case.v_new.to(dev),
                         rig.i32(range(B)), rig.i32(ctx), max(ctx), shape.softmax_scale, out, ws,
                         status=rig.status)
    torch.cuda.synchronize()
    assert int(rig.status.item()) == 0


@pytest.mark.parametrize("bs,bad_value", [(16, -1), (64, -1), (64, 10 ** 6)])
def test_decode_bad_block_skipped(bs, bad_value):
    _bad_decode(one_layer(SHAPE_8B, block_size=bs), [300, 5000, 129], bad_req=1, bad_page=2,
                bad_value=bad_value)


def test_decode_bad_block_fp32_generic_path():
    _bad_decode(synth.CFG1_TINY, [15, 100, 256], bad_req=1, bad_page=3, bad_value=-1)


def test_decode_bad_block_mla_tensor_kernel():
    _bad_decode(one_layer(synth.CFG5_MLA), [300, 1500, 64], bad_req=1, bad_page=4, bad_value=-1)


def _bad_prefill(shape, chunks, prefixes, bad_req, bad_page, seed=9):
    bs = shape.block_size
    nblk = [-(-(c + p) // bs) for c, p in zip(chunks, prefixes)]
    rig = Rig(shape, num_blocks=sum(nblk) + 4, max_reqs=len(chunks) + 1, mbr=max(nblk) + 1)
    for i, n in enumerate(nblk):
        rig.alloc([i], [n])
    case = synth.prefill_case(shape, chunks, prefixes, seed, synth.FLAT)
    for i in range(len(chunks)):
        rig.scatter(0, i, case.k_prefix[i], case.v_prefix[i])
    kp, vp = rig.host_pool(0)
    _, _, BT, _ = rig.pool.views(0)
    BT[bad_req, bad_page] = -1
    dev = rig.dev
    T, Hq, dv = sum(chunks), shape.num_q_heads, shape.head_dim_v
    out = torch.zeros(T, Hq, dv, dtype=shape.dtype, device=dev)
    rig.pool.prefill_attn(0, case.q.to(dev), case.k_new.to(dev),
                          None if case.v_new is None else case.v_new.to(dev),
                          rig.i32(case.cu_seqlens), rig.i32(range(len(chunks))), rig.i32(prefixes),
                          T, max(chunks), shape.softmax_scale, out, status=rig.status)
    torch.cuda.synchronize()
    assert int(rig.status.item()) == 5, "expected SEMIPD_ERR_BAD_BLOCK"
    # the other requests are unaffected
    cu = case.cu_seqlens
    for i in range(len(chunks)):
        if i == bad_req:
            continue
        sl = slice(cu[i], cu[i + 1])
        ref = oracle.prefill(np_bits(case.q[sl]), np_bits(case.k_new[sl]),
                             None if case.v_new is None else np_bits(case.v_new[sl]), kp.copy(),
                             None if vp is None else vp.copy(), rig.ref_alloc.bt,
                             [0, chunks[i]], [i], [prefixes[i]], shape.softmax_scale,
                             kv_shared=shape.kv_shared, dv=dv)
        compare(out[sl].float().cpu().double().numpy(), ref, shape.dtype,
                f"prefill request {i} beside a bad table")


def test_prefill_bad_block_prefix_page_tcgen05():
    _bad_prefill(one_layer(SHAPE_8B, block_size=64), [200, 300], [100, 500], bad_req=1,
                 bad_page=3)


def test_prefill_bad_block_mla():
    _bad_prefill(one_layer(synth.CFG5_MLA), [130, 90], [64, 300], bad_req=1, bad_page=2)


# ----------------------------------------------------------------------------- host INVALID
def test_attention_calls_reject_bad_arguments():
    """Host argument errors return INVALID synchronously and launch nothing (§8(b))."""
    from paper_2504_19867_b200 import INVALID, SemipdError
    shape = one_layer(SHAPE_8B, block_size=64)
    rig = Rig(shape, num_blocks=40, max_reqs=3, mbr=20)
    rig.alloc([0, 1], [5, 5])
    dev = rig.dev
    q = torch.zeros(2, 32, 128, dtype=torch.bfloat16, device=dev)
    kv = torch.zeros(2, 8, 128, dtype=torch.bfloat16, device=dev)
    out = torch.zeros(2, 32, 128, dtype=torch.bfloat16, device=dev)
    ids, ctx = rig.i32([0, 1]), rig.i32([10, 20])
    ws = rig.pool.new_decode_workspace(2, 32, 20)
    c0 = rig.pool.launch_count()

    def dec(**kw):
        a = dict(layer=0, q=q, k_new=kv, v_new=kv, req_ids=ids, ctx_lens=ctx, max_ctx_len=20,
                 scale=0.1, out=out, workspace=ws)
        a.update(kw)
        return rig.pool.decode_attn(**a)

    def pre(**kw):
        a = dict(layer=0, q=q, k_new=kv, v_new=kv, cu_seqlens=rig.i32([0, 2]), req_ids=rig.i32([0]),
                 prefix_lens=rig.i32([0]), total_q=2, max_chunk_len=2, scale=0.1, out=out)
        a.update(kw)
        return rig.pool.prefill_attn(**a)

    bad = [lambda: dec(sm_budget=149), lambda: dec(sm_budget=-2), lambda: dec(layer=1),
           lambda: dec(layer=-1), lambda: dec(q=torch.zeros(2, 30, 128, dtype=torch.bfloat16,
                                                            device=dev)),  # 30 % 8 != 0
           lambda: dec(workspace=ws[:64]),  # workspace too small
           lambda: dec(max_ctx_len=-1),
           lambda: pre(sm_budget=149), lambda: pre(layer=3),
           lambda: pre(q=torch.zeros(2, 12, 128, dtype=torch.bfloat16, device=dev))]
    for i, fn in enumerate(bad):
        with pytest.raises(SemipdError) as ei:
            fn()
        assert ei.value.status == INVALID, i
    for xy in [(0, 50), (50, 0), (101, 50), (50, 100.5), (-3, 40)]:
        with pytest.raises(SemipdError) as ei:
            rig.pool.set_partition(*xy)
        assert ei.value.status == INVALID
    torch.cuda.synchronize()
    assert rig.pool.launch_count() == c0, "an INVALID call launched a kernel"
    # a valid call after all that still works
    dec()
    torch.cuda.synchronize()
