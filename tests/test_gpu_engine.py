"""Co-run engine on a dense GQA pool (Llama shapes, 64-token pages): a few iterations of
alloc -> prefill (stream P) || decode (stream D) -> free, with layer-0 outputs of the last
iteration checked against the fp64 oracle and the op log replayed on the allocator model."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from harness import compare

pytestmark = pytest.mark.gpu


def _bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def test_engine_gqa_iterations_match_oracle():
    from paper_2504_19867_b200 import KVPool, PoolConfig
    from paper_2504_19867_b200.engine import CoRunEngine
    dev = torch.device("cuda", 0)
    Hq, Hkv, d, bs, L = 8, 2, 128, 64, 2
    pool = KVPool(PoolConfig(L, 160, bs, Hkv, d, d, 64, 40, oplog_words=1 << 16), dev)
    eng = CoRunEngine(pool, Hq, 1 / math.sqrt(d), chunk_budget=256, max_decode=32,
                      partition=(40, 60), seed=3, max_ctx=2048)
    trace = synth.mla_trace(n_req=24, lam=2.0, seed=9)
    trace = [synth.TraceRequest(r.rid, r.arrival_iter, min(r.input_len, 500), min(r.output_len, 40))
             for r in trace]
    idx = 0
    checked = 0
    while (idx < len(trace) or not eng.idle) and eng.it < 400:
        arr = []
        while idx < len(trace) and trace[idx].arrival_iter <= eng.it:
            arr.append(trace[idx])
            idx += 1
        check = eng.it % 7 == 3
        if check:
            torch.cuda.synchronize()
            K, V, _, _ = pool.views(0)
            kp, vp = _bits(K), _bits(V)
        s, plan = eng.step(arr)
        if check and (plan.prefill or plan.decode):
            bt = pool.views(0)[2].cpu().numpy()
            if plan.prefill:
                T = s.prefill_tokens
                cu = [0]
                for _, ch, _ in plan.prefill:
                    cu.append(cu[-1] + ch)
                ref = oracle.prefill(_bits(eng.q_pre[:T]), _bits(eng.k_pre[:T]), _bits(eng.v_pre[:T]),
                                     kp.copy(), vp.copy(), bt, cu, [r.slot for r, _, _ in plan.prefill],
                                     [pf for _, _, pf in plan.prefill], 1 / math.sqrt(d))
                compare(eng.o_pre[0][:T].float().cpu().double().numpy(), ref, torch.bfloat16,
                        f"engine prefill it {s.it}")
            live = [(j, r, c) for j, (r, c) in enumerate(plan.decode) if r.slot >= 0]
            if live:
                sel = [j for j, _, _ in live]
                ref = oracle.decode(_bits(eng.q_dec[sel]), _bits(eng.k_dec[sel]), _bits(eng.v_dec[sel]),
                                    kp.copy(), vp.copy(), bt, [r.slot for _, r, _ in live],
                                    [c for _, _, c in live], 1 / math.sqrt(d))
                compare(eng.o_dec[0][sel].float().cpu().double().numpy(), ref, torch.bfloat16,
                        f"engine decode it {s.it}")
            checked += 1
    assert eng.idle and len(eng.finished) == len(trace) and checked >= 3
    words, dropped = pool.oplog()
    assert dropped == 0
    ref = oracle.Allocator(160, 64, 40)
    i = 0
    while i < len(words):
        seq, kind, n, status = words[i:i + 4]
        ids = words[i + 4:i + 4 + n]
        if kind == 1:
            assert ref.alloc(ids, words[i + 4 + n:i + 4 + 2 * n]) == status
            i += 4 + 2 * n
        else:
            assert ref.free(ids) == status
            i += 4 + n
    bt, nb = pool.views(0)[2].cpu().numpy(), pool.views(0)[3].cpu().numpy()
    np.testing.assert_array_equal(bt, ref.bt)
    np.testing.assert_array_equal(nb, ref.nblk)
