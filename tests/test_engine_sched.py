"""Host logic of the co-run engine (paper_2504_19867_b200.engine.Scheduler) on CPU: FCFS
chunked-prefill admission, decode stepping, host block accounting against the oracle
allocator (every planned grant must succeed on the sequential allocator model),
preemption on a full pool, and that a tight cfg-5 style trace drains."""
import numpy as np
import pytest

import oracle
import synth
from paper_2504_19867_b200.engine import Scheduler


def run_trace(sched: Scheduler, trace, max_iters=200000, check=None):
    ref = oracle.Allocator(sched.num_blocks, len(sched.free_slots), 4096)
    idx, it = 0, 0
    while (idx < len(trace) or not sched.idle) and it < max_iters:
        arr = []
        while idx < len(trace) and trace[idx].arrival_iter <= it:
            arr.append(trace[idx])
            idx += 1
        sched.add(arr)
        waiting_before = list(sched.waiting)
        plan, allocs, preempt = sched.plan()
        # every planned grant succeeds on the allocator model, in call order (S10)
        for slot, n in allocs:
            assert ref.alloc([slot], [n]) == oracle.OK
        assert ref.free_blocks == sched.free_blocks
        if check:
            check(sched, plan, allocs, preempt, waiting_before)
        finishing = sched.finishing(plan)
        frees = [r.slot for r in finishing] + [v.slot for v in preempt]
        sched.commit(plan, preempt)
        if frees:
            assert ref.free(frees) == oracle.OK
        assert ref.free_blocks == sched.free_blocks
        held = sum(r.nblk for r in list(sched.waiting) + sched.running)
        assert sched.free_blocks + held == sched.num_blocks  # conservation
        it += 1
    return it


def test_fcfs_budget_and_decode_cap():
    sched = Scheduler(num_blocks=400, block_size=64, max_reqs=64, chunk_budget=300, max_decode=5)
    trace = synth.mla_trace(n_req=40, lam=4.0, seed=3)

    def check(s, plan, allocs, preempt, waiting_before):
        chunks = [ch for _, ch, _ in plan.prefill]
        assert sum(chunks) <= s.chunk_budget
        # prefill takes a prefix of the FCFS queue
        assert [r for r, _, _ in plan.prefill] == waiting_before[:len(plan.prefill)]
        for r, ch, pf in plan.prefill:
            assert 0 < ch <= r.input_len - pf and pf == r.prefilled
        assert len(plan.decode) <= s.max_decode
        for r, ctx in plan.decode:
            assert ctx == r.input_len + r.generated and r.nblk * s.bs >= ctx + 1

    run_trace(sched, trace, check=check)
    assert len(sched.finished) == 40


def test_tight_pool_preempts_and_drains():
    sched = Scheduler(num_blocks=40, block_size=16, max_reqs=32, chunk_budget=128, max_decode=16)
    trace = synth.mla_trace(n_req=60, lam=2.0, seed=11)
    pre = []

    def check(s, plan, allocs, preempt, waiting_before):
        pre.extend(preempt)

    run_trace(sched, trace, check=check)
    assert len(sched.finished) + len(sched.rejected) == 60 and len(sched.finished) > 30
    assert all(sched.blocks(r.input_len + r.output_len) > 40 for r in sched.rejected)
    fin = {r.trace_id: r for r in sched.finished}
    assert all(fin[t.rid].generated == t.output_len for t in trace if t.rid in fin)
    assert pre, "a 40-block pool under this trace must preempt"


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_traces_conserve_blocks(seed):
    rng = np.random.default_rng(seed)
    sched = Scheduler(num_blocks=int(rng.integers(60, 300)), block_size=int(rng.choice([16, 64])),
                      max_reqs=48, chunk_budget=int(rng.integers(64, 1024)),
                      max_decode=int(rng.integers(4, 64)))
    trace = synth.mla_trace(n_req=50, lam=float(rng.uniform(0.5, 4.0)), seed=seed)
    run_trace(sched, trace)
    assert len(sched.finished) + len(sched.rejected) == 50
    assert sched.free_blocks == sched.num_blocks
