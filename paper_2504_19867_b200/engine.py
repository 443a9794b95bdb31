"""Co-run iteration engine over the C ABI: one prefill worker and one decode worker sharing the
unified paged KV pool (semi-PD, §4.2, §4.4), each iteration = allocation, then
every layer's prefill attention on stream P and decode attention on stream D concurrently
under the SM partition (x, y) (§4.3), then frees.  This is the cfg-5 trace driver of
SURVEY §8(d): Poisson arrivals on a virtual clock of decode iterations, a 2048-token FCFS
chunked-prefill budget, every running request decoded each iteration (cap 512),
admission only when the allocator grants the blocks (one call per request, S10 / S:326-331).

Host-side block accounting mirrors the device allocator exactly (it is deterministic: LIFO
stack, all-or-nothing per call), so the engine never issues a call that can fail; the device
statuses are still checked after every iteration and the op log can be replayed by the test
oracle.  Nothing here computes attention: every step runs in libsemipd's kernels.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

import torch

from . import KVPool


@dataclass(eq=False)  # identity: queues hold distinct requests
class Request:
    trace_id: int
    input_len: int
    output_len: int
    slot: int = -1          # pool request id
    prefilled: int = 0      # prompt tokens already written by prefill
    generated: int = 0      # decode steps done
    nblk: int = 0           # blocks held (host mirror of the device table row)
    preempted: int = 0
    admit_seq: int = -1     # order of the last slot grant (preemption picks the newest)

    @property
    def ctx(self) -> int:   # tokens cached before the next decode step (R5)
        return self.input_len + self.generated


@dataclass
class IterStats:
    it: int
    prefill_reqs: int
    prefill_tokens: int
    prefill_pairs: int      # unmasked (q, k) pairs of this iteration's chunks (one layer)
    decode_reqs: int
    decode_keys: int        # sum of (ctx + 1) over decoded requests (one layer)
    t_prefill_ms: float
    t_decode_ms: float
    t_iter_ms: float
    alloc_calls: int
    free_calls: int
    free_blocks: int
    finished: int
    preempted: int


@dataclass
class Plan:
    """What one iteration launches (kept for the caller's parity sampling)."""
    prefill: list = field(default_factory=list)   # (Request, chunk_len, prefix_len)
    decode: list = field(default_factory=list)    # (Request, ctx)


class Scheduler:
    """Host-side admission and block accounting of the co-run engine (no device work; unit
    tested on CPU).  Mirrors the device allocator's free count exactly: every grant it plans
    succeeds on the device (LIFO stack, all-or-nothing per call, R9/R10)."""

    def __init__(self, num_blocks: int, block_size: int, max_reqs: int, *, chunk_budget: int = 2048,
                 max_decode: int = 512):
        self.bs = block_size
        self.chunk_budget, self.max_decode = chunk_budget, max_decode
        self.num_blocks = num_blocks
        self.free_blocks = num_blocks
        self.free_slots = deque(range(max_reqs))
        self.waiting: deque[Request] = deque()     # arrived, prompt not fully prefilled (FCFS)
        self.running: list[Request] = []           # prompt done, decoding (admission order)
        self.finished: list[Request] = []
        self.rejected: list[Request] = []        # can never fit the pool, even alone
        self.n_admit = 0

    def blocks(self, tokens: int) -> int:
        return -(-tokens // self.bs)  # semipd_blocks_for_tokens

    def add(self, reqs):
        for r in reqs:
            q = Request(r.rid, int(r.input_len), int(r.output_len))
            if self.blocks(q.input_len + q.output_len) > self.num_blocks:
                self.rejected.append(q)  # admission could only livelock (S:331 waits forever)
            else:
                self.waiting.append(q)

    @property
    def idle(self) -> bool:
        return not self.waiting and not self.running

    def plan(self):
        """-> (Plan, allocs [(slot, n_blocks)] in call order, preempted requests)."""
        plan = Plan()
        allocs = []
        # decode first: every running request steps (cap max_decode); a request whose next
        # slot opens a new block needs one (R8: blocks are taken before layer 0)
        for r in self.running[:self.max_decode]:
            need = self.blocks(r.ctx + 1) - r.nblk
            if need > self.free_blocks:
                continue  # stalls this iteration (its blocks stay resident)
            if need > 0:
                self.free_blocks -= need
                r.nblk += need
                allocs.append((r.slot, need))
            plan.decode.append((r, r.ctx))
        # the decode batch goes to the device longest context first: the persistent decode
        # grids take units in batch order, so this is LPT scheduling of the requests (the
        # outputs are per row; the order changes no result, R26)
        plan.decode.sort(key=lambda rc: -rc[1])
        # prefill: FCFS chunk budget; headroom of one block per running request keeps
        # decode from starving (a waiting request never takes the last blocks)
        budget = self.chunk_budget
        headroom = len(self.running)
        for r in list(self.waiting):
            if budget == 0:
                break
            chunk = min(r.input_len - r.prefilled, budget)
            need = self.blocks(r.prefilled + chunk) - r.nblk
            if need > self.free_blocks - headroom:
                break  # FCFS: the head waits
            if r.slot < 0:
                if not self.free_slots:
                    break
                r.slot = self.free_slots.popleft()
                r.admit_seq = self.n_admit
                self.n_admit += 1
            if need > 0:
                self.free_blocks -= need
                r.nblk += need
                allocs.append((r.slot, need))
            plan.prefill.append((r, chunk, r.prefilled))
            budget -= chunk
        preempt = []
        if not plan.decode and not plan.prefill:
            # nothing can run on a full pool: recompute-preempt the newest block holder
            # (running, or partially prefilled); the oldest request then always progresses
            holders = self.running + [r for r in self.waiting if r.nblk > 0]
            if holders:
                victim = max(holders, key=lambda r: r.admit_seq)
                if victim in self.running:
                    self.running.remove(victim)
                preempt.append(victim)
        return plan, allocs, preempt

    def finishing(self, plan: Plan):
        """Requests whose decode step in `plan` is their last (freed after the iteration)."""
        return [r for r, _ in plan.decode if r.generated + 1 >= r.output_len]

    def commit(self, plan: Plan, preempt) -> tuple[int, int, list]:
        """Host state after the iteration ran: -> (prefill pairs, decode keys, finished)."""
        pairs = 0
        for r, ch, pf in plan.prefill:
            pairs += ch * pf + ch * (ch + 1) // 2
            r.prefilled += ch
            if r.prefilled == r.input_len:
                self.waiting.remove(r)
                self.running.append(r)
        finished = self.finishing(plan)
        dkeys = 0
        for r, ctx in plan.decode:
            dkeys += ctx + 1
            r.generated += 1
        for r in finished:
            self.running.remove(r)
        for r in finished + list(preempt):
            self.free_blocks += r.nblk
            r.nblk = 0
            self.free_slots.append(r.slot)
            r.slot = -1
        for v in preempt:  # recompute: the request restarts from its prompt
            v.prefilled, v.generated = 0, 0
            v.preempted += 1
            if v not in self.waiting:
                self.waiting.appendleft(v)
        self.finished.extend(finished)
        return pairs, dkeys, finished


class CoRunEngine:
    def __init__(self, pool: KVPool, num_q_heads: int, scale: float, *, chunk_budget: int = 2048,
                 max_decode: int = 512, partition=(50.0, 50.0), seed: int = 0,
                 max_ctx: int = 8192 + 2048, mla_expanded: bool = False):
        c = pool.cfg
        self.pool, self.c = pool, c
        self.dev = pool.device
        self.Hq, self.scale = num_q_heads, scale
        self.L = c.num_layers
        self.bs = c.block_size
        self.chunk_budget, self.max_decode = chunk_budget, max_decode
        self.sched = Scheduler(c.num_blocks, c.block_size, c.max_reqs, chunk_budget=chunk_budget,
                               max_decode=max_decode)
        self.it = 0
        pool.set_partition(*partition)
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        dk, dv = c.head_dim_k, c.head_dim_v
        bf = torch.bfloat16
        rnd = lambda *s: torch.randn(*s, device=self.dev, generator=g).to(bf)  # noqa: E731
        # expanded-form MLA prefill (include/semipd.h semipd_prefill_mla_expanded, reading R32):
        # q [T, H, 192], the chunk's latent rows [T, 576], per-layer up-projections W_UK / W_UV
        # [H, 128, 512] (random, scaled to unit-size outputs); out [T, H, 128]
        self.mla_exp = mla_expanded
        if mla_expanded:
            assert c.kv_shared and dk == 576
            self.w_uk = [(rnd(num_q_heads, 128, 512).float() / 512 ** 0.5).to(bf) for _ in range(self.L)]
            self.w_uv = [(rnd(num_q_heads, 128, 512).float() / 512 ** 0.5).to(bf) for _ in range(self.L)]
            self.ws_exp, self.ws_exp_cap = None, (0, 0)
        self.q_pre = rnd(chunk_budget, num_q_heads, 192 if mla_expanded else dk)
        self.k_pre = rnd(chunk_budget, c.num_kv_heads, dk)
        self.v_pre = None if c.kv_shared else rnd(chunk_budget, c.num_kv_heads, dv)
        self.q_dec = rnd(max_decode, num_q_heads, dk)
        self.k_dec = rnd(max_decode, c.num_kv_heads, dk)
        self.v_dec = None if c.kv_shared else rnd(max_decode, c.num_kv_heads, dv)
        # layer 0 writes its own outputs (kept for parity sampling); other layers share one
        dv_pre = 128 if mla_expanded else dv
        self.o_pre = [torch.empty(chunk_budget, num_q_heads, dv_pre, dtype=bf, device=self.dev)
                      for _ in range(2)]
        self.o_dec = [torch.empty(max_decode, num_q_heads, dv, dtype=bf, device=self.dev)
                      for _ in range(2)]
        self.ws = pool.new_decode_workspace(max_decode, num_q_heads, max_ctx)
        self.max_ctx = max_ctx
        i32 = dict(dtype=torch.int32)
        self.h_meta = torch.zeros(4 * 4096, **i32).pin_memory()
        self.d_meta = torch.zeros(4 * 4096, **i32, device=self.dev)
        self.status = torch.zeros(8192, **i32, device=self.dev)
        self.sCtl, self.sP, self.sD = (torch.cuda.Stream(device=self.dev) for _ in range(3))
        self.ev_prev_p = None

    def add(self, reqs):
        self.sched.add(reqs)

    @property
    def finished(self):
        return self.sched.finished

    # ------------------------------------------------------------------ one iteration
    def step(self, arrivals=()) -> tuple[IterStats, Plan]:
        self.sched.add(arrivals)
        plan, allocs, preempt = self.sched.plan()
        pool, dev = self.pool, self.dev
        n_p, n_d = len(plan.prefill), len(plan.decode)
        # metadata: [cu_seqlens (n_p+1) | req_ids (n_p) | prefix (n_p) | dec rids | dec ctx |
        #            alloc ids | alloc counts | free ids]
        finished = self.sched.finishing(plan)
        frees = [r.slot for r in finished] + [v.slot for v in preempt]
        meta, off = [], {}

        def put(name, xs):
            off[name] = len(meta)
            meta.extend(int(x) for x in xs)

        cu = [0]
        for _, ch, _ in plan.prefill:
            cu.append(cu[-1] + ch)
        put("cu", cu)
        put("prid", [r.slot for r, _, _ in plan.prefill])
        put("pre", [pf for _, _, pf in plan.prefill])
        put("drid", [r.slot for r, _ in plan.decode])
        put("dctx", [ctx for _, ctx in plan.decode])
        put("aid", [a for a, _ in allocs])
        put("acnt", [n for _, n in allocs])
        put("fid", frees)
        assert len(meta) <= self.h_meta.numel()
        self.h_meta[:len(meta)] = torch.tensor(meta, dtype=torch.int32)
        d = self.d_meta

        def view(name, n):
            return d[off[name]:off[name] + n]

        ev = {k: torch.cuda.Event(enable_timing=True) for k in ("i0", "i1", "p0", "p1", "d0", "d1")}
        self.status.zero_()
        st_i = 0
        with torch.cuda.stream(self.sCtl):
            ev["i0"].record(self.sCtl)
            d[:len(meta)].copy_(self.h_meta[:len(meta)], non_blocking=True)
            # S10: one all-or-nothing call per request
            for j in range(len(allocs)):
                pool.alloc_blocks(view("aid", len(allocs))[j:j + 1], view("acnt", len(allocs))[j:j + 1],
                                  status=self.status[st_i:st_i + 1], stream=self.sCtl)
                st_i += 1
        ev_alloc = torch.cuda.Event()
        ev_alloc.record(self.sCtl)
        T = cu[-1]
        max_chunk = max((ch for _, ch, _ in plan.prefill), default=0)
        if n_p and self.mla_exp:
            keys = sum(ch + pf for _, ch, pf in plan.prefill)
            if self.ws_exp is None or n_p > self.ws_exp_cap[0] or keys > self.ws_exp_cap[1]:
                cap = (max(n_p, 2 * self.ws_exp_cap[0], 8), max(keys, 2 * self.ws_exp_cap[1], 4096))
                torch.cuda.synchronize(self.dev)  # earlier iterations may still read the old one
                self.ws_exp = pool.new_mla_expanded_workspace(cap[0], cap[1], self.Hq)
                self.ws_exp_cap = cap
            self.sP.wait_event(ev_alloc)
            ev["p0"].record(self.sP)
            for l in range(self.L):
                pool.prefill_mla_expanded(l, self.q_pre[:T], self.k_pre[:T, 0], self.w_uk[l],
                                          self.w_uv[l], view("cu", n_p + 1), view("prid", n_p),
                                          view("pre", n_p), T, max_chunk, keys, 1 / 192 ** 0.5,
                                          self.o_pre[min(l, 1)][:T], self.ws_exp,
                                          status=self.status[st_i + l:st_i + l + 1], stream=self.sP)
            st_i += self.L
            ev["p1"].record(self.sP)
        elif n_p:
            self.sP.wait_event(ev_alloc)
            ev["p0"].record(self.sP)
            for l in range(self.L):
                pool.prefill_attn(l, self.q_pre[:T], self.k_pre[:T],
                                  None if self.v_pre is None else self.v_pre[:T],
                                  view("cu", n_p + 1), view("prid", n_p), view("pre", n_p), T,
                                  max_chunk, self.scale, self.o_pre[min(l, 1)][:T],
                                  status=self.status[st_i + l:st_i + l + 1], stream=self.sP)
            st_i += self.L
            ev["p1"].record(self.sP)
        if n_d:
            self.sD.wait_event(ev_alloc)
            if self.ev_prev_p is not None:
                self.sD.wait_event(self.ev_prev_p)  # H4: prefill -> decode handoff
            ev["d0"].record(self.sD)
            max_ctx = max(ctx for _, ctx in plan.decode)
            for l in range(self.L):
                pool.decode_attn(l, self.q_dec[:n_d], self.k_dec[:n_d],
                                 None if self.v_dec is None else self.v_dec[:n_d],
                                 view("drid", n_d), view("dctx", n_d), max_ctx, self.scale,
                                 self.o_dec[min(l, 1)][:n_d], self.ws,
                                 status=self.status[st_i + l:st_i + l + 1], stream=self.sD)
            st_i += self.L
            ev["d1"].record(self.sD)
        if n_p:
            self.sCtl.wait_stream(self.sP)
            self.ev_prev_p = ev["p1"]
        if n_d:
            self.sCtl.wait_stream(self.sD)
        with torch.cuda.stream(self.sCtl):
            if frees:
                pool.free_blocks(view("fid", len(frees)), status=self.status[st_i:st_i + 1],
                                 stream=self.sCtl)
                st_i += 1
            ev["i1"].record(self.sCtl)
        ev["i1"].synchronize()
        bad = torch.nonzero(self.status[:st_i]).flatten().tolist()
        if bad:
            raise RuntimeError(f"iteration {self.it}: device status {self.status[bad].tolist()}")
        pairs, dkeys, finished = self.sched.commit(plan, preempt)
        el = lambda a, b: ev[a].elapsed_time(ev[b])  # noqa: E731
        s = IterStats(self.it, n_p, T, pairs, n_d, dkeys,
                      el("p0", "p1") if n_p else 0.0, el("d0", "d1") if n_d else 0.0,
                      el("i0", "i1"), len(allocs), 1 if frees else 0, self.sched.free_blocks,
                      len(finished), len(preempt))
        self.it += 1
        return s, plan

    @property
    def idle(self) -> bool:
        return self.sched.idle


def mla_flops_per_pair(shape_dk: int, shape_dv: int, Hq: int) -> float:
    """Attention FLOPs per unmasked (q, k) pair (all heads, one layer): 2 Hq (dk + dv)."""
    return 2.0 * Hq * (shape_dk + shape_dv)


__all__ = ["CoRunEngine", "Scheduler", "Request", "IterStats", "Plan", "mla_flops_per_pair"]
