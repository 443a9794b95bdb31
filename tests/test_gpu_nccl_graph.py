"""The N > 1 bench's collective path on the one GPU the round's boxes have:
a one-rank NCCL process group per phase built exactly as bench.py builds them
(tp.PhaseGroups with ncclConfig_t.maxCTAs = 4 through ProcessGroupNCCL.Options), the head
all-gather captured into a CUDA graph with the attention kernel in front of it, and replayed.
With one rank the gather is a copy, so the replayed result must equal the kernel's output bit
for bit; what this checks is that the options are accepted and that the collective is
capturable under this torch / NCCL, which the 8-GPU bench relies on."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _main(port, q):
    try:
        import torch.distributed as dist

        import synth
        from paper_2504_19867_b200 import KVPool, PoolConfig, tp
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        groups = tp.PhaseGroups.create(backend="nccl", max_ctas=4)
        shape = synth.AttnShape("llama3-8b", 32, 8, 128, 128, 64, torch.bfloat16)
        ctx = [300, 2048, 64]
        B = len(ctx)
        dc = synth.decode_case(shape, ctx, seed=6000)
        i32 = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
        nb = [c // 64 + 1 for c in ctx]
        pool = KVPool(PoolConfig(1, sum(nb) + 2, 64, 8, 128, 128, B, max(nb)), dev)
        for b, n in enumerate(nb):
            pool.alloc_blocks(i32([b]), i32([n]))
        K, V, BT, _ = pool.views(0)
        bt = BT.cpu()
        for b, c in enumerate(ctx):
            pos = torch.arange(c)
            blk = bt[b].long()[pos // 64].to(dev)
            K[blk, :, (pos % 64).to(dev)] = dc.k_ctx[b].to(dev)
            V[blk, :, (pos % 64).to(dev)] = dc.v_ctx[b].to(dev)
        qd, kd, vd = dc.q.to(dev), dc.k_new.to(dev), dc.v_new.to(dev)
        od = torch.empty(32, B, 128, dtype=torch.bfloat16, device=dev)
        gd = torch.full((32, B, 128), float("nan"), dtype=torch.bfloat16, device=dev)
        ws = pool.new_decode_workspace(B, 32, max(ctx))
        s = torch.cuda.Stream(dev)
        ids, ctx_d = i32(range(B)), i32(ctx)

        def step():
            pool.decode_attn(0, qd, kd, vd, ids, ctx_d, max(ctx),
                             shape.softmax_scale, od, ws, out_head_major=True,
                             stream=torch.cuda.current_stream(dev))
            tp.gather_heads(od, gd, groups.decode)

        with torch.cuda.stream(s):
            step()  # eager warm-up (communicator + kernels)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        gd.fill_(float("nan"))
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ok = torch.equal(gd.view(torch.int16), od.view(torch.int16))
        dist.destroy_process_group()
        q.put("ok" if ok else "gathered output differs from the kernel output")
    except Exception as e:  # pragma: no cover
        import traceback
        q.put("".join(traceback.format_exception(e))[-3000:])


def test_nccl_phase_group_gather_is_graph_capturable():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_main, args=(_port(), q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=60)
    assert res == "ok", res
