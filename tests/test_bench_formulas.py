"""Host-side checks of bench.py's roofline numerators (no GPU): the algorithmic bytes / FLOPs
per launch that `roofline*.achieved` divide by must equal the closed forms of SURVEY §8(a)/(d)
for the cfg-2 workload:
  decode  Σ_r (ctx_r + 1)·Hkv·(dk + dv)·eb + B·Hq·(dk + dv)·eb  = 538.2 MB  (§8(d) cfg 2 row: 538.5 MB
          counts q / o in fp32 partial form; the bench counts the bf16 q in / o out it moves)
  prefill 2·Hq·(dk + dv)·C(C + 1)/2                              = 34.38 GFLOP (P = 0)
  bytes   q + o (C·Hq·(dk+dv)·eb) + k_new / v_new in and their pool copy (2·C·Hkv·(dk+dv)·eb)
"""
import dataclasses
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _workload(mod, block_size=64):
    import synth
    w = mod.Workload.__new__(mod.Workload)  # the formulas only read shapes (no pool, no GPU)
    w.shape = dataclasses.replace(synth.CFG2_LLAMA8B, block_size=block_size)
    w.B, w.ctx, w.C, w.P = mod.DECODE_BATCH, mod.DECODE_CTX, mod.PREFILL_TOKENS, 0
    w.ctx_list = [w.ctx] * w.B
    w.L = w.shape.num_layers
    return w


def test_decode_bytes_closed_form():
    mod = _bench()
    w = _workload(mod)
    B, ctx, Hq, Hkv, d = 64, 2048, 32, 8, 128
    assert (w.B, w.ctx) == (B, ctx)
    kv = B * (ctx + 1) * Hkv * (d + d) * 2
    io = B * Hq * (d + d) * 2
    assert w.decode_bytes_per_launch() == kv + io
    assert abs(w.decode_bytes_per_launch() / 1e6 - 538.2) < 0.1
    # FP8 (E4M3) pool, reading R31: one byte per cached K / V element, q / o still bf16
    w.kv_fp8 = True
    assert w.decode_bytes_per_launch() == kv // 2 + io
    assert abs(w.decode_bytes_per_launch() / 1e6 - 269.6) < 0.1


def test_prefill_flops_closed_form():
    mod = _bench()
    w = _workload(mod)
    C, Hq, d = 2048, 32, 128
    assert w.C == C
    # brute-force count of unmasked causal pairs for a small chunk, then the closed form
    assert sum(t + 1 for t in range(37)) == 37 * 38 // 2
    flops = 2 * Hq * (d + d) * (C * (C + 1) / 2)
    assert w.prefill_flops_per_launch() == flops
    assert abs(flops / 1e9 - 34.38) < 0.01


def test_prefill_bytes_and_step_bytes():
    mod = _bench()
    w = _workload(mod)
    C, Hq, Hkv, d = 2048, 32, 8, 128
    assert w.prefill_bytes_per_launch() == C * Hq * 2 * d * 2 + 2 * C * Hkv * 2 * d * 2
    step = w.L * (w.decode_bytes_per_launch() + w.prefill_bytes_per_launch())
    assert abs(step / 1e9 - 18.83) < 0.01  # the roofline_step numerator


def test_bytes_independent_of_block_size():
    mod = _bench()
    assert _workload(mod, 16).decode_bytes_per_launch() == _workload(mod, 64).decode_bytes_per_launch()


def test_parallelism_label_names_the_gather():
    import dataclasses
    import bench
    shape = dataclasses.replace(bench.MODELS["llama3-8b"], block_size=64)
    assert bench.workload_config(shape, 1)["parallelism"] == "tp1"
    assert "NCCL" in bench.workload_config(shape, 4)["parallelism"]
    assert "copy-engine" in bench.workload_config(shape, 4, "peer")["parallelism"]
    assert "epilogues" in bench.workload_config(shape, 8, "fused")["parallelism"]


def test_mla_and_prefix_work_formulas():
    """cfg 5: the latent row (576 x bf16) is read once per key (V aliases K); cfg 4: the
    prefix adds C*P pairs (SURVEY §8(a) FLOP table: 549.8 GFLOP at P = 0, 3.85 TFLOP at
    P = 24576 for C = 8192)."""
    import synth
    mod = _bench()
    mla = synth.CFG5_MLA
    assert mod.decode_bytes(mla, [100, 200]) == (101 + 201) * 576 * 2 + 2 * 16 * (576 + 512) * 2
    s8 = synth.CFG2_LLAMA8B
    assert abs(mod.prefill_flops(s8, 8192, 0) / 1e9 - 549.8) < 0.1
    assert abs(mod.prefill_flops(s8, 8192, 24576) / 1e12 - 3.85) < 0.01


def test_phase_record_fractions():
    """The per-split record divides the algorithmic work by the span-timed launch: decode vs
    the HBM peak, prefill vs the burst peak scaled by the partition's SM share."""
    mod = _bench()
    w = _workload(mod)
    w.pool = type("P", (), {"num_sms": 148})()
    pk = {"hbm": 6500.0, "burst": 1600.0, "sustained": 1400.0}
    ks = {"decode": {"ms": 0.1, "stream_ms": 3.2}, "prefill": {"ms": 0.05, "stream_ms": 1.6}}
    r = mod.phase_record(w, 74, 74, 3.2e-3, ks, pk)
    assert abs(r["decode_gbs"] - w.decode_bytes_per_launch() / 1e-4 / 1e9) < 1e-6
    assert abs(r["decode_frac"] - r["decode_gbs"] / 6500.0) < 1e-12
    tf = w.prefill_flops_per_launch() / 5e-5 / 1e12
    assert abs(r["prefill_frac_share_burst"] - tf / 800.0) < 1e-9
    assert abs(r["prefill_frac_share_sustained"] - tf / 700.0) < 1e-9
    assert abs(r["overlap"] - 0.5) < 1e-12
    assert r["target_score"] == min(r["decode_frac"] / 0.7, r["prefill_frac_share_burst"] / 0.5)
    assert abs(r["tokens_per_s"] - (2048 + 64) / 3.2e-3) < 1e-6


def test_nccl_options_cap_ctas():
    from paper_2504_19867_b200 import tp
    o = tp.nccl_options(4)
    assert o.config.max_ctas == 4 and o.config.min_ctas == 1


def test_mla_expanded_flops_closed_form():
    """Expanded-form MLA prefill (R32): projection 2 x 512 x (2 H 128) per key plus 2 H (192 + 128)
    per unmasked pair; C = 2048, P = 0, H = 16 by hand."""
    mod = _bench()
    pairs = 2048 * 2049 // 2
    assert mod.mla_expanded_flops(16, 2048, 0) == 2 * 2048 * 512 * 4096 + 2 * 16 * 320 * pairs
    assert mod.mla_expanded_flops(16, 2048, 0) == 30_075_256_832
    # a prefix adds P keys to the projection and C x P pairs
    assert mod.mla_expanded_flops(16, 10, 100) == 2 * 110 * 512 * 4096 + 2 * 16 * 320 * (1000 + 55)
