"""N1: the SLO-aware partition controller in the loop on the GPU (PAPER §5:
Alg. 1, Eqs. 1-4, `fig:modeling` P:339-345).

- fig:modeling from isolated curves: each phase of the cfg-5 MLA workload alone at SM shares
  x in {15, 30, 50, 70, 100} %, timed with the library's device launch spans; the Eq. 1 / 4
  forms l = a / x + b (prefill) and TPOT = a2 / y + b2 (decode) are fitted with the
  controller's own OLS (controller.fit_tpot) and must explain the curves (R^2 > 0.9).
- closed loop: an under-capacity cfg-5 trace (Poisson 0.5 / iteration, 160 requests, 4
  layers) through the co-run engine (scripts/mla_trace.py) first at a fixed (15, 85) split to
  measure p90 TTFT / TPOT, then with Alg. 1 driving semipd_set_partition every 40 iterations
  under a TTFT SLO of 0.7 x the measured p90 (so the prefill side fails) and a loose TPOT
  SLO: the partition must move toward prefill, TTFT attainment must rise, every sampled
  iteration must match the oracle and the device op log must replay bit-exactly."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fig_modeling_fit_from_isolated_curves():
    import importlib.util

    import synth
    from paper_2504_19867_b200.controller import fit_tpot
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    dev = torch.device("cuda", 0)
    import numpy as np
    rng = np.random.default_rng(5005)
    ctx = [int(c) for c in np.clip(rng.lognormal(np.log(350.0) - 0.125, 0.5, 256), 64, 4096)]
    w = bench.Workload(synth.CFG5_MLA, 1, dev, seed=77, B=256, ctx=ctx, C=2048, layers=4)
    run = bench.Runner(w, dev)
    N = w.pool.num_sms
    shares = [15, 30, 50, 70, 100]
    pre, dec = [], []
    for x in shares:
        n = max(1, round(N * x / 100))
        for ph, out in (("prefill", pre), ("decode", dec)):
            fn = (lambda n=n: w.phase_prefill(n, stream=torch.cuda.current_stream(dev))) \
                if ph == "prefill" else (lambda n=n: w.phase_decode(n, stream=torch.cuda.current_stream(dev)))
            step = run.capture(fn)
            run.time(step, 3)
            out.append(w.kernel_stats(order=(ph,))[ph]["ms"])
    a1, b1, r2_pre = fit_tpot(shares, pre)   # l_x = a / x + b (Eq. 1 with a fixed part)
    a2, b2, r2_dec = fit_tpot(shares, dec)   # TPOT_y = a2 / y + b2 (Eq. 4)
    rec = {"shares": shares, "prefill_ms": pre, "decode_ms": dec,
           "prefill_fit": [a1, b1, r2_pre], "decode_fit": [a2, b2, r2_dec]}
    print(json.dumps(rec))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fig_modeling_fit.json"), "w") as f:
        json.dump(rec, f)
    assert all(pre[i] > pre[i + 1] for i in range(len(pre) - 1)), "prefill must speed up with SMs"
    assert a1 > 0 and a2 > 0
    assert r2_pre > 0.9 and r2_dec > 0.9, rec


def _trace(tmp_path, name, *extra):
    out = tmp_path / f"{name}.json"
    cmd = [sys.executable, os.path.join(ROOT, "scripts", "mla_trace.py"), "--requests", "160",
           "--lam", "0.5", "--layers", "4", "--blocks", "2048", "--samples", "3",
           "--out", str(out), *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return json.load(open(out))["summary"]


def test_controller_closed_loop_moves_partition(tmp_path):
    base = _trace(tmp_path, "base", "--x", "15")
    assert base["parity_all_ok"] and base["op_log_replay_tables_equal"]
    ttft_slo = 0.7 * base["p90_ttft_s"]
    tpot_slo = 3.0 * base["p90_tpot_s"]
    ctl = _trace(tmp_path, "ctl", "--x", "15", "--controller", "--window", "40",
                 "--ttft-slo", repr(ttft_slo), "--tpot-slo", repr(tpot_slo))
    assert ctl["parity_all_ok"] and ctl["op_log_replay_tables_equal"]
    c = ctl["controller"]
    traj = c["trajectory"]
    xs = [t["x"] / (t["x"] + t["y"]) for t in traj]
    summary = {"base_p90_ttft_s": base["p90_ttft_s"], "ctl_p90_ttft_s": ctl["p90_ttft_s"],
               "ttft_slo_s": ttft_slo, "tpot_slo_s": tpot_slo,
               "attainment": [c["ttft_slo_attainment"], c["tpot_slo_attainment"]],
               "trajectory": [(t["it"], t["x"], t["y"], t["next"]) for t in traj],
               "model": c["model"]}
    print(json.dumps(summary))
    with open(os.path.join(ROOT, "gpurun_out", "controller_loop.json"), "w") as f:
        json.dump(summary, f)
    moved = [t for t in traj if t["next"] != [t["x"], t["y"]]]
    assert moved, "Alg. 1 never moved the partition"
    assert max(xs) > 0.15 + 1e-9, "the prefill share must grow under a failing TTFT SLO"
    assert ctl["p90_ttft_s"] < base["p90_ttft_s"], summary
    assert c["tpot_slo_attainment"] >= 0.9, summary
