"""bench.py's end-to-end step (host buffers, copies inside the step) computes what the
device-resident step computes: its host outputs equal the device-timed path's outputs bit for bit
(same kernels, same inputs, R26), for the packed per-layer copy layout and the declared copy
bytes cover every input / output tensor."""
import dataclasses
import importlib.util
import os
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod_e2e", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_e2e_step_matches_device_step():
    mod = _bench()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    shape = dataclasses.replace(mod.MODELS["llama3-8b"], block_size=64)
    w = mod.Workload(shape, 1, dev, layers=3, B=16, ctx=700, C=384)
    w.corun_step(30, 70)
    torch.cuda.synchronize()
    ref_p = [t.clone() for t in w.op]
    ref_d = [t.clone() for t in w.od]
    ee = mod.E2E(w)
    assert ee.packed
    tensors_in = sum(t.numel() * t.element_size() for lst in (w.qp, w.kp, w.vp, w.qd, w.kd, w.vd)
                     for t in lst if t is not None)
    tensors_out = sum(t.numel() * t.element_size() for lst in (w.op, w.od) for t in lst)
    assert tensors_in <= ee.h2d < tensors_in + 6 * 4096 * w.L
    assert tensors_out <= ee.d2h < tensors_out + 2 * 4096 * w.L
    for h in ee.h_op + ee.h_od:
        h.zero_()
    ee.step(30, 70)
    torch.cuda.synchronize()
    for l in range(w.L):
        assert torch.equal(ee.h_op[l], ref_p[l].cpu()), f"prefill output of layer {l}"
        assert torch.equal(ee.h_od[l], ref_d[l].cpu()), f"decode output of layer {l}"
