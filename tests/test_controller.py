"""Pins for the SLO-aware controller (PAPER §5 Alg. 1, Eqs. 1-4) against the SPEC
examples (Eq. 1, S:440-471 fit / estimate / adjust) and closed forms."""
import math

import pytest

from paper_2504_19867_b200.controller import (ControllerConfig, LatencyModel, Observation,
                                              SloConfig, SloController, fit_tpot, fit_ttft,
                                              nearest_rank, scaled_latency)


def test_eq1_examples():
    assert scaled_latency(40e-3, 50) == pytest.approx(80e-3)
    assert scaled_latency(40e-3, 100) == pytest.approx(40e-3)
    assert scaled_latency(30e-3, 25) == pytest.approx(120e-3)
    for x in (10, 37, 50, 99):  # l_x * x is constant (Eq. 1 exactness)
        assert scaled_latency(0.03, x) * x == pytest.approx(3.0)


def test_nearest_rank():
    assert nearest_rank([i / 10 for i in range(1, 11)], 0.9) == pytest.approx(0.9)
    assert nearest_rank([0.42], 0.9) == 0.42
    assert nearest_rank([], 0.9) is None


def test_fit_recovers_spec_examples():
    xs = [30, 40, 50, 60, 70, 80, 90]
    a1, b1, lam, r2 = fit_ttft(xs, [5 / (x - 20) + 0.05 for x in xs])
    assert abs(a1 - 5) < 1e-6 and abs(lam - 20) < 1e-6 and abs(b1 - 0.05) < 1e-6
    assert r2 == pytest.approx(1.0)
    ys = [20, 30, 40, 50, 60, 70, 80]
    a2, b2, r2 = fit_tpot(ys, [8 / y + 0.01 for y in ys])
    assert abs(a2 - 8) < 1e-9 and abs(b2 - 0.01) < 1e-9 and r2 == pytest.approx(1.0)


def test_estimates_and_pole():
    m = LatencyModel(a1=5, b1=0.05, lam=20, a2=8, b2=0.01)
    assert m.estimate_ttft(70) == pytest.approx(0.15)
    assert m.estimate_tpot(40) == pytest.approx(0.21)
    assert math.isinf(m.estimate_ttft(20))


def _ctl(**kw):
    c = SloController(SloConfig(0.2, 0.1), ControllerConfig(window_size=10, max_step=6, step_size=5))
    c.model = LatencyModel(fitted_ttft=True, fitted_tpot=True, **kw)
    return c


def test_alg1_examples():
    # both fail -> unchanged (line 19)
    c = _ctl(a1=5, b1=0.05, lam=20, a2=8, b2=0.01)
    assert c.adjust(10, 60, 60, 0.5, 0.5) == (60, 60)
    # not a window boundary -> unchanged (lines 1-2)
    assert c.adjust(7, 60, 60, 0.5, 0.01) == (60, 60)
    # TTFT fails; estimate satisfied after one step -> (65, 60).  With (60,60) x'=50;
    # choose a model where est(50) > S^p and est(100*65/125 = 52) <= S^p.
    c2 = _ctl(a1=1.0, b1=0.0, lam=46.0, a2=1.0, b2=0.0)
    assert c2.model.estimate_ttft(50) > 0.2 and c2.model.estimate_ttft(52) <= 0.2
    assert c2.adjust(10, 60, 60, 0.3, 0.05) == (65, 60)
    # TTFT fails at x = 100: the first step reduces y instead -> (100, 55) when satisfied
    c3 = _ctl(a1=1.0, b1=0.0, lam=58.0, a2=1.0, b2=0.0)
    assert c3.model.estimate_ttft(100 * 100 / 160) > 0.2
    assert c3.model.estimate_ttft(100 * 100 / 155) <= 0.2
    assert c3.adjust(10, 100, 60, 0.3, 0.05) == (100, 55)
    # both pass -> unchanged
    assert c.adjust(20, 40, 70, 0.1, 0.05) == (40, 70)


def test_alg1_invariants_bounded_and_monotone():
    c = _ctl(a1=50, b1=0.1, lam=0, a2=8, b2=0.01)  # TTFT never satisfiable -> max_step steps
    x, y = c.adjust(10, 50, 50, 1.0, 0.01)
    assert (x, y) == (80, 50)                     # 6 steps of 5 percent
    for (x0, y0) in [(95, 95), (100, 10), (5, 100)]:
        x, y = c.adjust(0, x0, y0, 1.0, 0.01)
        assert 0 < x <= 100 and 0 < y <= 100 and x >= x0 and y <= y0
        assert x - x0 <= 30 and y0 - y <= 30


def test_update_model_needs_two_distinct_shares():
    c = SloController(SloConfig(0.2, 0.1))
    m = c.update_estimate_model(Observation(50, 50, 5 / 30 + 0.05, 8 / 50 + 0.01))
    assert not m.fitted_ttft and not m.fitted_tpot
    for x in (30, 40, 60, 70, 80):
        c.update_estimate_model(Observation(x, 100 - x, 5 / (x - 20) + 0.05, 8 / (100 - x) + 0.01))
    assert c.model.fitted_ttft and c.model.fitted_tpot
    assert c.model.r2_tpot > 0.99


def test_closed_loop_convergence_on_exact_model():
    """With the true Eq. 4 model and a stationary load, the controller reaches a
    partition satisfying the TTFT SLO within ceil((x_needed - x0)/step) windows."""
    true = LatencyModel(a1=4, b1=0.02, lam=15, a2=6, b2=0.005, fitted_ttft=True, fitted_tpot=True)
    c = SloController(SloConfig(0.12, 0.2), ControllerConfig(window_size=1, max_step=1,
                                                             step_size=5))
    c.model = true
    x, y = 40.0, 60.0
    for it in range(40):
        xn = 100 * x / (x + y)
        x, y = c.adjust(it, x, y, true.estimate_ttft(xn), true.estimate_tpot(100 * y / (x + y)))
    assert true.estimate_ttft(100 * x / (x + y)) <= 0.12


def test_unfitted_model_takes_one_probing_step():
    """R24: without a fit (one share observed) a failing SLO moves one step toward the
    failing phase; passing SLOs or both failing leave the partition unchanged."""
    c = SloController(SloConfig(0.2, 0.1), ControllerConfig(window_size=10, max_step=6, step_size=5))
    c.update_estimate_model(Observation(50, 50, 0.3, 0.05))
    assert c.adjust(10, 50, 50, 0.3, 0.05) == (55, 50)      # TTFT fails
    assert c.adjust(10, 50, 50, 0.1, 0.2) == (50, 55)       # TPOT fails
    assert c.adjust(10, 100, 50, 0.3, 0.05) == (100, 45)    # TTFT fails at x = 100
    assert c.adjust(10, 50, 50, 0.1, 0.05) == (50, 50)      # both pass
    assert c.adjust(10, 50, 50, 0.3, 0.2) == (50, 50)       # both fail
