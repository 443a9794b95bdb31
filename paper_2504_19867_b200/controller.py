"""SLO-aware dynamic partition controller (PAPER §5: Alg. 1, Eqs. 1-4).

Host-side decision logic on top of the hot path: it picks the (x, y)
SM partition that `semipd_set_partition` applies at each phase's next launch.

  Eq. 1  l_x = 100 / x * l_100                       (processing latency vs SM share)
  Eq. 2  w = 1 / (mu_x - r)                          (M/M/1 wait + service)
  Eq. 3  w ~ 1 / (x - lambda),  lambda = 100 r l_100
  Eq. 4  TTFT_x = a1 / (x - lambda) + b1,   TPOT_y = a2 / y + b2

Readings (R22): Alg. 1's `step` is incremented once per loop
iteration; observed percentiles decide the fail branches, the fitted model is used only
inside the while loops; estimates use the normalised shares x' = 100 x / (x + y)
(lines 11, 16); lambda is fitted by a 0.25 % grid search with OLS at each lambda.  Until a
side has been observed at two distinct shares (no fit), a failing SLO takes one probing step
(R24).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field


@dataclass
class SloConfig:
    ttft_slo: float           # S^p, seconds
    tpot_slo: float           # S^d, seconds
    percentile: float = 0.9   # p^SLO in (0, 1]

    def __post_init__(self):
        if not (self.ttft_slo > 0 and self.tpot_slo > 0 and 0 < self.percentile <= 1):
            raise ValueError("invalid SLO config")


@dataclass
class ControllerConfig:
    window_size: int = 200    # iterations between adjustments
    max_step: int = 6
    step_size: float = 5.0    # percent per step

    def __post_init__(self):
        if not (self.window_size > 0 and self.max_step > 0 and self.step_size > 0):
            raise ValueError("invalid controller config")


@dataclass
class LatencyModel:
    a1: float = 0.0
    b1: float = 0.0
    lam: float = 0.0
    a2: float = 0.0
    b2: float = 0.0
    r2_ttft: float | None = None
    r2_tpot: float | None = None
    fitted_ttft: bool = False
    fitted_tpot: bool = False
    degraded: bool = False

    def estimate_ttft(self, x_norm: float) -> float:
        """Eq. 4; x_norm <= lambda is the unstable queue (Eq. 2 needs mu_x > r): +inf."""
        if x_norm <= self.lam:
            return math.inf
        return self.a1 / (x_norm - self.lam) + self.b1

    def estimate_tpot(self, y_norm: float) -> float:
        if y_norm <= 0:
            return math.inf
        return self.a2 / y_norm + self.b2


def scaled_latency(l100: float, share: float) -> float:
    """Eq. 1: l_x = 100 / x * l_100."""
    if share <= 0:
        raise ValueError("share must be > 0")
    return 100.0 / share * l100


def nearest_rank(values, p: float):
    """p-th percentile, nearest-rank definition (SPEC); None if empty."""
    vals = sorted(values)
    if not vals:
        return None
    k = max(1, math.ceil(p * len(vals)))
    return vals[k - 1]


def _ols(xs, ys):
    """y = a x + b by least squares; returns (a, b, r2)."""
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    a = sxy / sxx if sxx > 0 else 0.0
    b = my - a * mx
    ss_res = sum((y - (a * x + b)) ** 2 for x, y in zip(xs, ys))
    ss_tot = sum((y - my) ** 2 for y in ys)
    r2 = 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0
    return a, b, r2, ss_res


def fit_tpot(y_norms, tpots):
    """OLS of TPOT against 1 / y' (Eq. 4 right)."""
    a2, b2, r2, _ = _ols([1.0 / y for y in y_norms], list(tpots))
    return a2, b2, r2


def fit_ttft(x_norms, ttfts, grid: float = 0.25, eps: float = 0.5):
    """Eq. 4 left: grid-search lambda in [0, min(x') - eps], OLS of TTFT on
    1 / (x' - lambda) at each lambda, keep the smallest residual."""
    xs, ys = list(x_norms), list(ttfts)
    best = None
    lam = 0.0
    hi = min(xs) - eps
    while lam <= hi + 1e-12:
        a1, b1, r2, res = _ols([1.0 / (x - lam) for x in xs], ys)
        if best is None or res < best[4] - 1e-18:
            best = (a1, b1, lam, r2, res)
        lam += grid
    if best is None:
        raise ValueError("no feasible lambda")
    return best[0], best[1], best[2], best[3]


@dataclass
class Observation:
    x_norm: float
    y_norm: float
    ttft: float | None
    tpot: float | None


@dataclass
class SloController:
    slo: SloConfig
    cfg: ControllerConfig = field(default_factory=ControllerConfig)
    model: LatencyModel = field(default_factory=LatencyModel)
    history: list = field(default_factory=list)

    def update_estimate_model(self, obs: Observation) -> LatencyModel:
        """Alg. 1 line 6: refit with all observations (>= 2 distinct shares per side,
        else the previous fit is kept).  Negative slopes clamp to 0 (degraded)."""
        self.history.append(obs)
        t = [(o.x_norm, o.ttft) for o in self.history if o.ttft is not None]
        d = [(o.y_norm, o.tpot) for o in self.history if o.tpot is not None]
        m = self.model
        if len({round(x, 9) for x, _ in t}) >= 2:
            a1, b1, lam, r2 = fit_ttft([x for x, _ in t], [v for _, v in t])
            if a1 < 0:
                a1, m.degraded = 0.0, True
            m.a1, m.b1, m.lam, m.r2_ttft, m.fitted_ttft = a1, b1, lam, r2, True
        if len({round(y, 9) for y, _ in d}) >= 2:
            a2, b2, r2 = fit_tpot([y for y, _ in d], [v for _, v in d])
            if a2 < 0:
                a2, m.degraded = 0.0, True
            m.a2, m.b2, m.r2_tpot, m.fitted_tpot = a2, b2, r2, True
        return m

    def adjust(self, it: int, x0: float, y0: float, ttft_obs, tpot_obs):
        """Algorithm 1, returns the new (x, y)."""
        if it % self.cfg.window_size > 0:                       # lines 1-2
            return x0, y0
        x, y = x0, y0                                           # line 3
        ttft_fail = ttft_obs is not None and ttft_obs > self.slo.ttft_slo
        tpot_fail = tpot_obs is not None and tpot_obs > self.slo.tpot_slo
        if ttft_fail and tpot_fail:                             # no space for adjustment
            return x0, y0
        step, s = 0, self.cfg.step_size
        m = self.model
        if (ttft_fail and not m.fitted_ttft) or (tpot_fail and not m.fitted_tpot and not ttft_fail):
            # no model yet (< 2 distinct shares observed, R24): one probing step in
            # the failing phase's favour, which also gives the fit its second share
            if ttft_fail:
                return (x + s, y) if x + s <= 100 else ((x, y - s) if y - s > 0 else (x, y))
            return (x, y + s) if y + s <= 100 else ((x - s, y) if x - s > 0 else (x, y))
        if ttft_fail and m.fitted_ttft:                         # lines 8-11
            while step < self.cfg.max_step and m.estimate_ttft(100 * x / (x + y)) > self.slo.ttft_slo:
                if x + s <= 100:                                # increase_x_ratio
                    x += s
                elif y - s > 0:                                 # overflow: reduce y instead
                    y -= s
                else:
                    break
                step += 1
        elif tpot_fail and m.fitted_tpot:                       # lines 13-16
            while step < self.cfg.max_step and m.estimate_tpot(100 * y / (x + y)) > self.slo.tpot_slo:
                if y + s <= 100:
                    y += s
                elif x - s > 0:
                    x -= s
                else:
                    break
                step += 1
        else:
            return x0, y0                                       # line 19
        return x, y
