#!/usr/bin/env python
"""Eq. 1 check (feeds N1): does processing latency scale as
l_x = 100/x * l_100 on B200?  From isolated per-budget kernel curves
(scripts/microbench.py output, one JSON line per (kernel, budget)) this reports, per kernel,
t(n) * n / N / t(N) for every budget n (Eq. 1 predicts 1) and the R^2 of the fit
t = a / n + b (cf. fig:modeling).

  python scripts/eq1_check.py profiles/r1_isolated_curves.jsonl [--out profiles/r1_eq1.json]
"""
import argparse
import json
import sys


def fit_inv(ns, ts):
    xs = [1.0 / n for n in ns]
    k = len(xs)
    mx, my = sum(xs) / k, sum(ts) / k
    sxx = sum((x - mx) ** 2 for x in xs)
    a = sum((x - mx) * (y - my) for x, y in zip(xs, ts)) / sxx
    b = my - a * mx
    ss_res = sum((y - (a * x + b)) ** 2 for x, y in zip(xs, ts))
    ss_tot = sum((y - my) ** 2 for y in ts)
    return a, b, 1.0 - ss_res / ss_tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("curves")
    ap.add_argument("--N", type=int, default=148)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    by = {}
    for line in open(args.curves):
        line = line.strip()
        if not line.startswith("{"):
            continue
        r = json.loads(line)
        by.setdefault(r["kernel"], {})[int(r["budget"])] = float(r["ms"])
    out = {}
    for k, d in by.items():
        if args.N not in d or len(d) < 3:
            continue
        ns = sorted(d)
        tN = d[args.N]
        ratio = {n: d[n] * n / args.N / tN for n in ns}
        a, b, r2 = fit_inv(ns, [d[n] for n in ns])
        out[k] = {"budgets": ns, "ms": [d[n] for n in ns],
                  "eq1_ratio_t_n_times_n_over_N_over_t_N": [round(ratio[n], 3) for n in ns],
                  "fit_t_eq_a_over_n_plus_b": {"a_ms_sm": a, "b_ms": b, "r2": r2}}
        print(f"{k}: Eq.1 ratio by budget " +
              ", ".join(f"{n}:{ratio[n]:.2f}" for n in ns) + f"; fit t = {a:.3f}/n + {b:.4f} ms, R^2 = {r2:.4f}")
    if args.out:
        json.dump(out, open(args.out, "w"), indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
