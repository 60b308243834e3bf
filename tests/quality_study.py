"""Solution-quality runs on the GPU path: paper-scale budgets
(Table I: K = 2000 SA runs x 1000 MCS for QKP) on synthetic instances shaped like the
paper's, SAIM (eta = 20) vs the penalty method (eta = 0, same P, same budget; PAPER.md:300-302,
Table II), reporting the paper's metrics: feasibility %, best and average
accuracy of feasible samples.  OPT is exact (brute force) for n <= 24; otherwise accuracy is
relative to the best feasible cost found by any run (labelled "best-known").

  python tests/quality_study.py [--R 64] [--K 2000] [--T 1000]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import saim_inputs as si  # noqa: E402
import paper_2501_04971_b200 as P  # noqa: E402
from oracle.reference import brute_force_opt  # noqa: E402  (OPT for tiny instances only)


def run(prob, eta, R, K, T, seed):
    import torch
    sol = P.Solver(prob.Q, prob.c, prob.A, prob.b, si.paper_P(prob, 2.0), eta, 10.0)
    out = sol.run(seed, R, K, T, trace=True)
    torch.cuda.synchronize()
    f = out["tr_f"].cpu().numpy()[0]
    feas = out["tr_feas"].cpu().numpy()[0].astype(bool)
    sol.close()
    return f, feas


def summarize(f, feas, ref):
    """accuracy = 100 c(x)/OPT over feasible samples (costs are negative)."""
    if not feas.any():
        return {"feasible_pct": 0.0, "best_acc": None, "avg_acc": None}
    acc = 100.0 * f[feas] / ref
    return {"feasible_pct": 100.0 * feas.mean(), "best_acc": float(acc.max()), "avg_acc": float(acc.mean())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", type=int, default=64)
    ap.add_argument("--K", type=int, default=2000)
    ap.add_argument("--T", type=int, default=1000)
    a = ap.parse_args()
    cases = [("qkp_n20_d0.5", si.qkp(20, 0.5, [0, 0, 0])), ("qkp_n24_d0.5", si.qkp(24, 0.5, [9, 0, 1])),
             ("qkp_n100_d0.25_a", si.qkp(100, 0.25, [7, 0, 0])), ("qkp_n100_d0.25_b", si.qkp(100, 0.25, [7, 0, 1])),
             ("qkp_n100_d0.5_a", si.qkp(100, 0.5, [7, 1, 0])), ("qkp_n100_d0.5_b", si.qkp(100, 0.5, [7, 1, 1]))]
    for name, prob in cases:
        fs, fe = run(prob, 20.0, a.R, a.K, a.T, 1)
        ps, pe = run(prob, 0.0, a.R, a.K, a.T, 1)
        if prob.n <= 24:
            ref, _ = brute_force_opt(prob.Q, prob.c, prob.A, prob.b)
            ref_kind = "OPT (brute force)"
        else:
            cand = [x[m].min() for x, m in ((fs, fe), (ps, pe)) if m.any()]
            ref = min(cand) if cand else None
            ref_kind = "best-known (min over both methods' samples)"
        row = {"instance": name, "R": a.R, "K": a.K, "T": a.T, "reference": int(ref) if ref is not None else None,
               "reference_kind": ref_kind,
               "saim_eta20": summarize(fs, fe, ref) if ref is not None else None,
               "penalty_eta0": summarize(ps, pe, ref) if ref is not None else None}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
