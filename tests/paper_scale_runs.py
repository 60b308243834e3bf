"""Paper-scale runs on the GPU path -- an evaluation script, not a test
(it sits in tests/ because it replays sampled replicas with the oracle to check parity at these
budgets; only tests/ may load oracle/).

  qkp300   PAPER.md:163-175 (Fig. 3): a 300-item, 50%-density QKP instance (synthetic analogue of
           300-50-8), P = 2dN, Table I budget K = 2000 SA runs x 1000 MCS, beta_max = 10, eta = 20.
  mkp250   PAPER.md:314-333 (Fig. 5): MKP 250 items x 5 constraints, tightness 0.25/0.5/0.75
           (Chu-Beasley-shaped generator, R15), P = 5dN (~10), K = 5000 x 1000 MCS, beta_max = 50,
           eta = 0.05.
  penalty  PAPER.md:300 (NEXT-1): the penalty method's long single anneals ("10 SA runs of 2x10^5
           MCS") at eta = 0 against SAIM's 2000 x 1000 MCS at the same total budget, n = 100,
           d in {0.25, 0.5}.

Each study launches the statistics replicas and, with another seed in a separate launch, a larger
set of independent runs whose best feasible cost is the "best-known" reference for the accuracy
(accuracy = 100 c(x)/OPT over feasible samples; the paper's instance optima
are not available).  Sampled replicas of the statistics runs are replayed by the
oracle at the full budget and compared element-wise.

  python tests/paper_scale_runs.py {qkp300,mkp250,penalty} --out profiles/r02
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import saim_inputs as si  # noqa: E402
import paper_2501_04971_b200 as P  # noqa: E402


def gpu(probs, alpha, eta, beta_max, seed, R, K, T, trace=True):
    import torch
    Q, c, A, b = si.stack(probs)
    sol = P.Solver(Q, c, A, b, [si.paper_P(p, alpha) for p in probs], eta, beta_max)
    inst = [sol.instance(s) for s in range(len(probs))]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = sol.run(seed, R, K, T, trace=trace, final=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res = {k: v.cpu().numpy() for k, v in out.items()}
    res["counters"] = P.counters_dict(out["counters"])
    res["seconds"] = dt
    res["inst"] = inst
    sol.close()
    return res


def accuracy(f, feas, ref):
    if ref is None or not feas.any():
        return {"feasible_pct": float(100.0 * feas.mean()), "best_acc": None, "avg_acc": None, "optimal_pct": None}
    acc = 100.0 * f[feas] / ref
    return {"feasible_pct": float(100.0 * feas.mean()), "best_acc": float(acc.max()), "avg_acc": float(acc.mean()),
            "optimal_pct": float(100.0 * (f[feas] == ref).mean())}


def best_known(res, s):
    bf = res["best_f"][s]
    ok = bf != np.iinfo(np.int64).max
    return int(bf[ok].min()) if ok.any() else None


def oracle_check(prob, alpha, eta, beta_max, seed, rep, K, T, g, s):
    """Replay replica `rep` (global index) of instance s with the oracle; element-wise compare."""
    import oracle
    op = oracle.OracleProblem.from_inputs(prob, si.paper_P(prob, alpha), eta, beta_max, inst=s)
    t0 = time.perf_counter()
    o = op.run(seed, 1, K, T, rep0=rep, trace=True, final=True, nthreads=1)
    WN = (op.N + 31) // 32
    same = {
        "x_k": bool(np.array_equal(g["tr_x"][s, rep].view(np.uint32)[:, :WN], o["tr_x"][0])),
        "f": bool(np.array_equal(g["tr_f"][s, rep], o["tr_f"][0])),
        "feasible": bool(np.array_equal(g["tr_feas"][s, rep], o["tr_feas"][0])),
        "r": bool(np.array_equal(g["tr_r"][s, rep], o["tr_r"][0])),
        "Lambda": bool(np.array_equal(g["tr_lam"][s, rep], o["tr_lam"][0])),
        "best": bool(g["best_f"][s, rep] == o["best_f"][0] and g["best_k"][s, rep] == o["best_k"][0]),
        "flips": bool(int(g["rep_flips"][s, rep]) == o["counters"]["flips"]),
    }
    return {"replica": rep, "instance": s, "K": K, "T": T, "decisions": o["counters"]["decisions"],
            "oracle_seconds": time.perf_counter() - t0, "near_ties_2^-20": o["counters"]["near_ties"],
            "all_equal": all(same.values()), "fields": same}


def lam_series(res, s, reps, eta, s_c):
    """lambda_k = (eta / s_c) Lambda_k (R10), mean over the given replicas, per constraint row."""
    L = res["tr_lam"][s, reps].astype(np.float64) * (eta / s_c)      # [R, K, M]
    return L.mean(axis=0)                                             # [K, M]


def window(x, w):
    return [float(v) for v in x.reshape(-1, w).mean(axis=1)]


def study_qkp300(a):
    prob = si.qkp(300, 0.5, [20, 0, 8], name="qkp_n300_d0.5 (300-50-8 analogue)")
    K, T, R = 2000, 1000, 64
    stats = gpu([prob], 2.0, 20.0, 10.0, 1, R, K, T)
    ref_run = gpu([prob], 2.0, 20.0, 10.0, 1001, a.ref_R, K, T, trace=False)
    ref = best_known(ref_run, 0)
    f, feas = stats["tr_f"][0], stats["tr_feas"][0].astype(bool)
    s_c = stats["inst"][0]["s_c"]
    lam = lam_series(stats, 0, list(range(R)), 20.0, s_c)[:, 0]
    first_feas = [int(np.argmax(feas[r])) if feas[r].any() else None for r in range(R)]
    out = {"study": "NEXT-2 QKP (PAPER.md:163-175, Fig. 3 analogue)", "instance": prob.name, "N": stats["inst"][0]["N"],
           "P": si.paper_P(prob, 2.0), "eta": 20.0, "beta_max": 10.0, "R": R, "K": K, "T": T,
           "gpu_seconds": stats["seconds"], "best_known": ref,
           "best_known_from": f"{a.ref_R} independent runs (seed 1001, separate launch), {ref_run['seconds']:.1f} s",
           "saim": accuracy(f, feas, ref),
           "saim_best_per_run_acc": [None if b == np.iinfo(np.int64).max else float(100.0 * b / ref) for b in stats["best_f"][0]][:16],
           "first_feasible_k_median": float(np.median([k for k in first_feas if k is not None])) if any(k is not None for k in first_feas) else None,
           "feasible_pct_per_200_iterations": window(feas.mean(axis=0) * 100.0, 200),
           "lambda_mean_per_200_iterations": window(lam, 200),
           "lambda_star_last500_mean": float(lam[-500:].mean()), "lambda_star_last500_std_over_k": float(lam[-500:].std()),
           "counters": stats["counters"],
           "oracle_parity": oracle_check(prob, 2.0, 20.0, 10.0, 1, 0, K, T, stats, 0) if not a.no_oracle else None}
    trace = np.stack([np.arange(K), f[0], feas[0].astype(int), stats["tr_lam"][0, 0, :, 0] * (20.0 / s_c)], axis=1)
    return out, {"qkp300_trace_replica0.csv": ("k,f,feasible,lambda", trace)}


def study_mkp250(a):
    ts = [0.25, 0.5, 0.75]
    probs = [si.mkp(250, 5, t, [21, v, 0], name=f"mkp_n250_m5_t{t}") for v, t in enumerate(ts)]
    K, T, R = 5000, 1000, 64
    stats = gpu(probs, 5.0, 0.05, 50.0, 1, R, K, T)
    ref_run = gpu(probs, 5.0, 0.05, 50.0, 1001, a.ref_R, K, T, trace=False)
    rows, files = [], {}
    for s, prob in enumerate(probs):
        ref = best_known(ref_run, s)
        f, feas = stats["tr_f"][s], stats["tr_feas"][s].astype(bool)
        s_c = stats["inst"][s]["s_c"]
        lam = lam_series(stats, s, list(range(R)), 0.05, s_c)               # [K, M]
        # stabilisation: first k after which the 100-iteration running mean of every row stays
        # within 5% of its final (last 1000) mean
        final = lam[-1000:].mean(axis=0)
        run = np.stack([np.convolve(lam[:, m], np.ones(100) / 100, mode="valid") for m in range(lam.shape[1])], axis=1)
        ok = np.all(np.abs(run - final) <= 0.05 * np.abs(final), axis=1)
        stab = None
        for k in range(len(ok)):
            if ok[k:].all():
                stab = int(k + 99)
                break
        rows.append({"instance": prob.name, "N": stats["inst"][s]["N"], "P": si.paper_P(prob, 5.0),
                     "best_known": ref, "saim": accuracy(f, feas, ref),
                     "feasible_pct_per_500_iterations": window(feas.mean(axis=0) * 100.0, 500),
                     "lambda_rows_mean_at_k": {str(k): [float(v) for v in lam[k]] for k in (0, 100, 500, 1000, 2000, 4999)},
                     "lambda_stabilised_at_k": stab})
        files[f"mkp250_t{prob.name.split("_t")[-1]}_lambda_mean.csv"] = (
            "k," + ",".join(f"lambda_{m}" for m in range(lam.shape[1])),
            np.concatenate([np.arange(K)[:, None], lam], axis=1)[::10])
    out = {"study": "NEXT-2 MKP (PAPER.md:314-333, Fig. 5 analogue)", "eta": 0.05, "beta_max": 50.0, "R": R, "K": K, "T": T,
           "gpu_seconds": stats["seconds"],
           "best_known_from": f"{a.ref_R} independent runs per instance (seed 1001, separate launch), {ref_run['seconds']:.1f} s",
           "instances": rows, "counters": stats["counters"],
           "oracle_parity": oracle_check(probs[1], 5.0, 0.05, 50.0, 1, 0, K, T, stats, 1) if not a.no_oracle else None}
    return out, files


def study_penalty(a):
    cases = [("qkp_n100_d0.25_a", si.qkp(100, 0.25, [7, 0, 0])), ("qkp_n100_d0.25_b", si.qkp(100, 0.25, [7, 0, 1])),
             ("qkp_n100_d0.5_a", si.qkp(100, 0.5, [7, 1, 0])), ("qkp_n100_d0.5_b", si.qkp(100, 0.5, [7, 1, 1]))]
    R = 64
    rows = []
    parity = None
    for name, prob in cases:
        saim = gpu([prob], 2.0, 20.0, 10.0, 1, R, 2000, 1000)
        pen = gpu([prob], 2.0, 0.0, 10.0, 1, R, 10, 200000)
        ref_run = gpu([prob], 2.0, 20.0, 10.0, 1001, a.ref_R, 2000, 1000, trace=False)
        ref = best_known(ref_run, 0)
        rows.append({"instance": name, "best_known": ref,
                     "saim_2000x1000": accuracy(saim["tr_f"][0], saim["tr_feas"][0].astype(bool), ref),
                     "penalty_10x200000": accuracy(pen["tr_f"][0], pen["tr_feas"][0].astype(bool), ref),
                     "gpu_seconds": {"saim": saim["seconds"], "penalty": pen["seconds"]}})
        if parity is None and not a.no_oracle:
            parity = oracle_check(prob, 2.0, 0.0, 10.0, 1, 0, 10, 200000, pen, 0)
    return {"study": "NEXT-1 penalty method, long anneals vs SAIM at equal budget (PAPER.md:300-302)",
            "budget_per_run_MCS": 2000000, "R": R, "P": "2dN", "beta_max": 10.0,
            "best_known_from": f"{a.ref_R} independent SAIM runs per instance (seed 1001, separate launch)",
            "instances": rows, "oracle_parity_penalty_T200000": parity}, {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("study", choices=["qkp300", "mkp250", "penalty"])
    ap.add_argument("--out", default="profiles/r02")
    ap.add_argument("--ref-R", type=int, default=1024)
    ap.add_argument("--no-oracle", action="store_true")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    fn = {"qkp300": study_qkp300, "mkp250": study_mkp250, "penalty": study_penalty}[a.study]
    out, files = fn(a)
    with open(os.path.join(a.out, f"next_{a.study}.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    for name, (hdr, arr) in files.items():
        np.savetxt(os.path.join(a.out, name), arr, delimiter=",", header=hdr, comments="", fmt="%.6g")
    print(json.dumps(out)[:3000])


if __name__ == "__main__":
    main()
