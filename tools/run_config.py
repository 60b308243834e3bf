"""Run one saim_run of a BASELINE config (optionally with K/T/R overrides) -- for ncu captures.
python tools/run_config.py --config 2 --K 4 [--reps 2]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import saim_inputs as si  # noqa: E402
import paper_2501_04971_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--K", type=int, default=None)
    ap.add_argument("--T", type=int, default=None)
    ap.add_argument("--R", type=int, default=None)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--inst", type=int, default=None, help="run only this instance of the config")
    a = ap.parse_args()
    import torch
    cfg = si.config_instances(a.config)
    if a.inst is not None:
        p = cfg.instances[a.inst]
        sol = P.Solver(p.Q, p.c, p.A, p.b, cfg.P[a.inst], cfg.eta, cfg.beta_max, flags=a.flags)
    else:
        sol = P.Solver.from_config(cfg, flags=a.flags)
    R, K, T = a.R or cfg.R, a.K or cfg.K, a.T or cfg.T
    out = sol.alloc_outputs(R, K)
    for i in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sol.run(1 + i, R, K, T, out=out)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        c = P.counters_dict(out["counters"])
        print(f"config {a.config} flags={a.flags} lanes={sol.info['lanes_per_replica']} R={R} K={K} T={T}: {dt*1e3:.2f} ms, {c['decisions']/dt:.3e} updates/s, {c}")
    sol.close()


if __name__ == "__main__":
    main()
