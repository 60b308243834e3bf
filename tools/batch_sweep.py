"""Config-4 replica/instance batching sweep (BASELINE.json config 4): the same total
number of chains (16,384) split as n_inst instances x R replicas in one launch, MKP n=500, M=30,
t=0.5 (config 4's generator), T=2000, K reduced (default 10) so each point takes seconds.
Device time by CUDA events; one JSON line per point.

python tools/batch_sweep.py [--K 10] [--total 16384] [--points 1 4 16 64 128]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import saim_inputs as si  # noqa: E402
import paper_2501_04971_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", type=int, default=10)
    ap.add_argument("--total", type=int, default=16384)
    ap.add_argument("--points", type=int, nargs="*", default=[1, 4, 16, 64, 128])
    ap.add_argument("--flags", type=int, default=0)
    a = ap.parse_args()
    import torch
    base = si.config_instances(4)
    for n_inst in a.points:
        R = a.total // n_inst
        probs = [si.mkp(500, 30, 0.5, [4, 0, s]) for s in range(n_inst)]
        Q, c, A, b = si.stack(probs)
        Ps = [si.paper_P(p, base.alpha) for p in probs]
        sol = P.Solver(Q, c, A, b, Ps, base.eta, base.beta_max, flags=a.flags)
        out = sol.alloc_outputs(R, a.K)
        sol.run(100, R, a.K, base.T, out=out)                     # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sol.run(1, R, a.K, base.T, out=out)
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        cnt = P.counters_dict(out["counters"])
        print(json.dumps({"n_inst": n_inst, "replicas_per_inst": R, "K": a.K, "T": base.T,
                          "kernel_lanes_per_replica": sol.info["lanes_per_replica"], "seconds": t,
                          "updates_per_s": cnt["decisions"] / t, "samples_per_s": R * n_inst * a.K / t,
                          "counters": cnt}), flush=True)
        sol.close()


if __name__ == "__main__":
    main()
