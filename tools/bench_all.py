"""Time one full saim_run of every BASELINE config (device time, CUDA events) and print a table row
per config: updates/s, samples/s, counters.  python tools/bench_all.py [--configs 0 1 2 3 4]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import saim_inputs as si  # noqa: E402
import paper_2501_04971_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[0, 1, 2, 3, 4])
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch
    rows = []
    for c in a.configs:
        cfg = si.config_instances(c)
        sol = P.Solver.from_config(cfg)
        out = sol.alloc_outputs(cfg.R, cfg.K)
        sol.run(100, cfg.R, cfg.K, cfg.T, out=out)            # warm-up
        torch.cuda.synchronize()
        best = None
        for r in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sol.run(1 + r, cfg.R, cfg.K, cfg.T, out=out)
            e1.record()
            e1.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            best = t if best is None else min(best, t)
        cnt = P.counters_dict(out["counters"])
        row = {"config": c, "name": cfg.name, "kernel": sol.info["kernel"], "seconds": best,
               "updates_per_s": cnt["decisions"] / best, "samples_per_s": cfg.R * cfg.K * sol.n_inst / best,
               "counters": cnt}
        rows.append(row)
        print(json.dumps(row), flush=True)
        sol.close()


if __name__ == "__main__":
    main()
