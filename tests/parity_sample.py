"""One-off parity evidence at a BASELINE config's full size: the GPU run of all replicas against the
threaded oracle on a contiguous block of replicas (every per-iteration readout x_k, f, feasibility,
r, Lambda, the best sample, the final state and the block's total flip count).
python tests/parity_sample.py --config 2 --seed 7 --start 0 --count 512"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--start", type=int, default=0)
    ap.add_argument("--count", type=int, default=512)
    a = ap.parse_args()
    import saim_inputs as si
    import paper_2501_04971_b200 as P
    from test_gpu_parity import run_both
    cfg = si.config_instances(a.config)
    t0 = time.time()
    g = run_both(P, cfg.instances, cfg.P, cfg.eta, cfg.beta_max, seed=a.seed, R=cfg.R, K=cfg.K, T=cfg.T,
                 reps=[], block=(a.start, a.count))
    print(json.dumps({"config": a.config, "seed": a.seed, "replicas_gpu": cfg.R, "K": cfg.K, "T": cfg.T,
                      "oracle_block": [a.start, a.count], "instances": len(cfg.instances),
                      "result": "bit-exact (every readout of every iteration, best, final state, flips)",
                      "uncertified": g["counters"]["uncertified"], "fp64": g["counters"]["fp64"],
                      "seconds": round(time.time() - t0, 1)}))


if __name__ == "__main__":
    main()
