"""Time split of the QKP kernel by anneal phase (development profiling, not the product build).
Builds a -DSAIM_PROF copy of libsaim.so (clock64 totals per sweep phase: t < T/10, [T/10, 3T/10),
the rest; saim_qkp.cu) into /tmp, runs one BASELINE config through it and prints the shares.
python tools/prof_phases.py [--config 2] [--K 20]"""
import argparse
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_04971_b200 import build as B  # noqa: E402


def build_prof(out="/tmp/libsaim_prof.so"):
    objs = []
    for src in B.SOURCES:
        obj = os.path.join("/tmp", src.replace(".cu", "_prof.o"))
        subprocess.run([B.NVCC] + B.FLAGS + ["-DSAIM_PROF", "-c", os.path.join(B.CSRC, src), "-o", obj],
                       check=True, capture_output=True)
        objs.append(obj)
    subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out] + objs + ["-lcudart"],
                   check=True, capture_output=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--K", type=int, default=20)
    a = ap.parse_args()
    lib = build_prof()
    import paper_2501_04971_b200 as P
    P.LIB_PATH = lib
    import saim_inputs as si
    import torch
    cfg = si.config_instances(a.config)
    sol = P.Solver.from_config(cfg)
    prof = C.CDLL(lib).saim_prof_read
    h = (C.c_ulonglong * 8)()
    sol.run(1, cfg.R, a.K, cfg.T)
    torch.cuda.synchronize()
    prof(h, 1)
    sol.run(2, cfg.R, a.K, cfg.T)
    torch.cuda.synchronize()
    prof(h, 1)
    cyc, sw = list(h[:3]), list(h[4:7])
    tot = sum(cyc)
    names = ["t < T/10", "T/10 <= t < 3T/10", "t >= 3T/10"]
    for nm, c, s in zip(names, cyc, sw):
        print(f"{nm:20s} {100 * c / tot:5.1f}% of warp-cycles, {s} warp-sweeps, {c / max(s, 1):8.1f} cycles/sweep")


if __name__ == "__main__":
    main()
