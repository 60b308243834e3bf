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
    """-DSAIM_PROF copy of libsaim.so (translation units compiled in parallel)."""
    objs = [os.path.join("/tmp", src.replace(".cu", "_prof.o")) for src in B.SOURCES]
    procs = [subprocess.Popen([B.NVCC] + B.FLAGS + ["-DSAIM_PROF", "-c", os.path.join(B.CSRC, src), "-o", obj],
                              stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL) for src, obj in zip(B.SOURCES, objs)]
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed")
    subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out] + objs + ["-lcudart"],
                   check=True, capture_output=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--K", type=int, default=20)
    ap.add_argument("--lib", default=None, help="a prebuilt -DSAIM_PROF libsaim (else built to /tmp)")
    ap.add_argument("--build-only", default=None, help="build the profiling library to this path and exit")
    a = ap.parse_args()
    if a.build_only:
        print(build_prof(a.build_only))
        return
    lib = a.lib or build_prof()
    import paper_2501_04971_b200 as P
    P.LIB_PATH = lib
    import saim_inputs as si
    import torch
    cfg = si.config_instances(a.config)
    sol = P.Solver.from_config(cfg)
    prof = C.CDLL(lib).saim_prof_read
    h = (C.c_ulonglong * 48)()
    sol.run(1, cfg.R, a.K, cfg.T)
    torch.cuda.synchronize()
    prof(h, 1)
    sol.run(2, cfg.R, a.K, cfg.T)
    torch.cuda.synchronize()
    prof(h, 1)
    cyc, it, fl = list(h[:16]), list(h[16:32]), list(h[32:48])
    tot = sum(cyc)
    print(f"config {a.config}, K={a.K}: warp-cycles by 1/16 of the anneal (t range), sweep-loop iterations, flips")
    for b in range(16):
        lo, hi = b * cfg.T // 16, (b + 1) * cfg.T // 16
        print(f"t in [{lo:5d}, {hi:5d}): {100 * cyc[b] / tot:5.1f}% cycles, {it[b]:10d} iterations, "
              f"{fl[b]:10d} flips, {cyc[b] / max(it[b], 1):8.1f} cycles/iteration")


if __name__ == "__main__":
    main()
