"""Build libsaim.so in-tree with nvcc for sm_100a (B200).  Usage: python -m paper_2501_04971_b200.build"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsaim.so")
SOURCES = ["saim_api.cu", "saim_qkp.cu", "saim_qkp_replay.cu", "saim_mkp.cu", "saim_mkp_replay.cu", "saim_mkp_tree.cu",
           "saim_mkp_tree_replay.cu", "saim_mkp_split.cu", "saim_mkp_split_replay.cu", "saim_mkp_spec.cu", "saim_mkp_spec_replay.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "saim.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    objs = [os.path.join(CSRC, src.replace(".cu", f".{os.getpid()}.o")) for src in SOURCES]
    procs = [subprocess.Popen([NVCC] + FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for src, obj in zip(SOURCES, objs)]
    logs = []
    for src, p in zip(SOURCES, procs):           # translation units compile in parallel
        out, _ = p.communicate()
        logs.append(out)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{out}")
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + objs + ["-lcudart"]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"link failed:\n{p.stdout}\n{p.stderr}")
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    with open(os.path.join(HERE, "build.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
