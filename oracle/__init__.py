"""CPU oracle for the SAIM hot path (arXiv 2501.04971) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg may
import this package.  It shares no code with `paper_2501_04971_b200` (the product path) and never
imports it; the product never imports this.

`saim_oracle.c` is the oracle proper (plain scalar C, fp64 decisions certified with a binary128
fallback, see its header for the paper citations); this module only compiles it with gcc and
marshals numpy arrays through ctypes.  `reference.py` holds pure-Python (fractions) definitions
used to pin the oracle in tests.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "saim_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

FROM_DEFINITION = 0
INCREMENTAL = 1
COUNTER_NAMES = ["decisions", "unsaturated", "flips", "near_ties", "quad_fallbacks", "feasible"]


def build(force: bool = False) -> str:
    """Compile oracle/liboracle.so with gcc (plain C, -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-ffp-contract=off", "-pthread",
            _SRC, "-o", tmp, "-lquadmath", "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Problem(C.Structure):
    _fields_ = [("n", C.c_int32), ("M", C.c_int32),
                ("Q", C.c_void_p), ("c", C.c_void_p), ("A", C.c_void_p), ("b", C.c_void_p),
                ("P", C.c_double), ("eta", C.c_double), ("beta_max", C.c_double),
                ("inst", C.c_int32)]


class _RunArgs(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("rep0", C.c_int32), ("nrep", C.c_int32),
                ("K", C.c_int32), ("T", C.c_int32), ("field_mode", C.c_int32),
                ("nthreads", C.c_int32), ("x_init", C.c_void_p)]


class _Out(C.Structure):
    _fields_ = [("best_f", C.c_void_p), ("best_x", C.c_void_p), ("best_k", C.c_void_p),
                ("n_feasible", C.c_void_p), ("tr_f", C.c_void_p), ("tr_feas", C.c_void_p),
                ("tr_r", C.c_void_p), ("tr_lam", C.c_void_p), ("tr_x", C.c_void_p),
                ("final_x", C.c_void_p), ("final_lam", C.c_void_p),
                ("counters", C.c_uint64 * 8)]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = C.CDLL(build())
            lib.orc_run.argtypes = [C.POINTER(_Problem), C.POINTER(_RunArgs), C.POINTER(_Out)]
            lib.orc_run.restype = C.c_int
            lib.orc_uniform.argtypes = [C.c_uint64] + [C.c_int32] * 5
            lib.orc_uniform.restype = C.c_double
            lib.orc_philox.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            lib.orc_philox.restype = None
            lib.orc_num_spins.argtypes = [C.POINTER(_Problem)]
            lib.orc_num_spins.restype = C.c_int
            lib.orc_scales.argtypes = [C.POINTER(_Problem), C.c_void_p]
            lib.orc_scales.restype = C.c_int
            lib.orc_field.argtypes = [C.POINTER(_Problem), C.c_void_p, C.c_void_p, C.c_int,
                                      C.c_void_p, C.POINTER(C.c_double)]
            lib.orc_field.restype = C.c_int
            lib.orc_decide.argtypes = [C.POINTER(_Problem), C.c_double, C.c_int, C.c_int,
                                       C.c_int64, C.c_int64, C.c_int64]
            lib.orc_decide.restype = C.c_int
            lib.orc_readout.argtypes = [C.POINTER(_Problem), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            lib.orc_readout.restype = C.c_int
            _lib = lib
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


class OracleProblem:
    """One instance, arrays kept alive for the C calls."""

    def __init__(self, Q, c, A, b, P, eta, beta_max, inst=0):
        self.Q = None if Q is None else np.ascontiguousarray(Q, dtype=np.int32)
        self.c = np.ascontiguousarray(c, dtype=np.int32)
        self.A = np.ascontiguousarray(A, dtype=np.int32)
        self.b = np.ascontiguousarray(b, dtype=np.int64)
        self.n = int(self.c.shape[0])
        self.M = int(self.b.shape[0])
        self.P, self.eta, self.beta_max, self.inst = float(P), float(eta), float(beta_max), int(inst)
        self._s = _Problem(self.n, self.M, _ptr(self.Q), _ptr(self.c), _ptr(self.A), _ptr(self.b),
                           self.P, self.eta, self.beta_max, self.inst)

    @classmethod
    def from_inputs(cls, prob, P, eta, beta_max, inst=0):
        return cls(prob.Q, prob.c, prob.A, prob.b, P, eta, beta_max, inst)

    @property
    def N(self) -> int:
        return int(_load().orc_num_spins(C.byref(self._s)))

    def scales(self):
        out = np.zeros(2, dtype=np.int64)
        if _load().orc_scales(C.byref(self._s), out.ctypes.data):
            raise ValueError("invalid problem")
        return int(out[0]), int(out[1])

    def field(self, x, Lam, i):
        x = np.ascontiguousarray(x, dtype=np.uint8)
        Lam = np.ascontiguousarray(Lam, dtype=np.int64)
        out = np.zeros(3, dtype=np.int64)
        F = C.c_double()
        if _load().orc_field(C.byref(self._s), x.ctypes.data, Lam.ctypes.data, int(i), out.ctypes.data, C.byref(F)):
            raise ValueError("invalid problem")
        return int(out[0]), int(out[1]), int(out[2]), F.value

    def readout(self, x):
        """(f(x), feasible, r(x)) for a full state x of length N."""
        x = np.ascontiguousarray(x, dtype=np.uint8)
        f = np.zeros(1, np.int64)
        feas = np.zeros(1, np.int32)
        r = np.zeros(max(self.M, 1), np.int64)
        if _load().orc_readout(C.byref(self._s), x.ctypes.data, f.ctypes.data, feas.ctypes.data, r.ctypes.data):
            raise ValueError("invalid problem")
        return int(f[0]), bool(feas[0]), r[:self.M].copy()

    def decide(self, u, t, T, phi, pi, kappa) -> int:
        return int(_load().orc_decide(C.byref(self._s), float(u), int(t), int(T), int(phi), int(pi), int(kappa)))

    def run(self, seed, nrep, K, T, rep0=0, mode=INCREMENTAL, nthreads=None, trace=False, x_init=None,
            final=False):
        lib = _load()
        n, M, N = self.n, self.M, self.N
        Wn, WN = (n + 31) // 32, (N + 31) // 32
        res = {
            "best_f": np.zeros(nrep, np.int64), "best_x": np.zeros((nrep, Wn), np.uint32),
            "best_k": np.zeros(nrep, np.int32), "n_feasible": np.zeros(nrep, np.int32),
        }
        if trace:
            res.update(tr_f=np.zeros((nrep, K), np.int64), tr_feas=np.zeros((nrep, K), np.uint8),
                       tr_r=np.zeros((nrep, K, M), np.int64), tr_lam=np.zeros((nrep, K, M), np.int64),
                       tr_x=np.zeros((nrep, K, WN), np.uint32))
        if final:
            res.update(final_x=np.zeros((nrep, WN), np.uint32), final_lam=np.zeros((nrep, M), np.int64))
        xi = None
        if x_init is not None:
            xi = np.ascontiguousarray(x_init, dtype=np.uint8).reshape(nrep, N)
        args = _RunArgs(int(seed) & ((1 << 64) - 1), int(rep0), int(nrep), int(K), int(T), int(mode),
                        int(nthreads or os.cpu_count() or 1), _ptr(xi))
        out = _Out(*[_ptr(res.get(k)) for k in ["best_f", "best_x", "best_k", "n_feasible", "tr_f",
                                                 "tr_feas", "tr_r", "tr_lam", "tr_x", "final_x",
                                                 "final_lam"]])
        if lib.orc_run(C.byref(self._s), C.byref(args), C.byref(out)):
            raise ValueError("oracle rejected the problem/run arguments")
        res["counters"] = {name: int(out.counters[i]) for i, name in enumerate(COUNTER_NAMES)}
        return res


def uniform(seed, s, rho, k, t, i) -> float:
    return float(_load().orc_uniform(int(seed) & ((1 << 64) - 1), int(s), int(rho), int(k), int(t), int(i)))


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _load().orc_philox(c.ctypes.data, k.ctypes.data, out.ctypes.data)
    return [int(v) for v in out]


def run_config_instance(cfg, inst_idx, seed, nrep, rep0=0, **kw):
    """Run the oracle on instance `inst_idx` of a saim_inputs.Config."""
    prob = cfg.instances[inst_idx]
    op = OracleProblem.from_inputs(prob, cfg.P[inst_idx], cfg.eta, cfg.beta_max, inst=inst_idx)
    return op.run(seed, nrep, cfg.K, cfg.T, rep0=rep0, **kw)
