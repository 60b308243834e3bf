"""Python binding of libsaim -- the B200 (sm_100a) SAIM hot path (arXiv 2501.04971).

Argument marshalling only: every step of the path (slack extension, scales, range proofs and
layout in `saim_create`; all sweeps, decisions, readouts and Lagrange steps in the CUDA kernels
launched by `saim_run`) happens inside `libsaim.so` behind the C ABI of `include/saim.h`.
PyTorch provides device memory and the stream.  There is no CPU fallback: importing this module
without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsaim.so")

SAIM_OK, SAIM_EINVAL, SAIM_ERANGE, SAIM_ESMEM, SAIM_ECUDA, SAIM_EUNSUPPORTED, SAIM_ENOMEM = 0, -1, -2, -3, -4, -5, -6
COUNTER_NAMES = ["decisions", "flips", "sweeps", "uniforms", "fp64", "uncertified", "feasible", "philox", "replayed"]
FLAG_NO_FREEZE_EXIT = 1
FLAG_MKP_LOCKSTEP = 2      # MKP: lane-per-replica kernel instead of the outcome tree
FLAG_MKP_L2 = 4            # MKP: outcome tree with 2 lanes per replica
FLAG_MKP_L4 = 8            # MKP: outcome tree with 4 lanes per replica
FLAG_MKP_SPLIT2 = 16       # MKP: constraint rows of a replica split over 2 lanes (M > 8)
FLAG_MKP_NO_PRODUCER = 64  # MKP lockstep: consumer warps draw their own logits (identical results)
FLAG_QKP_NO_HOT_LOOP = 32  # QKP: disable the hot-block loop (identical results)
FLAG_MKP_SPEC4 = 256       # MKP (M <= 8): speculative sub-warp kernel, 4 lanes per replica
FLAG_MKP_SPEC8 = 512       # ... 8 lanes per replica
FLAG_MKP_SPEC2 = 1024      # ... 2 lanes per replica
FLAG_MKP_SPEC16 = 2048     # ... 16 lanes per replica
FLAG_MKP_SPEC32 = 4096     # ... 32 lanes per replica (one replica per warp)
FLAG_TEST_REPLAY = 128     # test hook: every fp64-level decision re-decided in double-double (identical results)
EXPORTS = ["saim_create", "saim_run", "saim_get_info", "saim_get_instance", "saim_destroy",
           "saim_last_error", "saim_selftest"]


class SaimError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libsaim error {code}: {msg}")
        self.code = code


class _Problem(C.Structure):
    _fields_ = [("n_inst", C.c_int32), ("n_items", C.c_int32), ("n_cons", C.c_int32),
                ("Q", C.c_void_p), ("c", C.c_void_p), ("A", C.c_void_p), ("b", C.c_void_p)]


class _Params(C.Structure):
    _fields_ = [("P", C.c_void_p), ("eta", C.c_double), ("beta_max", C.c_double),
                ("device", C.c_int32), ("flags", C.c_int32)]


_OUT_FIELDS = ["best_f", "best_x", "best_k", "n_feasible", "inst_best", "counters",
               "tr_f", "tr_feas", "tr_r", "tr_lam", "tr_x", "final_x", "final_lam", "rep_flips"]


class _Outputs(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in _OUT_FIELDS]


class _Info(C.Structure):
    _fields_ = [(f, C.c_int32) for f in ["n_inst", "n_items", "n_cons", "n_spins_max", "words_items",
                                         "words_full", "kernel", "smem_bytes", "q_bytes",
                                         "lanes_per_replica", "phi_packed"]]


_lib = None


def load_library():
    """Load libsaim.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2501_04971_b200.build` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        lib.saim_create.argtypes = [C.POINTER(_Problem), C.POINTER(_Params), C.POINTER(C.c_void_p)]
        lib.saim_create.restype = C.c_int
        lib.saim_run.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                 C.c_void_p, C.POINTER(_Outputs)]
        lib.saim_run.restype = C.c_int
        lib.saim_get_info.argtypes = [C.c_void_p, C.POINTER(_Info)]
        lib.saim_get_info.restype = C.c_int
        lib.saim_get_instance.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.saim_get_instance.restype = C.c_int
        lib.saim_destroy.argtypes = [C.c_void_p]
        lib.saim_destroy.restype = None
        lib.saim_last_error.argtypes = []
        lib.saim_last_error.restype = C.c_char_p
        lib.saim_selftest.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.saim_selftest.restype = C.c_int
        _lib = lib
    return _lib


def _check(code):
    if code != SAIM_OK:
        raise SaimError(code, load_library().saim_last_error().decode())


def _arr(x, dtype, shape):
    a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
    return a.reshape(shape)


class Solver:
    """A compiled SAIM problem batch resident on one GPU (saim_create / saim_destroy)."""

    def __init__(self, Q, c, A, b, P, eta: float, beta_max: float, device: int = 0, flags: int = 0):
        lib = load_library()
        c = np.asarray(c)
        if c.ndim == 1:
            c = c[None]
        S, n = c.shape
        A = np.asarray(A)
        M = A.shape[-2] if A.ndim >= 2 else 0
        self._c = _arr(c, np.int32, (S, n))
        self._A = _arr(A, np.int32, (S, M, n)) if M else None
        self._b = _arr(b, np.int64, (S, M)) if M else None
        self._Q = None if Q is None else _arr(Q, np.int32, (S, n, n))
        self._P = _arr(np.broadcast_to(np.asarray(P, dtype=np.float64), (S,)), np.float64, (S,))
        prob = _Problem(S, n, M, None if self._Q is None else self._Q.ctypes.data, self._c.ctypes.data,
                        None if self._A is None else self._A.ctypes.data,
                        None if self._b is None else self._b.ctypes.data)
        par = _Params(self._P.ctypes.data, float(eta), float(beta_max), int(device), int(flags))
        h = C.c_void_p()
        _check(lib.saim_create(C.byref(prob), C.byref(par), C.byref(h)))
        self._h = h
        self.device = int(device)
        info = _Info()
        _check(lib.saim_get_info(self._h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in _Info._fields_}
        self.n_inst, self.n, self.M = S, n, M

    @classmethod
    def from_config(cls, cfg, device: int = 0, flags: int = 0):
        """Build from a saim_inputs.Config (all its instances in one batch)."""
        import saim_inputs as si
        Q, c, A, b = si.stack(cfg.instances)
        return cls(Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, device=device, flags=flags)

    def instance(self, s: int):
        N = C.c_int32()
        so = C.c_int64()
        sc = C.c_int64()
        q = np.zeros(max(self.M, 1), np.int32)
        _check(load_library().saim_get_instance(self._h, int(s), C.byref(N), C.byref(so), C.byref(sc),
                                                q.ctypes.data))
        return {"N": N.value, "s_o": so.value, "s_c": sc.value, "q": q[:self.M].tolist()}

    def alloc_outputs(self, R: int, K: int, trace: bool = False, final: bool = False):
        import torch
        dev = torch.device("cuda", self.device)
        specs = self.output_specs(R, K)
        fields = ["best_f", "best_x", "best_k", "n_feasible", "inst_best", "counters"]
        if trace:
            fields += ["tr_f", "tr_feas", "tr_r", "tr_lam", "tr_x"]
        if final:
            fields += ["final_x", "final_lam", "rep_flips"]
        return {f: torch.empty(specs[f][0], dtype=specs[f][1], device=dev) for f in fields}

    def output_specs(self, R: int, K: int):
        """Shape and dtype of every saim_outputs field for a run of R replicas x K iterations."""
        import torch
        S, Wn, WN, M = self.n_inst, self.info["words_items"], self.info["words_full"], self.M
        return {"best_f": ((S, R), torch.int64), "best_x": ((S, R, Wn), torch.int32),
                "best_k": ((S, R), torch.int32), "n_feasible": ((S, R), torch.int32),
                "inst_best": ((S,), torch.int64), "counters": ((len(COUNTER_NAMES),), torch.int64),
                "tr_f": ((S, R, K), torch.int64), "tr_feas": ((S, R, K), torch.uint8),
                "tr_r": ((S, R, K, M), torch.int64), "tr_lam": ((S, R, K, M), torch.int64),
                "tr_x": ((S, R, K, WN), torch.int32), "final_x": ((S, R, WN), torch.int32),
                "final_lam": ((S, R, M), torch.int64), "rep_flips": ((S, R), torch.int32)}

    def check_outputs(self, out: Dict, R: int, K: int):
        """Raise ValueError unless every tensor in `out` matches the run's shape, dtype, device and is
        contiguous (the kernel writes through raw pointers: a stale buffer would be overrun)."""
        import torch
        specs = self.output_specs(R, K)
        for f in ("best_f", "best_x", "best_k", "n_feasible"):
            if out.get(f) is None:
                raise ValueError(f"outputs: '{f}' is required")
        for f, t in out.items():
            if f not in specs:
                raise ValueError(f"outputs: unknown field '{f}'")
            if t is None:
                continue
            shape, dtype = specs[f]
            if not isinstance(t, torch.Tensor) or tuple(t.shape) != shape or t.dtype != dtype:
                raise ValueError(f"outputs['{f}']: expected {dtype} of shape {shape}, got "
                                 f"{getattr(t, 'dtype', type(t))} {tuple(getattr(t, 'shape', ()))}")
            if t.device != torch.device("cuda", self.device) or not t.is_contiguous():
                raise ValueError(f"outputs['{f}']: must be a contiguous tensor on cuda:{self.device}")

    def run(self, seed: int, R: int, K: int, T: int, rep0: int = 0, trace: bool = False, final: bool = False,
            out: Optional[Dict] = None, stream=None):
        """Launch saim_run asynchronously on `stream` (default: torch's current stream)."""
        import torch
        if out is None:
            out = self.alloc_outputs(R, K, trace=trace, final=final)
        else:
            self.check_outputs(out, R, K)
        ptrs = _Outputs(*[out[f].data_ptr() if f in out and out[f] is not None else None for f in _OUT_FIELDS])
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        _check(load_library().saim_run(self._h, int(seed) & ((1 << 64) - 1), int(rep0), int(R), int(K), int(T),
                                       C.c_void_p(stream.cuda_stream), C.byref(ptrs)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            load_library().saim_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def counters_dict(t) -> Dict[str, int]:
    v = t.cpu().numpy().view(np.uint64)
    return {name: int(v[i]) for i, name in enumerate(COUNTER_NAMES)}


def selftest_philox(inputs, device: int = 0):
    inp = np.ascontiguousarray(np.asarray(inputs, dtype=np.uint32).reshape(-1, 6))
    out = np.zeros((inp.shape[0], 4), np.uint32)
    _check(load_library().saim_selftest(0, int(device), inp.shape[0], inp.ctypes.data, out.ctypes.data, None))
    return out


DD_RECORD = np.dtype([("phi", "<i8"), ("pi", "<i8"), ("kappa", "<i8"), ("s_o", "<i8"), ("s_c", "<i8"),
                      ("P", "<f8"), ("eta", "<f8"), ("beta_max", "<f8"), ("tn", "<i4"), ("td", "<i4"),
                      ("w", "<u4"), ("pad", "<i4")])


def selftest_decide_dd(records, device: int = 0):
    """Double-double decision level (saim_selftest(2)) on a DD_RECORD array: x | uncertified << 1."""
    rec = np.ascontiguousarray(records, dtype=DD_RECORD)
    assert rec.dtype.itemsize == 80
    out = np.zeros(rec.shape[0], np.uint32)
    _check(load_library().saim_selftest(2, int(device), rec.shape[0], rec.ctypes.data, out.ctypes.data, None))
    return out


def selftest_logit_table(words, device: int = 0):
    """saim_selftest(3): (table entry, direct device computation) of logit(u) for each Philox word."""
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32).ravel())
    out = np.zeros((w.shape[0], 2), np.float64)
    _check(load_library().saim_selftest(3, int(device), w.shape[0], w.ctypes.data, None, out.ctypes.data))
    return out[:, 0], out[:, 1]


def selftest_logit(device: int = 0):
    out = np.zeros(2, np.float64)
    _check(load_library().saim_selftest(1, int(device), 0, None, None, out.ctypes.data))
    return {"max_ratio": float(out[0]), "max_abs_err": float(out[1])}
