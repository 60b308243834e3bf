"""Seeded synthetic inputs for the SAIM hot path (shared by the oracle side and the CUDA side).

This module holds NO arithmetic of the method: it draws integer instances (Q, c, A, b) with the
shapes and value distributions BASELINE.json's configs name, picks the run constants of
PAPER.md Table I, and computes the penalty parameter P = alpha*d*N with the
paper's own rule (Algorithm 1 line 1 "(lambda_0, P) <- (0, alpha d N)") -- P is an
*input* of Algorithm 1, chosen by the harness.  Everything the method computes from these inputs
(slack extension, normalisation, fields, decisions, Lagrange steps) lives separately in `oracle/`
and in `paper_2501_04971_b200/`, which never import each other.

Minimisation convention (Eq. 2, 12, 14): f(x) = 1/2 x^T Q x + c^T x over the n items,
Q symmetric integer with zero diagonal, c integer; constraints A x <= b (A: M x n, entries >= 0,
b >= 1).  For QKP Q = -W and c = -h; for MKP Q = 0 and c = -h.

Recipes:
  QKP: upper triangle incl. the diagonal of a profit matrix p, each entry nonzero w.p. d with
       value U{1..100}; diagonal -> h, off-diagonal -> W (symmetric); weights U{1..50};
       capacity U{50..sum w} (clamped to sum w if sum w < 50).
  MKP: A_kj ~ U{0..1000}; b_k = floor(t * sum_j A_kj); h_j = floor(sum_k A_kj / M) + floor(500 u_j).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "Problem", "qkp", "mkp", "paper_P", "Config", "CONFIGS", "config_instances", "stack",
]


@dataclasses.dataclass
class Problem:
    """One constrained binary problem: min 1/2 x^T Q x + c^T x  s.t.  A x <= b."""
    kind: str                 # "qkp" | "mkp"
    n: int                    # items
    M: int                    # constraints
    Q: Optional[np.ndarray]   # int32 [n, n] symmetric, zero diagonal; None for a linear objective
    c: np.ndarray             # int32 [n]
    A: np.ndarray             # int32 [M, n], >= 0
    b: np.ndarray             # int64 [M], >= 1
    d: float                  # density used in P = alpha*d*N
    name: str = ""


def qkp(n: int, d: float, seed: Sequence[int], name: str = "") -> Problem:
    """QKP instance shaped like Billionnet-Soutif, BASELINE.json configs 0-2."""
    rng = np.random.default_rng(list(seed))
    mask = rng.random((n, n)) < d
    vals = rng.integers(1, 101, size=(n, n))
    p = np.triu(np.where(mask, vals, 0))            # upper triangle incl. diagonal
    h = np.diag(p).astype(np.int64)
    W = p - np.diag(np.diag(p))
    W = W + W.T
    w = rng.integers(1, 51, size=n)
    hi = int(w.sum())
    cap = int(rng.integers(50, max(hi, 50) + 1))
    cap = min(cap, hi) if hi >= 1 else 1
    return Problem(
        kind="qkp", n=n, M=1,
        Q=(-W).astype(np.int32), c=(-h).astype(np.int32),
        A=w.reshape(1, n).astype(np.int32), b=np.array([cap], dtype=np.int64),
        d=float(d), name=name or f"qkp_n{n}_d{d}")


def mkp(n: int, m: int, t: float, seed: Sequence[int], name: str = "") -> Problem:
    """MKP instance shaped like Chu-Beasley OR-Library, BASELINE.json configs 3-4."""
    rng = np.random.default_rng(list(seed))
    A = rng.integers(0, 1001, size=(m, n)).astype(np.int64)
    b = np.floor(t * A.sum(axis=1)).astype(np.int64)
    b = np.maximum(b, 1)
    u = rng.random(n)
    h = A.sum(axis=0) // m + np.floor(500.0 * u).astype(np.int64)
    return Problem(
        kind="mkp", n=n, M=m, Q=None, c=(-h).astype(np.int32),
        A=A.astype(np.int32), b=b, d=float("nan"), name=name or f"mkp_n{n}_m{m}_t{t}")


def n_spins(prob: Problem) -> int:
    """Number of Ising spins incl. slack bits, as PAPER.md:102 requires for P = alpha d N.

    The slack count per row is the bit length of b_k ("Q = floor(log2(b)+1)");
    this is the only piece of the slack rule the harness needs to choose P.
    """
    return prob.n + sum(int(bk).bit_length() for bk in prob.b)


def paper_P(prob: Problem, alpha: float) -> float:
    """Penalty parameter P = alpha * d * N (MKP d = 2/(N+1))."""
    N = n_spins(prob)
    d = 2.0 / (N + 1) if prob.kind == "mkp" else prob.d
    return float(alpha) * d * N


@dataclasses.dataclass
class Config:
    """A BASELINE.json config: instances + Algorithm 1 constants (Table I)."""
    idx: int
    name: str
    instances: List[Problem]
    R: int            # replicas per instance
    K: int            # Lagrange iterations (SA runs)
    T: int            # sweeps (MCS) per SA run
    alpha: float
    eta: float
    beta_max: float

    @property
    def P(self) -> List[float]:
        return [paper_P(p, self.alpha) for p in self.instances]


def config_instances(idx: int, variant: Optional[int] = None) -> Config:
    """BASELINE.json configs 0..4 (seeded: numpy default_rng([cfg, variant, instance]))."""
    qkp_c = dict(alpha=2.0, eta=20.0, beta_max=10.0)     # PAPER.md Table I, QKP row
    mkp_c = dict(alpha=5.0, eta=0.05, beta_max=50.0)     # PAPER.md Table I, MKP row
    if idx == 0:
        return Config(0, "qkp_n20", [qkp(20, 0.5, [0, 0, 0])], R=64, K=20, T=100, **qkp_c)
    if idx == 1:
        ds = [0.25, 1.0] if variant is None else [[0.25, 1.0][variant]]
        inst = [qkp(100, d, [1, v, 0]) for v, d in enumerate([0.25, 1.0]) if d in ds]
        return Config(1, "qkp_n100", inst, R=1024, K=100, T=1000, **qkp_c)
    if idx == 2:
        return Config(2, "qkp_n300_d1", [qkp(300, 1.0, [2, 0, 0])], R=4096, K=200, T=1000, **qkp_c)
    if idx == 3:
        ts = [0.25, 0.5, 0.75] if variant is None else [[0.25, 0.5, 0.75][variant]]
        inst = [mkp(100, 5, t, [3, v, 0]) for v, t in enumerate([0.25, 0.5, 0.75]) if t in ts]
        return Config(3, "mkp_n100_m5", inst, R=2048, K=200, T=1000, **mkp_c)
    if idx == 4:
        inst = [mkp(500, 30, 0.5, [4, 0, s]) for s in range(64)]
        return Config(4, "mkp_n500_m30_x64", inst, R=256, K=100, T=2000, **mkp_c)
    raise ValueError(f"unknown config {idx}")


def stack(probs: Sequence[Problem]):
    """Stack same-shape instances into batched arrays (Q may be None for all)."""
    n, M = probs[0].n, probs[0].M
    for p in probs:
        if p.n != n or p.M != M:
            raise ValueError("all instances in a batch must share (n, M)")
    Q = None if probs[0].Q is None else np.ascontiguousarray(np.stack([p.Q for p in probs]).astype(np.int32))
    c = np.ascontiguousarray(np.stack([p.c for p in probs]).astype(np.int32))
    A = np.ascontiguousarray(np.stack([p.A for p in probs]).astype(np.int32))
    b = np.ascontiguousarray(np.stack([p.b for p in probs]).astype(np.int64))
    return Q, c, A, b
