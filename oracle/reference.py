"""Pure-Python definitions used to PIN the C oracle (test infrastructure only).

Every function here is the paper's formula written out with exact rationals (fractions.Fraction),
or a brute-force enumeration, so that the oracle's incremental integer decomposition
(phi, pi, kappa) can be checked against something other than itself:

  * `lagrangian(x)`  -- Eq. 3 + Eq. 5 with the normalisation of PAPER.md:170
                       and the slack extension of PAPER.md:162, evaluated literally.
  * `field_fd(x, i)` -- F_i = -(L(x^{i<-1}) - L(x^{i<-0})), the finite difference that Eq. 9-10 turn
                       into a p-bit input (binary form of I_i, R1).
  * `ising(...)`     -- the spin form of L (Eq. 1 "Ising_hamiltonian") with J and h
                       read off the expanded QUBO (dense P*A^T*A couplings, which the hot path never
                       forms), and `p_bit_input` = Eq. 9 I_i = sum_j J_ij m_j + h_i.
  * `brute_force_opt` -- OPT of Eq. 2 over all 2^n item states (stands in for B&B).
  * `boltzmann`      -- Eq. 11 over all 2^N states.
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction
from typing import List, Optional, Sequence

import numpy as np


def slack_bits(b: int) -> int:
    """Q = floor(log2(b) + 1), evaluated without floating point: the smallest q
    with 2^q > b."""
    q = 0
    while (1 << q) <= b:
        q += 1
    return q


class RefProblem:
    """Slack-extended, normalised problem in exact arithmetic."""

    def __init__(self, Q, c, A, b, P, eta):
        self.n = len(c)
        self.M = len(b)
        self.Q = None if Q is None else [[int(v) for v in row] for row in np.asarray(Q)]
        self.c = [int(v) for v in c]
        self.A = [[int(v) for v in row] for row in np.asarray(A).reshape(self.M, self.n)] if self.M else []
        self.b = [int(v) for v in b]
        self.P = Fraction(P)          # exact value of the fp64 input
        self.eta = Fraction(eta)
        self.q = [slack_bits(bk) for bk in self.b]
        self.N = self.n + sum(self.q)
        # A_ext: items, then row 0's slack bits LSB..MSB, then row 1's, ...
        self.Aext = []
        col = self.n
        for k in range(self.M):
            row = list(self.A[k]) + [0] * (self.N - self.n)
            for bit in range(self.q[k]):
                row[col] = 1 << bit
                col += 1
            self.Aext.append(row)
        mags = [abs(v) for v in self.c] + ([abs(v) for r in self.Q for v in r] if self.Q else [])
        self.s_o = max(mags) if mags and max(mags) > 0 else 1
        cm = [v for r in self.A for v in r] + self.b
        self.s_c = max(cm) if cm and max(cm) > 0 else 1

    # -- Eq. 2/12/14 objective and constraints --------------------------------------------
    def f(self, x: Sequence[int]) -> int:
        """f(x) = 1/2 x^T Q x + c^T x on the items (x may be the full N-vector)."""
        v = sum(self.c[i] * x[i] for i in range(self.n))
        if self.Q:
            v2 = sum(self.Q[i][j] * x[i] * x[j] for i in range(self.n) for j in range(self.n))
            assert v2 % 2 == 0
            v += v2 // 2
        return v

    def r(self, x: Sequence[int]) -> List[int]:
        """Equality-form residual g (unnormalised): A_ext x - b."""
        return [sum(self.Aext[k][j] * x[j] for j in range(self.N)) - self.b[k] for k in range(self.M)]

    def feasible(self, x: Sequence[int]) -> bool:
        """A^T x <= b on the items."""
        return all(sum(self.A[k][j] * x[j] for j in range(self.n)) <= self.b[k] for k in range(self.M))

    # -- Eq. 3 + Eq. 5 -------------------------------------------------------------------
    def lagrangian(self, x: Sequence[int], lam: Sequence[Fraction]) -> Fraction:
        """L = f/s_o + P ||g||^2 + lambda^T g with g = r/s_c (normalised)."""
        g = [Fraction(rk, self.s_c) for rk in self.r(x)]
        return (Fraction(self.f(x), self.s_o) + self.P * sum(gk * gk for gk in g)
                + sum(Fraction(lk) * gk for lk, gk in zip(lam, g)))

    def lam_from_Lambda(self, Lam: Sequence[int]) -> List[Fraction]:
        """lambda_k for the integer accumulator Lambda: iterate Algorithm 1's update literally
        would need the sample history; for a given Lambda, lambda = eta * Lambda / s_c (R10)."""
        return [self.eta * Fraction(int(L), self.s_c) for L in Lam]

    def field_fd(self, x: Sequence[int], lam: Sequence[Fraction], i: int) -> Fraction:
        """F_i = -(L(x^{i<-1}) - L(x^{i<-0}))."""
        x1 = list(x); x1[i] = 1
        x0 = list(x); x0[i] = 0
        return -(self.lagrangian(x1, lam) - self.lagrangian(x0, lam))

    # -- spin form (Eq. 1, Eq. 9) ----------------------------------------------------------
    def qubo(self, lam: Sequence[Fraction]):
        """Expand L(x) = const + sum_i l_i x_i + sum_{i<j} q_ij x_i x_j (dense; x_i^2 = x_i)."""
        N, n = self.N, self.n
        l = [Fraction(0)] * N
        q = [[Fraction(0)] * N for _ in range(N)]
        const = Fraction(0)
        for i in range(n):
            l[i] += Fraction(self.c[i], self.s_o)
            if self.Q:
                for j in range(i + 1, n):
                    q[i][j] += Fraction(self.Q[i][j], self.s_o)
        sc2 = Fraction(self.s_c * self.s_c)
        for k in range(self.M):
            a, bk = self.Aext[k], self.b[k]
            # P (a.x - b)^2 / s_c^2
            const += self.P * bk * bk / sc2
            for i in range(N):
                l[i] += self.P * (a[i] * a[i] - 2 * bk * a[i]) / sc2
                for j in range(i + 1, N):
                    q[i][j] += self.P * 2 * a[i] * a[j] / sc2
            # lambda_k (a.x - b) / s_c
            lk = Fraction(lam[k]) if k < len(lam) else Fraction(0)
            const -= lk * bk / self.s_c
            for i in range(N):
                l[i] += lk * a[i] / self.s_c
        return const, l, q

    def ising(self, lam: Sequence[Fraction]):
        """J, h of H = -sum_{i<j} J_ij S_i S_j - sum_i h_i S_i with H = L + const, x = (1+S)/2."""
        const, l, q = self.qubo(lam)
        N = self.N
        J = [[Fraction(0)] * N for _ in range(N)]
        h = [Fraction(0)] * N
        for i in range(N):
            h[i] -= l[i] / 2
            for j in range(i + 1, N):
                if q[i][j]:
                    J[i][j] -= q[i][j] / 4
                    J[j][i] -= q[i][j] / 4
                    h[i] -= q[i][j] / 4
                    h[j] -= q[i][j] / 4
        return J, h

    @staticmethod
    def p_bit_input(J, h, m: Sequence[int], i: int) -> Fraction:
        """Eq. 9: I_i = sum_j J_ij m_j + h_i."""
        return sum(J[i][j] * m[j] for j in range(len(m)) if j != i) + h[i]


def brute_force_opt(Q, c, A, b):
    """OPT = min f(x) over item states x in {0,1}^n with A x <= b (vectorised enumeration)."""
    n = len(c)
    if n > 24:
        raise ValueError("brute force limited to n <= 24")
    X = ((np.arange(1 << n)[:, None] >> np.arange(n)[None, :]) & 1).astype(np.int64)
    f = X @ np.asarray(c, np.int64)
    if Q is not None:
        Qa = np.asarray(Q, np.int64)
        f = f + ((X @ Qa) * X).sum(axis=1) // 2
    load = X @ np.asarray(A, np.int64).T
    feas = (load <= np.asarray(b, np.int64)[None, :]).all(axis=1)
    fmin = f[feas].min()
    idx = np.nonzero(feas & (f == fmin))[0]
    return int(fmin), X[idx]


def boltzmann(rp: RefProblem, lam: Sequence[Fraction], beta: float) -> np.ndarray:
    """Eq. 11 over all 2^N full states, index = sum_i x_i 2^i."""
    N = rp.N
    E = np.array([float(rp.lagrangian([(s >> i) & 1 for i in range(N)], lam)) for s in range(1 << N)])
    w = np.exp(-beta * (E - E.min()))
    return w / w.sum()


def sigma_exact(z: Fraction, digits: int = 60):
    """sigma(z) = 1/(1+exp(-z)) to `digits` significant digits (decimal module)."""
    import decimal
    ctx = decimal.Context(prec=digits)
    zd = ctx.divide(decimal.Decimal(z.numerator), decimal.Decimal(z.denominator))
    return ctx.divide(1, ctx.add(1, ctx.exp(-zd)))
