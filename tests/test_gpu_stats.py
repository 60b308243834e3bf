"""Statistical validation of the GPU sampler independent of the oracle:
with T = 1 the anneal is a single sweep at fixed beta = beta_max and eta = 0 keeps L fixed, so the
per-iteration samples x_k of a replica form a Gibbs chain whose stationary law is Eq. 11
(PAPER.md:133-136).  The empirical distribution over all 2^N states is compared with the exact
Boltzmann weights computed by brute force (oracle/reference.py, exact rationals)."""
from fractions import Fraction

import numpy as np
import pytest

from oracle.reference import RefProblem, boltzmann

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_04971_b200 as P
    from paper_2501_04971_b200 import build
    build.build()
    return P


def _tv(P, Q, c, A, b, Pen, beta, R=64, K=20000, burn=500):
    import torch
    sol = P.Solver(Q, c, A, b, Pen, 0.0, beta)
    out = sol.run(77, R, K, 1, trace=True)
    torch.cuda.synchronize()
    x = out["tr_x"].cpu().numpy().view(np.uint32)[0, :, burn:, 0].ravel()
    sol.close()
    rp = RefProblem(Q, c, A, b, Pen, 0.0)
    ref = boltzmann(rp, [Fraction(0)] * rp.M, beta)
    emp = np.bincount(x, minlength=1 << rp.N) / x.size
    return 0.5 * np.abs(emp - ref).sum(), rp.N


def test_qkp_kernel_samples_eq11(P):
    """QKP kernel (quadratic objective, one constraint): N = 5 items + 3 slack bits = 8 spins."""
    rng = np.random.default_rng(5)
    n = 5
    W = np.triu(rng.integers(0, 5, size=(n, n)), 1)
    W = W + W.T
    tv, N = _tv(P, -W, -rng.integers(0, 5, size=n), rng.integers(1, 4, size=(1, n)), [5], 0.75, 1.5)
    assert N == 8 and tv < 0.02, tv


def test_mkp_kernel_samples_eq11(P):
    """MKP kernel (linear objective, two constraints): N = 4 items + 2 + 2 slack bits = 8 spins."""
    rng = np.random.default_rng(6)
    n = 4
    tv, N = _tv(P, None, -rng.integers(1, 6, size=n), rng.integers(0, 3, size=(2, n)), [3, 2], 0.6, 2.0)
    assert N == 8 and tv < 0.02, tv


def test_beta_zero_sweep_is_uniform(P):
    """beta = 0 (T = 1, beta_max -> tiny): every decision is u < 1/2 up to O(beta)."""
    import torch
    rng = np.random.default_rng(7)
    sol = P.Solver(None, -rng.integers(1, 6, size=6), rng.integers(0, 3, size=(2, 6)), [4, 3], 1.0, 0.0, 1e-9)
    out = sol.run(3, 64, 4000, 1, trace=True)
    torch.cuda.synchronize()
    x = out["tr_x"].cpu().numpy().view(np.uint32)[0, :, :, 0]
    N = sol.instance(0)["N"]
    bits = (x[..., None] >> np.arange(N)) & 1
    assert np.all(np.abs(bits.mean(axis=(0, 1)) - 0.5) < 0.01)
