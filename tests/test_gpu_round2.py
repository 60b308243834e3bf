"""GPU tests added in round 2 (marked gpu; run on a B200), all through the C ABI:

* the double-double decision level (R18, third certification level) against the exact
  predicate (60-digit decimal sigma) and the oracle's binary128 path on constructed near ties;
* full-size parity where round 1 sampled less: config 4 at its BASELINE K = 100 (all 64 instances
  launched, sampled (instance, replica) pairs replayed by the oracle), config 3 with a 32-replica
  block per instance, config 2 at a second seed;
* the paper's long budgets on small instances: MKP at K = 5000 (Table I, int64 Lambda
  growth) and the penalty method's long single anneals T = 200000;
* API hygiene: the per-launch shared-memory attribute (a later, smaller saim_create of the same
  kernel template must not break an earlier context) and output-buffer validation.
"""
import dataclasses
import math
from concurrent.futures import ThreadPoolExecutor
from fractions import Fraction

import numpy as np
import pytest

import oracle
import saim_inputs as si
from oracle.reference import sigma_exact

from test_gpu_parity import P, compare, gpu_run, run_both, _mkp, _qkp  # noqa: F401  (fixture P)

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------------------------------------
# Double-double decision level

def _exact(u, z: Fraction) -> int:
    return int(Fraction(u) < Fraction(str(sigma_exact(z))))


def _rec(P_, phi, pi, kappa, s_o, s_c, eta, beta_max, tn, td, m):
    """One selftest record; u = (2m + 1) 2^-24 via the Philox word w = m << 9 (R2)."""
    return (phi, pi, kappa, s_o, s_c, P_, eta, beta_max, tn, td, m << 9, 0)


def test_dd_level_unit_near_ties(P):
    """z = -P (s_o = s_c = 1, pi = 1, beta = 1) within +-1000 ulps of logit(u): the double-double
    decision equals the exact predicate and is certified, including the +-1 ulp cases that the
    fp64 level cannot settle."""
    rng = np.random.default_rng(7)
    recs, want = [], []
    for _ in range(200):
        m = int(rng.integers(0, 2 ** 23))
        u = (2 * m + 1) / 2.0 ** 24
        P0 = -math.log(u / (1 - u))
        for ulps in (-1000, -3, -1, 0, 1, 3, 1000):
            Pv = P0
            for _k in range(abs(ulps)):
                Pv = float(np.nextafter(Pv, math.inf if ulps > 0 else -math.inf))
            recs.append(_rec(Pv, 0, 1, 0, 1, 1, 0.0, 1.0, 1, 1, m))
            want.append(_exact(u, -Fraction(Pv)))
    got = P.selftest_decide_dd(np.array(recs, dtype=P.DD_RECORD))
    assert np.all(got >> 1 == 0), "a near tie was left uncertified"
    assert np.array_equal(got & 1, np.array(want, np.uint32))


def test_dd_level_general_components(P):
    """General exact components (phi, pi, kappa, s_o, s_c, eta, beta_max t/(T-1)) with P tuned so
    that z lands within a few ulps of logit(u): every term of z and the beta ramp enter the
    double-double evaluation; answers equal the exact predicate (Fractions + 60-digit sigma) and the
    oracle's binary128 decision."""
    rng = np.random.default_rng(11)
    recs, want, orc = [], [], []
    for _ in range(150):
        m = int(rng.integers(2 ** 20, 2 ** 23 - 2 ** 20))
        u = (2 * m + 1) / 2.0 ** 24
        s_o, s_c = int(rng.integers(1, 200)), int(rng.integers(1, 3000))
        phi, pi, kappa = int(rng.integers(-30000, 30000)), int(rng.integers(1, 10 ** 8)), int(rng.integers(-10 ** 9, 10 ** 9))
        eta, beta_max = float(rng.uniform(0.01, 30)), float(rng.uniform(1, 60))
        T = int(rng.integers(2, 5000))
        t = int(rng.integers(1, T))
        beta = Fraction(beta_max) * t / (T - 1)
        zstar = math.log(u / (1 - u))
        # z = beta (phi/s_o - P pi/s_c^2 - eta kappa/s_c^2) = zstar  =>  P
        P0 = float((Fraction(phi, s_o) - Fraction(eta) * kappa / s_c ** 2 - Fraction(zstar) / beta) * s_c ** 2 / pi)
        if not (P0 > 0 and math.isfinite(P0)):
            continue
        for ulps in (-2, 0, 2):
            Pv = P0
            for _k in range(abs(ulps)):
                Pv = float(np.nextafter(Pv, math.inf if ulps > 0 else -math.inf))
            z = beta * (Fraction(phi, s_o) - Fraction(Pv) * pi / s_c ** 2 - Fraction(eta) * kappa / s_c ** 2)
            recs.append(_rec(Pv, phi, pi, kappa, s_o, s_c, eta, beta_max, t, T - 1, m))
            want.append(_exact(u, z))
            # the oracle's decision on the same components (its problem fixes s_o, s_c through c, A, b)
            op = oracle.OracleProblem(None, [-s_o], [[s_c]], [s_c], Pv, eta, beta_max)
            assert op.scales() == (s_o, s_c)
            orc.append(op.decide(u, t, T, phi, pi, kappa))
    assert len(recs) > 200
    got = P.selftest_decide_dd(np.array(recs, dtype=P.DD_RECORD))
    assert np.all(got >> 1 == 0)
    assert np.array_equal(got & 1, np.array(want, np.uint32))
    assert np.array_equal(got & 1, np.array(orc, np.uint32))


# ---------------------------------------------------------------------------------------------
# Full-size parity

def _oracle_replay(cfg, g, pairs, seed, K, T):
    """Replay (instance, first replica, count) blocks with the oracle, in parallel threads (ctypes
    releases the GIL), and compare with the GPU result g element by element."""
    def one(job):
        s, r0, nb = job
        op = oracle.OracleProblem.from_inputs(cfg.instances[s], cfg.P[s], cfg.eta, cfg.beta_max, inst=s)
        return s, r0, nb, op.N, op.run(seed, nb, K, T, rep0=r0, trace=True, final=True, nthreads=nb)
    with ThreadPoolExecutor(max_workers=len(pairs)) as ex:
        results = list(ex.map(one, pairs))
    near = 0
    for s, r0, nb, N, o in results:
        compare(g, o, s, list(range(r0, r0 + nb)), N, K, cfg.instances[s].M)
        assert int(g["rep_flips"][s, r0:r0 + nb].sum()) == o["counters"]["flips"], "trajectories differ"
        near += o["counters"]["near_ties"]
    return near


def test_mkp_parity_config4_full_K(P):
    """BASELINE config 4 exactly as the bench launches it (64 instances x 256 replicas, n = 500,
    M = 30, K = 100, T = 2000); 4 replicas on each of 4 instances spread over the batch replayed by
    the oracle (K = 100 exercises the Lambda-dependent fp32 error term at the configured budget)."""
    cfg = si.config_instances(4)
    Q, c, A, b = si.stack(cfg.instances)
    g = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 1, cfg.R, cfg.K, cfg.T)
    assert g["counters"]["uncertified"] == 0
    near = _oracle_replay(cfg, g, [(0, 0, 4), (21, 85, 4), (42, 170, 4), (63, 252, 4)], 1, cfg.K, cfg.T)
    print(f"config 4: oracle near ties (|u - sigma| < 2^-20) in the replayed replicas: {near}; mismatches: 0")


def test_mkp_parity_config3_blocks(P):
    """Config 3 at full size: a contiguous block of 32 replicas of each of the three instances."""
    cfg = si.config_instances(3)
    Q, c, A, b = si.stack(cfg.instances)
    g = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 1, cfg.R, cfg.K, cfg.T)
    assert g["counters"]["uncertified"] == 0
    _oracle_replay(cfg, g, [(0, 1000, 32), (1, 16, 32), (2, 2000, 32)], 1, cfg.K, cfg.T)


def test_parity_config2_second_seed(P):
    cfg = si.config_instances(2)
    run_both(P, cfg.instances, cfg.P, cfg.eta, cfg.beta_max, seed=2, R=cfg.R, K=cfg.K, T=cfg.T,
             reps=[7, 4000], block=(2048, 48))


# ---------------------------------------------------------------------------------------------
# The paper's long budgets on small instances

def test_mkp_parity_K5000(P):
    """PAPER.md Table I's MKP budget K = 5000 on a small MKP instance: Lambda
    accumulates over 5000 Lagrange steps (int64), every kernel variant against the oracle."""
    p = _mkp(40, 5, 0.5, 31)
    for v in (0, 2, 4):
        g = run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=21, R=32, K=5000, T=20, flags=v)
        assert int(np.abs(g["final_lam"]).max()) > 0


def test_qkp_parity_K2000(P):
    """PAPER.md Table I's QKP budget K = 2000 on a small QKP instance (sampled replicas)."""
    p = _qkp(40, 0.5, 32)
    run_both(P, [p], [si.paper_P(p, 2.0)], 20.0, 10.0, seed=22, R=64, K=2000, T=50, reps=[0, 63], block=(16, 16))


def test_penalty_long_anneal_T200000(P):
    """The penalty method's long single anneals ("10 SA runs of 2x10^5 MCS"): eta = 0,
    K = 2 anneals of T = 200000 sweeps on an n = 100, d = 0.25 instance; the sweep index t runs to
    199999 in the beta ramp.  Sampled replicas against the oracle."""
    p = si.qkp(100, 0.25, [1, 0, 0])
    run_both(P, [p], [si.paper_P(p, 2.0)], 0.0, 10.0, seed=23, R=64, K=2, T=200000, reps=[0, 63], block=(20, 8))


# ---------------------------------------------------------------------------------------------
# API hygiene

def test_smem_attribute_is_per_launch(P):
    """A smaller instance of the same kernel template created after a larger one must not lower the
    larger context's dynamic shared-memory limit (the attribute is process-wide per function)."""
    import torch
    big, small = _qkp(300, 0.5, 40), _qkp(290, 0.5, 41)
    sb = P.Solver(big.Q, big.c, big.A, big.b, si.paper_P(big, 2.0), 20.0, 10.0)
    ss = P.Solver(small.Q, small.c, small.A, small.b, si.paper_P(small, 2.0), 20.0, 10.0)
    assert sb.info["smem_bytes"] > ss.info["smem_bytes"]
    R = 4096                                             # the big context's maximal warps per CTA
    ob = sb.run(3, R, 2, 10)
    os_ = ss.run(3, R, 2, 10)
    ob2 = sb.run(3, R, 2, 10)
    torch.cuda.synchronize()
    assert torch.equal(ob["best_f"], ob2["best_f"]) and torch.equal(ob["counters"], ob2["counters"])
    assert int(os_["counters"][0]) > 0
    sb.close()
    ss.close()


def test_run_rejects_mismatched_outputs(P):
    import torch
    p = _qkp(30, 0.5, 42)
    sol = P.Solver(p.Q, p.c, p.A, p.b, si.paper_P(p, 2.0), 20.0, 10.0)
    out = sol.alloc_outputs(16, 4, trace=True)
    sol.run(1, 16, 4, 10, out=out)                       # matching buffers are accepted
    with pytest.raises(ValueError):
        sol.run(1, 32, 4, 10, out=out)                   # more replicas than the buffers hold
    with pytest.raises(ValueError):
        sol.run(1, 16, 8, 10, out=out)                   # trace sized for another K
    bad = dict(out, best_f=out["best_f"].to(torch.int32))
    with pytest.raises(ValueError):
        sol.run(1, 16, 4, 10, out=bad)
    bad = dict(out, best_x=torch.empty((1, 16, 2), dtype=torch.int32, device="cuda")[:, :, :1])
    with pytest.raises(ValueError):
        sol.run(1, 16, 4, 10, out=bad)                   # non-contiguous
    torch.cuda.synchronize()
    sol.close()


# ---------------------------------------------------------------------------------------------
# Exact replay / double-double level inside the kernels (SAIM_FLAG_TEST_REPLAY)

_ALL_OUT = ["tr_x", "tr_f", "tr_feas", "tr_r", "tr_lam", "best_f", "best_k", "best_x", "n_feasible",
            "final_x", "final_lam", "inst_best", "rep_flips"]


@pytest.mark.parametrize("cfg_idx", [1, 2])
def test_qkp_exact_replay(P, cfg_idx):
    """With SAIM_FLAG_TEST_REPLAY the QKP main kernel defers every replica that reached the fp64
    level to the replay kernel, which re-runs it with every such decision taken by the double-double
    level: outputs and data-determined counters are identical to the normal run, and sampled
    replicas (replayed ones among them) match the oracle."""
    cfg = si.config_instances(cfg_idx)
    Q, c, A, b = si.stack(cfg.instances)
    R, K = 1024, 12
    base = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 8, R, K, cfg.T)
    rep = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 8, R, K, cfg.T, flags=P.FLAG_TEST_REPLAY)
    assert base["counters"]["replayed"] == 0
    assert rep["counters"]["replayed"] > 0, "no replica reached the fp64 level: the test is vacuous"
    for k in _ALL_OUT:
        assert np.array_equal(base[k], rep[k]), k
    for k in ["decisions", "flips", "uniforms", "feasible", "sweeps", "uncertified"]:
        assert base["counters"][k] == rep["counters"][k], k
    assert rep["counters"]["fp64"] >= base["counters"]["fp64"]
    # replayed replicas against the oracle (those whose trajectory had fp64-level decisions)
    s = 0
    op = oracle.OracleProblem.from_inputs(cfg.instances[s], cfg.P[s], cfg.eta, cfg.beta_max, inst=s)
    o = op.run(8, 32, K, cfg.T, trace=True, final=True)
    compare(rep, o, s, list(range(32)), op.N, K, cfg.instances[s].M)


def test_mkp_dd_level_in_kernels(P):
    """MKP kernels take the double-double level in place (no replay): with SAIM_FLAG_TEST_REPLAY
    every fp64-level decision is re-decided in double-double; outputs are identical for every kernel
    variant and equal the oracle."""
    p = _mkp(100, 5, 0.5, 33)
    q = _mkp(60, 12, 0.5, 34)
    for prob in (p, q):
        Q, c, A, b = si.stack([prob])
        for v in (0, 2, 4, 8, 16) + ((256, 512, 1024, 2048, 4096) if prob.M <= 8 else ()):
            base = gpu_run(P, Q, c, A, b, [si.paper_P(prob, 5.0)], 0.05, 50.0, 4, 64, 6, 200, flags=v)
            dd = gpu_run(P, Q, c, A, b, [si.paper_P(prob, 5.0)], 0.05, 50.0, 4, 64, 6, 200, flags=v | P.FLAG_TEST_REPLAY)
            assert dd["counters"]["fp64"] > 0
            for k in _ALL_OUT:
                assert np.array_equal(base[k], dd[k]), (v, k)
        run_both(P, [prob], [si.paper_P(prob, 5.0)], 0.05, 50.0, seed=4, R=64, K=6, T=200, flags=P.FLAG_TEST_REPLAY)


def test_logit_table_matches_direct_computation(P):
    """The fp64 slow path reads logit(u) from a per-device table of all 2^23 uniforms: every entry it
    reads (word w -> entry w >> 9) equals the device's direct ln(u) - ln(1 - u) bit for bit, and the
    host's within a few ulps (R2's u = (2 floor(w / 2^9) + 1) 2^-24)."""
    rng = np.random.default_rng(5)
    words = np.concatenate([np.array([0, 511, 512, 1023, 2 ** 31 - 1, 2 ** 31, 2 ** 32 - 512, 2 ** 32 - 1], np.uint64),
                            rng.integers(0, 2 ** 32, size=20000, dtype=np.uint64)]).astype(np.uint32)
    tab, calc = P.selftest_logit_table(words)
    assert np.array_equal(tab.view(np.uint64), calc.view(np.uint64))
    u = (2.0 * (words >> 9).astype(np.float64) + 1.0) * 2.0 ** -24
    host = np.log(u) - np.log1p(-u)
    assert np.all(np.abs(tab - host) <= 4 * np.spacing(np.abs(host)) + 1e-300)
    assert tab[4] < 0 < tab[5]                           # u < 1/2 <=> w < 2^31


# ---------------------------------------------------------------------------------------------
# Row-interleaved slack phase of the MKP lockstep kernel: rows of very different
# slack widths, slack ranges that start exactly at / straddle a 128-spin group boundary, a spin
# count that is a multiple of 32, more rows than one batch and one group hold.

def _mkp_caps(n, m, caps, seed):
    """MKP instance with hand-set capacities (slack widths = bit lengths of caps)."""
    p = _mkp(n, m, 0.5, seed)
    b = np.array([caps[i % len(caps)] for i in range(m)], dtype=np.int64)
    return dataclasses.replace(p, b=b, name=f"mkp_caps_n{n}_m{m}")


@pytest.mark.parametrize("variant", [2, 2 | 64], ids=["lockstep", "lockstep_noprod"])
@pytest.mark.parametrize("n,m,caps", [
    (128, 30, [1, 3, 100000, 7, 65535, 2, 40000]),        # slack starts at a group boundary; widths 1..17
    (120, 30, [255, 255, 255, 255]),                      # 8-bit rows: 15 rows per group, several batches
    (96, 16, [1 << 20, 1, (1 << 20) - 1, 5]),             # 21-bit rows straddling the group boundary
    (100, 5, [4095, 1, 70000, 3, 2047]),                  # M <= 8 instantiation (2 rows per batch)
    (101, 12, [(1 << 17) - 1] * 12),                      # MM = 16, N = 101 + 12 * 17 = 305
    (107, 9, [(1 << 17) - 1] * 8 + [(1 << 13) - 1]),      # N = 107 + 8 * 17 + 13 = 256: a multiple of 32 and 128
])
def test_mkp_lockstep_slack_rows_edge_cases(P, n, m, caps, variant):
    p = _mkp_caps(n, m, caps, 31)
    g = run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=9, R=40, K=5, T=40, flags=variant)
    assert g["info"]["kernel"] == 2 and g["info"]["lanes_per_replica"] == 1
