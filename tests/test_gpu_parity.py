"""GPU <-> oracle parity through the C ABI (marked gpu; run on a B200).

The CUDA path and the oracle (oracle/, plain C) share no code; both receive the same seeded
inputs (saim_inputs) and must agree BIT-EXACTLY on every integer output: per-iteration samples
x_k (incl. slack bits), f(x_k), feasibility, residuals r(x_k), Lagrange accumulators Lambda_k,
per-replica best (f, x, k), feasible counts, and the flip count.  Decisions are the exact real
predicate on both sides (R18), so no decision may differ; the kernel's `uncertified`
counter must be 0.
"""
import os

import numpy as np
import pytest

import oracle
import saim_inputs as si
from oracle.reference import brute_force_opt

pytestmark = pytest.mark.gpu
I64MAX = np.iinfo(np.int64).max


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_04971_b200 as P
    from paper_2501_04971_b200 import build
    build.build()
    return P


def gpu_run(P, Q, c, A, b, Pen, eta, beta_max, seed, R, K, T, rep0=0, trace=True, final=True, flags=0):
    import torch
    sol = P.Solver(Q, c, A, b, Pen, eta, beta_max, flags=flags)
    out = sol.run(seed, R, K, T, rep0=rep0, trace=trace, final=final)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    res["counters"] = P.counters_dict(out["counters"])
    res["info"] = sol.info
    res["inst"] = [sol.instance(s) for s in range(sol.n_inst)]
    sol.close()
    return res


def compare(g, o, s, reps, N, K, M):
    """GPU result g (all replicas of instance s) vs oracle result o for replica indices reps."""
    WN = (N + 31) // 32
    reps = np.asarray(reps)
    gx = g["tr_x"][s, reps].view(np.uint32)
    assert np.array_equal(gx[..., :WN], o["tr_x"]), "samples x_k differ"
    assert np.all(gx[..., WN:] == 0)
    assert np.array_equal(g["tr_f"][s, reps], o["tr_f"])
    assert np.array_equal(g["tr_feas"][s, reps], o["tr_feas"])
    if M:
        assert np.array_equal(g["tr_r"][s, reps], o["tr_r"])
        assert np.array_equal(g["tr_lam"][s, reps], o["tr_lam"])
    assert np.array_equal(g["best_f"][s, reps], o["best_f"])
    assert np.array_equal(g["best_k"][s, reps], o["best_k"])
    assert np.array_equal(g["best_x"][s, reps].view(np.uint32), o["best_x"])
    assert np.array_equal(g["n_feasible"][s, reps], o["n_feasible"])
    if "final_x" in o:
        assert np.array_equal(g["final_x"][s, reps].view(np.uint32)[..., :WN], o["final_x"])
        if M:
            assert np.array_equal(g["final_lam"][s, reps], o["final_lam"])


def run_both(P, probs, Pens, eta, beta_max, seed, R, K, T, reps=None, rep0=0, flags=0, block=None):
    Q, c, A, b = si.stack(probs)
    g = gpu_run(P, Q, c, A, b, Pens, eta, beta_max, seed, R, K, T, rep0=rep0, flags=flags)
    assert g["counters"]["uncertified"] == 0
    flips = 0
    for s, pr in enumerate(probs):
        op = oracle.OracleProblem.from_inputs(pr, Pens[s], eta, beta_max, inst=s)
        assert g["inst"][s]["N"] == op.N and (g["inst"][s]["s_o"], g["inst"][s]["s_c"]) == op.scales()
        rr = list(range(R)) if reps is None else list(reps)
        if reps is None:
            o = op.run(seed, R, K, T, rep0=rep0, trace=True, final=True)
            flips += o["counters"]["flips"]
            compare(g, o, s, rr, op.N, K, pr.M)
        else:
            for r in rr:                       # sampled replicas, one oracle call each (global index)
                o = op.run(seed, 1, K, T, rep0=rep0 + r, trace=True, final=True)
                compare(g, o, s, [r], op.N, K, pr.M)
                assert int(g["rep_flips"][s, r]) == o["counters"]["flips"], "trajectory (flip count) differs"
            if block is not None:              # a contiguous block of replicas, oracle threaded over it
                b0, nb = block
                o = op.run(seed, nb, K, T, rep0=rep0 + b0, trace=True, final=True)
                compare(g, o, s, list(range(b0, b0 + nb)), op.N, K, pr.M)
                assert int(g["rep_flips"][s, b0:b0 + nb].sum()) == o["counters"]["flips"], "trajectories differ"
    if reps is None:
        assert g["counters"]["flips"] == flips
    assert g["counters"]["decisions"] == sum(K * T * R * g["inst"][s]["N"] for s in range(len(probs)))
    return g


# ---------------------------------------------------------------------------------------------
def test_device_philox_matches_oracle_and_kat(P):
    rng = np.random.default_rng(0)
    inp = rng.integers(0, 2 ** 32, size=(500, 6), dtype=np.uint64).astype(np.uint32)
    inp[0] = 0
    inp[1] = 0xFFFFFFFF
    out = P.selftest_philox(inp)
    for i in range(inp.shape[0]):
        assert list(out[i]) == oracle.philox(inp[i, :4], inp[i, 4:])
    assert list(out[0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def test_logit_error_bound_exhaustive(P):
    """The fp32 logit's error over ALL 2^23 uniforms is inside the bound used to certify decisions."""
    r = P.selftest_logit()
    assert r["max_ratio"] < 0.5, r


def test_parity_config0_full(P):
    cfg = si.config_instances(0)
    g = run_both(P, cfg.instances, cfg.P, cfg.eta, cfg.beta_max, seed=1, R=cfg.R, K=cfg.K, T=cfg.T)
    # Eq. 2 optimum by brute force: every best is >= OPT and inst_best decodes to (f, replica)
    pr = cfg.instances[0]
    opt, _ = brute_force_opt(pr.Q, pr.c, pr.A, pr.b)
    bf = g["best_f"][0][g["best_k"][0] >= 0]
    assert bf.size and np.all(bf >= opt) and (bf == opt).mean() >= 0.5
    key = int(g["inst_best"][0])
    assert key >> 20 == bf.min()
    rho = key & ((1 << 20) - 1)
    assert g["best_f"][0][rho] == bf.min() and np.all(g["best_f"][0][:rho] > bf.min())


@pytest.mark.parametrize("seed", [2, 0xDEADBEEFCAFEF00D])
def test_parity_config0_seeds(P, seed):
    cfg = si.config_instances(0)
    run_both(P, cfg.instances, cfg.P, cfg.eta, cfg.beta_max, seed=seed, R=32, K=6, T=50)


def _qkp(n, d, seed, cap=None):
    p = si.qkp(n, d, [77, n, seed])
    if cap is not None:
        p.b[:] = cap
    return p


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 63, 64, 65, 95, 129])
def test_parity_ragged_sizes(P, n):
    """Ragged tails: N = n + q spans several 32-spin blocks with a partial last block."""
    p = _qkp(n, 0.5, 1)
    run_both(P, [p], [si.paper_P(p, 2.0)], 20.0, 10.0, seed=3, R=8, K=4, T=30)


def test_parity_edge_cases(P):
    # capacity 1 (one slack bit), T = 1 (fixed beta = beta_max), K = 1
    p = _qkp(24, 0.5, 2, cap=1)
    run_both(P, [p], [2.0], 20.0, 10.0, seed=4, R=8, K=1, T=1)
    run_both(P, [p], [2.0], 20.0, 10.0, seed=4, R=8, K=5, T=1)
    # eta = 0: penalty-method baseline
    p = _qkp(40, 0.25, 3)
    run_both(P, [p], [si.paper_P(p, 2.0)], 0.0, 10.0, seed=5, R=8, K=5, T=40)
    # linear objective with one constraint (0-1 knapsack), Q = None
    p = _qkp(50, 0.0, 4)
    p.Q = None
    run_both(P, [p], [5.0], 0.05, 50.0, seed=6, R=8, K=5, T=40)
    # unconstrained (M = 0)
    q = _qkp(20, 1.0, 5)
    q.M, q.A, q.b = 0, np.zeros((0, 20), np.int32), np.zeros(0, np.int64)
    run_both(P, [q], [1.0], 1.0, 5.0, seed=7, R=8, K=3, T=30)
    # Q entries beyond int8 -> int16 shared-memory storage
    p = _qkp(45, 0.5, 6)
    p.Q = (p.Q * 300).astype(np.int32)
    g = run_both(P, [p], [si.paper_P(p, 2.0)], 20.0, 10.0, seed=8, R=8, K=4, T=40)
    assert (g["info"]["q_bytes"], g["info"]["phi_packed"]) == (2, 0)
    # int8 Q whose |phi| bound exceeds int16 (299 x 127): int8 rows with fp32 phi (not packed)
    p = _qkp(300, 1.0, 13)
    p.Q = np.where(p.Q != 0, -127, 0).astype(np.int32)
    g = run_both(P, [p], [si.paper_P(p, 2.0)], 20.0, 10.0, seed=12, R=8, K=3, T=30)
    assert (g["info"]["q_bytes"], g["info"]["phi_packed"]) == (1, 0)
    # a high-beta, tiny-field regime (decisions near the sigma boundary exercise the certification)
    p = _qkp(30, 0.5, 7)
    run_both(P, [p], [0.01], 0.001, 0.05, seed=9, R=8, K=4, T=50)


@pytest.mark.parametrize("c0,packed", [(-32667, 1), (-32668, 0)])
def test_packed_phi_boundary(P, c0, packed):
    """phi is held as biased int16 pairs iff max_i |c_i| + sum_j |Q_ij| <= 32767 (saim_api.cu);
    at the boundary phi reaches +-32767 (biased 1 / 65535), still bit-exact against the oracle."""
    p = _qkp(40, 0.5, 21)
    p.Q[0, :] = 0
    p.Q[:, 0] = 0
    p.Q[0, 1] = p.Q[1, 0] = -100
    p.c[0] = c0
    p.Q[1, 2:] = 0
    p.Q[2:, 1] = 0
    g = run_both(P, [p], [si.paper_P(p, 2.0)], 20.0, 10.0, seed=22, R=8, K=3, T=30)
    assert g["info"]["phi_packed"] == packed


def test_parity_multi_instance_batch(P):
    """Instances with different N (different slack counts) in one launch; RNG keyed on instance."""
    probs = [_qkp(60, 0.5, s, cap=c) for s, c in enumerate([3, 200, 1500, 70000 // 50])]
    run_both(P, probs, [si.paper_P(p, 2.0) for p in probs], 20.0, 10.0, seed=10, R=16, K=4, T=30)


def test_sharding_invariance(P):
    """RNG keyed on the global replica index: two half-range launches equal one full launch."""
    cfg = si.config_instances(0)
    Q, c, A, b = si.stack(cfg.instances)
    full = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 11, 64, 5, 40)
    lo = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 11, 32, 5, 40, rep0=0)
    hi = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 11, 32, 5, 40, rep0=32)
    for k in ["tr_x", "tr_f", "best_f", "best_x", "final_x"]:
        assert np.array_equal(full[k][:, :32], lo[k]) and np.array_equal(full[k][:, 32:], hi[k])


def test_parity_config1_sampled(P):
    """BASELINE config 1 at full size (both densities in one launch, the bench's configuration);
    the oracle recomputes sampled replicas one by one."""
    cfg = si.config_instances(1)
    run_both(P, cfg.instances, cfg.P, cfg.eta, cfg.beta_max, seed=1, R=cfg.R, K=cfg.K, T=cfg.T,
             reps=[0, 377, 1023], block=(512, 32))


def test_parity_config2_sampled(P):
    """BASELINE config 2 (headline) at full size; sampled replicas (the first, the last and a
    contiguous block of 48) against the oracle."""
    cfg = si.config_instances(2)
    g = run_both(P, cfg.instances, cfg.P, cfg.eta, cfg.beta_max, seed=1, R=cfg.R, K=cfg.K, T=cfg.T,
                 reps=[0, 4095], block=(1024, 48))
    assert (g["info"]["q_bytes"], g["info"]["phi_packed"]) == (1, 1)


@pytest.mark.parametrize("cfg_idx", [0, 1])
def test_freeze_exit_is_exact(P, cfg_idx):
    """Stopping an anneal after a fully certified-frozen sweep
    gives bit-identical outputs to evaluating every sweep."""
    cfg = si.config_instances(cfg_idx)
    Q, c, A, b = si.stack(cfg.instances)
    R, K = (64, cfg.K) if cfg_idx == 0 else (256, 10)
    on = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 5, R, K, cfg.T)
    off = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 5, R, K, cfg.T, flags=P.FLAG_NO_FREEZE_EXIT)
    for k in ["tr_x", "tr_f", "tr_feas", "tr_r", "tr_lam", "best_f", "best_k", "best_x", "n_feasible",
              "final_x", "final_lam", "inst_best"]:
        assert np.array_equal(on[k], off[k]), k
    for k in ["decisions", "flips", "uniforms", "feasible", "uncertified"]:
        assert on["counters"][k] == off["counters"][k], k
    assert off["counters"]["sweeps"] == R * K * cfg.T * len(cfg.instances)
    assert on["counters"]["sweeps"] <= off["counters"]["sweeps"]


@pytest.mark.parametrize("cfg_idx", [0, 1, 2])
def test_qkp_hot_loop_is_exact(P, cfg_idx):
    """The hot-block loop changes how sweeps are executed, not what
    they decide: every output, every replica's flip count and the data-determined counters agree
    with the general path alone."""
    cfg = si.config_instances(cfg_idx)
    Q, c, A, b = si.stack(cfg.instances)
    R, K = (64, cfg.K) if cfg_idx == 0 else (512, 8)
    on = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 6, R, K, cfg.T)
    off = gpu_run(P, Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, 6, R, K, cfg.T, flags=P.FLAG_QKP_NO_HOT_LOOP)
    for k in ["tr_x", "tr_f", "tr_feas", "tr_r", "tr_lam", "best_f", "best_k", "best_x", "n_feasible",
              "final_x", "final_lam", "inst_best", "rep_flips"]:
        assert np.array_equal(on[k], off[k]), k
    for k in ["decisions", "flips", "uniforms", "feasible", "uncertified", "sweeps"]:
        assert on["counters"][k] == off["counters"][k], k


# ---------------------------------------------------------------------------------------------
# MKP kernel (linear objective, M >= 2; BASELINE configs 3-4)

def _mkp(n, m, t, seed):
    return si.mkp(n, m, t, [88, n, m, seed])


# MKP kernel variants: default (speculative sub-warp kernel G = 8 for M <= 8, lockstep for M > 8), lockstep,
# outcome tree with L = 2 and 4, row split over 2 lanes (honoured for M > 8; else the default)
MKP_VARIANTS = [("default", 0), ("lockstep", 2), ("lockstep_noprod", 2 | 64), ("tree_L2", 4), ("tree_L4", 8),
                ("split2", 16)]
# speculative sub-warp kernel with G = 2, 4, 8, 16, 32 lanes per replica (instantiated for M <= 8)
MKP_SPEC = [("spec2", 1024), ("spec4", 256), ("spec8", 512), ("spec16", 2048), ("spec32", 4096)]
SPEC_LANES = {1024: 2, 256: 4, 512: 8, 2048: 16, 4096: 32}


@pytest.mark.parametrize("variant", [v for _, v in MKP_VARIANTS], ids=[k for k, _ in MKP_VARIANTS])
@pytest.mark.parametrize("n,m", [(7, 2), (30, 3), (33, 5), (64, 8), (40, 9), (26, 10), (20, 16), (25, 30), (22, 32)])
def test_mkp_parity_small(P, n, m, variant):
    """Small MKP instances across the constraint-count buckets (MM = 4, 8, 16, 32) with ragged N,
    for every MKP kernel (R = 40 leaves a partial replica group / warp)."""
    p = _mkp(n, m, 0.5, 1)
    g = run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=12, R=40, K=4, T=30, flags=variant)
    assert g["info"]["kernel"] == 2
    default = 8 if m <= 8 else 1          # speculative sub-warp kernel (G = 8) / lockstep
    want = {0: default, 2: 1, 66: 1, 4: 2, 8: 4, 16: 2}[variant]
    assert g["info"]["lanes_per_replica"] == want


@pytest.mark.parametrize("variant", [v for _, v in MKP_SPEC], ids=[k for k, _ in MKP_SPEC])
@pytest.mark.parametrize("n,m", [(7, 2), (30, 3), (33, 5), (64, 8), (100, 5), (131, 4)])
def test_mkp_spec_parity_small(P, n, m, variant):
    """The speculative sub-warp kernel for every G on small MKP instances with
    ragged N (partial last block, partial last word, N > 128: two Philox groups) and R = 41
    (a partial chain group in the last warp); T = 1 as well (fixed beta, no beta = 0 sweep)."""
    p = _mkp(n, m, 0.5, 1)
    g = run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=12, R=41, K=4, T=30, flags=variant)
    assert g["info"]["kernel"] == 2 and g["info"]["lanes_per_replica"] == SPEC_LANES[variant]
    run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=13, R=9, K=3, T=1, flags=variant)


@pytest.mark.parametrize("variant", [0, 256, 2048], ids=["default_spec8", "spec4", "spec16"])
def test_mkp_spec_edge_cases(P, variant):
    """Edge cases of the speculative sub-warp kernel: N > 256 (three Philox groups, a spin table of
    more than 8 words), T = 2 (only the beta = 0 sweep and beta_max), K = 1, the penalty method
    (eta = 0), no penalty (P = 0), a huge beta_max (every decision saturates after the first
    sweeps), a single replica, and a batch of two instances with different N in one launch."""
    big = _mkp(300, 4, 0.5, 41)
    run_both(P, [big], [si.paper_P(big, 5.0)], 0.05, 50.0, seed=31, R=9, K=2, T=12, flags=variant)
    p = _mkp(45, 6, 0.5, 42)
    run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=32, R=17, K=3, T=2, flags=variant)
    run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=33, R=17, K=1, T=1, flags=variant)
    run_both(P, [p], [si.paper_P(p, 5.0)], 0.0, 50.0, seed=34, R=8, K=3, T=20, flags=variant)      # eta = 0
    run_both(P, [p], [0.0], 0.05, 50.0, seed=35, R=8, K=3, T=20, flags=variant)                    # P = 0
    run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 1e6, seed=36, R=8, K=3, T=20, flags=variant)      # saturated
    run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=37, R=1, K=4, T=30, flags=variant)     # one replica
    q = _mkp(45, 6, 0.25, 43)
    run_both(P, [p, q], [si.paper_P(p, 5.0), si.paper_P(q, 5.0)], 0.05, 50.0, seed=38, R=13, K=3, T=25, flags=variant)
    # a large instance (N ~ 900 spins: 14 KB of per-chain tables, few warps per CTA) with more
    # chains than one wave of CTAs holds
    huge = _mkp(800, 5, 0.5, 44)
    g = run_both(P, [huge], [si.paper_P(huge, 5.0)], 0.05, 50.0, seed=39, R=700, K=2, T=6, reps=[0, 350, 699],
                 flags=variant)
    assert g["info"]["kernel"] == 2


def test_mkp_spec_needs_few_constraints(P):
    p = _mkp(26, 10, 0.5, 1)
    with pytest.raises(P.SaimError) as ei:
        P.Solver(p.Q, p.c, p.A, p.b, si.paper_P(p, 5.0), 0.05, 50.0, flags=P.FLAG_MKP_SPEC4)
    assert ei.value.code == P.SAIM_ESMEM


@pytest.mark.parametrize("variant", [v for _, v in MKP_VARIANTS], ids=[k for k, _ in MKP_VARIANTS])
def test_mkp_parity_tiny_capacities(P, variant):
    p = _mkp(12, 3, 0.1, 2)
    p.b[:] = [1, 2, 3]
    run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=13, R=32, K=5, T=25, flags=variant)
    run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=13, R=32, K=3, T=1, flags=variant)  # fixed beta


@pytest.mark.parametrize("variant", [v for _, v in MKP_SPEC], ids=[k for k, _ in MKP_SPEC])
def test_mkp_spec_parity_tiny_capacities(P, variant):
    p = _mkp(12, 3, 0.1, 2)
    p.b[:] = [1, 2, 3]
    run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=13, R=32, K=5, T=25, flags=variant)


def test_mkp_kernels_agree_on_counters(P):
    """All MKP kernels make the same decisions, so every output and the data-determined counters
    (flips, feasible samples, Philox calls) agree exactly.  ('uniforms' is not compared: whether a
    spin within a rounding margin of saturation counts as having drawn u depends on each kernel's
    error bound; the decision itself is certified either way.)"""
    for p in (_mkp(100, 5, 0.5, 21), _mkp(60, 12, 0.5, 22)):
        Q, c, A, b = si.stack([p])
        runs = [gpu_run(P, Q, c, A, b, [si.paper_P(p, 5.0)], 0.05, 50.0, 3, 70, 6, 60, flags=v)
                for _, v in MKP_VARIANTS + (MKP_SPEC if p.M <= 8 else [])]
        for r in runs[1:]:
            for k in ["tr_x", "tr_f", "tr_feas", "tr_r", "tr_lam", "best_f", "best_k", "best_x", "n_feasible",
                      "final_x", "final_lam", "inst_best"]:
                assert np.array_equal(runs[0][k], r[k]), k
            for k in ["decisions", "flips", "sweeps", "feasible", "philox", "uncertified"]:
                assert runs[0]["counters"][k] == r["counters"][k], k


@pytest.mark.parametrize("variant", [0, 2, 4, 256], ids=["default", "lockstep", "tree_L2", "spec4"])
def test_mkp_parity_config3_sampled(P, variant):
    """Config 3 (three tightness variants in one launch) at full size; sampled replicas."""
    cfg = si.config_instances(3)
    run_both(P, cfg.instances, cfg.P, cfg.eta, cfg.beta_max, seed=1, R=cfg.R, K=cfg.K, T=cfg.T,
             reps=[0, 2047], flags=variant)


@pytest.mark.parametrize("variant", [0, 16], ids=["default", "split2"])
def test_mkp_parity_config4_sampled(P, variant):
    """Config 4 shape (64 instances x 256 replicas, n=500, M=30) with K reduced to 4 so the
    oracle can replay sampled replicas; the launch configuration is the full one."""
    cfg = si.config_instances(4)
    g = run_both(P, cfg.instances[:8], cfg.P[:8], cfg.eta, cfg.beta_max, seed=1, R=cfg.R, K=4, T=cfg.T,
                 reps=[0, 255], flags=variant)
    assert g["info"]["kernel"] == 2


# ---------------------------------------------------------------------------------------------
# Maximum sizes and degenerate problems

def test_qkp_largest_resident_instance(P):
    """n = 420 items (int8 Q, 4 words per lane-row: ~212 KB of shared memory, one warp per CTA)."""
    p = _qkp(420, 0.5, 11)
    g = run_both(P, [p], [si.paper_P(p, 2.0)], 20.0, 10.0, seed=14, R=3, K=2, T=6)
    assert g["info"]["smem_bytes"] > 200_000


def test_qkp_too_large_is_esmem(P):
    p = _qkp(470, 0.5, 12)
    with pytest.raises(P.SaimError) as ei:
        P.Solver(p.Q, p.c, p.A, p.b, 10.0, 20.0, 10.0)
    assert ei.value.code == P.SAIM_ESMEM


@pytest.mark.parametrize("variant", [v for _, v in MKP_VARIANTS], ids=[k for k, _ in MKP_VARIANTS])
def test_mkp_largest_constraint_count(P, variant):
    """M = 32 constraints (the MKP kernels' maximum) with n = 300 items."""
    p = _mkp(300, 32, 0.5, 3)
    run_both(P, [p], [si.paper_P(p, 5.0)], 0.05, 50.0, seed=15, R=33, K=2, T=4, flags=variant)


def test_degenerate_problems(P):
    # zero objective: only the penalty and Lagrange terms act
    p = _qkp(40, 0.5, 13)
    p.Q[:] = 0
    p.c[:] = 0
    run_both(P, [p], [2.0], 20.0, 10.0, seed=16, R=8, K=4, T=20)
    # P = 0 (no penalty): the Lagrange term alone shapes L
    p = _qkp(40, 0.5, 14)
    run_both(P, [p], [0.0], 20.0, 10.0, seed=17, R=8, K=4, T=20)
    # huge beta_max: everything saturates after the first sweeps (deterministic descent)
    run_both(P, [p], [si.paper_P(p, 2.0)], 20.0, 1e6, seed=18, R=8, K=4, T=20)
    # MKP with a row of zero weights (its slack bits still exist)
    m = _mkp(30, 3, 0.5, 4)
    m.A[1, :] = 0
    m.b[1] = 7
    for v in (0, 2, 4, 8, 16, 256, 512, 1024, 2048, 4096):
        run_both(P, [m], [si.paper_P(m, 5.0)], 0.05, 50.0, seed=19, R=32, K=3, T=20, flags=v)
    # M > 8 with a row of zero weights in the second lane's half (row split)
    m = _mkp(30, 12, 0.5, 5)
    m.A[10, :] = 0
    m.b[10] = 5
    for v in (0, 2, 16):
        run_both(P, [m], [si.paper_P(m, 5.0)], 0.05, 50.0, seed=20, R=24, K=3, T=20, flags=v)
