#!/usr/bin/env python
"""Benchmark of the SAIM hot path on B200 (BASELINE.json metric: p-bit updates/s and SAIM
samples/s at QKP n=300 (config 2), 1 B200, as a fraction of the ALU roofline).

One step = one saim_run of the whole hot path (Algorithm 1 with all its anneals, readouts and
Lagrange steps) over config 2: 4096 replicas x K=200 iterations x T=1000 sweeps x N spins.
value = attempted p-bit updates per second = (replicas * K * T * N) / device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl reference]

N > 1 (torchrun): replicas are sharded by global replica index (weak scaling: every rank runs
4096 replicas with its own index range; the RNG is keyed on the global index so results equal a
one-GPU run of the union); the one exchange step is an all-reduce(MIN) of the packed per-instance
best (f << 20 | replica).  Timing: CUDA events on the launching stream around each step, L2
flushed (256 MiB write) between steps outside the events, barrier + synchronize around the timed
region, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import saim_inputs as si  # noqa: E402

# Per-SM, per-clock peaks of the B200 pipes (tools/ubench.cu, profiles/r01/ubench_b200.txt;
# B200_PROFILING.md unit counts): INT32 lanes, FP32 lanes, MUFU lanes, warp-instruction issue in
# lane-ops (4 SMSPs x 32), shared-memory bytes.
PEAK_PER_SM_CLK = {"int": 64, "fp32": 128, "mufu": 16, "issue": 128, "smem": 128}


def roofline_model(kind, M, N, c, sm_count, clk_mhz):
    """SURVEY.md 8(d) algorithmic op model per attempted p-bit update, path-weighted by this run's
    counters: f_u = uniforms / decisions (unsaturated decisions), p_f = flips / decisions.
      QKP (M <= 1): INT 4 + 18 f_u + p_f (0.75 N + M); FP32 5 + 3 f_u; MUFU f_u; SMEM p_f N bytes
      MKP:          INT 2M + 18 f_u + p_f M;          FP32 5 + 3 f_u; MUFU f_u; SMEM 2M + 2M p_f
    (issue = INT + FP32 + MUFU lane-ops).  The roof of each class is 148 SMs x its per-clock peak x
    the measured SM clock / its ops per update; the smallest roof binds."""
    dec = float(c["decisions"])
    f_u, p_f = c["uniforms"] / dec, c["flips"] / dec
    if kind == "qkp":
        ops = {"int": 4 + 18 * f_u + p_f * (0.75 * N + M), "fp32": 5 + 3 * f_u, "mufu": f_u,
               "smem": p_f * N}
    else:
        ops = {"int": 2 * M + 18 * f_u + p_f * M, "fp32": 5 + 3 * f_u, "mufu": f_u,
               "smem": 2 * M + 2 * M * p_f}
    ops["issue"] = ops["int"] + ops["fp32"] + ops["mufu"]
    hz = clk_mhz * 1e6
    roofs = {k: sm_count * PEAK_PER_SM_CLK[k] * hz / v for k, v in ops.items() if v > 0}
    bind = min(roofs, key=roofs.get)
    return {"f_u": f_u, "p_f": p_f, "ops_per_update": ops, "roof_updates_per_s": roofs, "binding": bind,
            "peak_per_s": sm_count * PEAK_PER_SM_CLK[bind] * hz}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def ncu_traffic_bytes(config):
    """dram__bytes_read.sum + dram__bytes_write.sum of the SAIM kernel per launch, from the committed
    ncu --set full capture of the same workload (a static artefact, not measured by this run: the
    path is on-chip and ncu cannot run inside the timed process)."""
    for p in (os.path.join(ROOT, "profiles", "r02", f"config{config}_ncu_raw_selected.csv"),
              os.path.join(ROOT, "profiles", "r01", "qkp_config2_K200_raw_selected.csv") if config == 2 else ""):
        if p and os.path.exists(p):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = 0.0
            for ln in open(p).read().splitlines()[1:]:
                name, unit, val = ln.split(",", 2)
                if name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    tot += float(val) * scale.get(unit, 1)
            return tot, os.path.relpath(p, ROOT)
    return None, None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(cfg, seconds_target=15.0, threads=None, seed=1, trace=False):
    """Time the oracle (as it stands) on a bounded sample of the workload on the host's cores:
    replicas [0, nrep) of instance 0, the first K = 2 Lagrange iterations."""
    import oracle
    threads = threads or os.cpu_count() or 1
    prob = cfg.instances[0]
    op = oracle.OracleProblem.from_inputs(prob, cfg.P[0], cfg.eta, cfg.beta_max, inst=0)
    N = op.N
    # calibrate: one replica, one iteration
    t0 = time.perf_counter()
    op.run(seed, 1, 1, cfg.T, nthreads=1)
    per_rep_iter = max(time.perf_counter() - t0, 1e-3)
    K = min(2, cfg.K)
    nrep = max(threads, int(round(seconds_target * threads / (per_rep_iter * K) / threads)) * threads)
    nrep = min(nrep, cfg.R)
    t0 = time.perf_counter()
    res = op.run(seed, nrep, K, cfg.T, nthreads=threads, trace=trace, final=trace)
    dt = time.perf_counter() - t0
    updates = nrep * K * cfg.T * N
    return {"updates_per_s": updates / dt, "samples_per_s": nrep * K / dt, "seconds": dt, "cores": threads,
            "nrep": nrep, "K": K, "seed": seed, "N": N, "result": res,
            "sample": f"{nrep} replicas x K={K} iterations x T={cfg.T} sweeps x N={N} spins of instance 0 of "
                      f"{cfg.name} (first {K} of {cfg.K} Lagrange iterations), {threads} threads, {cpu_model()}"}


def metric_name(cfg):
    return f"p-bit updates/sec (SAIM, {cfg.name}, BASELINE config {cfg.idx})"


def run_reference(args):
    """--impl reference: the oracle (plain C CPU SAIM) on the same workload/metric, bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = si.config_instances(args.config)
    per_step = max(5.0, 60.0 / max(1, args.steps + args.warmup))
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        r = oracle_sample(cfg, seconds_target=per_step, seed=1 + i)
        if i >= args.warmup:
            vals.append(r["updates_per_s"])
            info = r
    v = float(np.mean(vals))
    N = si.n_spins(cfg.instances[0])
    line = {
        "impl": "reference", "metric": metric_name(cfg), "value": v,
        "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cfg.R * cfg.K * cfg.T * N / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name} (BASELINE config {cfg.idx}): {cfg.R} replicas x K={cfg.K} x "
                               f"T={cfg.T} x N={N} (reference arm times a bounded sample of it)"},
        "samples_per_s": v / (cfg.T * N),
        "cpu_baseline": {"value": v, "unit": "updates/s", "cores": info["cores"], "kind": "oracle",
                         "sample": info["sample"]},
        "e2e": {"value": v, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-reference-variant", action="store_true",
                    help="skip timing the no-early-exit variant")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2501_04971_b200 as P
    from paper_2501_04971_b200 import dist as sdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    torch.cuda.set_device(dev)

    cfg = si.config_instances(args.config)
    Q, c, A, b = si.stack(cfg.instances)
    rep0, R = sdist.shard_range(rank, world, cfg.R)   # weak scaling: own global replica range
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    sol = P.Solver(Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, device=dev)   # saim_create (host -> HBM)
    t_create = time.perf_counter() - t0
    Ns = [sol.instance(s)["N"] for s in range(sol.n_inst)]
    kind = "qkp" if sol.info["kernel"] == 1 else "mkp"
    out = sol.alloc_outputs(R, cfg.K)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(seed):
        sol.run(seed, R, cfg.K, cfg.T, rep0=rep0, out=out, stream=stream)
        if world > 1:
            sdist.finalize(out, rep0, R)       # MIN of the packed best + the winning bitset (8(e))

    for i in range(args.warmup):
        step(1000 + i)
    torch.cuda.synchronize()

    # Transparency: the same workload with the exact frozen-anneal early exit disabled (every
    # sweep evaluated); identical outputs (tests/test_gpu_parity.py::test_freeze_exit_is_exact).
    nofreeze = None
    if not args.no_reference_variant and kind == "qkp":
        sol_nf = P.Solver(Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, device=dev, flags=P.FLAG_NO_FREEZE_EXIT)
        out_nf = sol_nf.alloc_outputs(R, cfg.K)
        sol_nf.run(999, R, cfg.K, cfg.T, rep0=rep0, out=out_nf, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sol_nf.run(1, R, cfg.K, cfg.T, rep0=rep0, out=out_nf, stream=stream)
        e1.record(stream)
        e1.synchronize()
        t_nf = e0.elapsed_time(e1) / 1e3
        nofreeze = {"value": R * cfg.K * cfg.T * sum(Ns) * world / t_nf, "unit": "updates/s",
                    "ms_per_step": 1e3 * t_nf, "counters": P.counters_dict(out_nf["counters"])}
        sol_nf.close()

    # ---- device-timed region: K steps, per-step CUDA events on the launching stream (init kernel +
    # SAIM kernel; the init kernel is ~2 us), L2 flush between steps outside the events ----
    clocks = ClockSampler(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    times, counters = [], []
    for i in range(args.steps):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(1 + i)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        counters.append(P.counters_dict(out["counters"]))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t_step = float(np.mean(times))
    t_total = float(np.sum(times))
    if world > 1:
        tt = torch.tensor([t_total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
    updates_per_step_rank = R * cfg.K * cfg.T * sum(Ns)
    updates_total = updates_per_step_rank * world * args.steps
    value = updates_total / t_total
    samples_per_s = R * cfg.K * sol.n_inst * world * args.steps / t_total

    # ---- roofline of the dominant kernel on SURVEY.md 8(d)'s algorithmic model ----
    c0 = counters[-1]
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    peaks = measured_peaks()
    sm_mhz = clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    N_avg = c0["decisions"] / float(R * cfg.K * cfg.T)    # decision-weighted mean N over instances
    M = cfg.instances[0].M
    rm = roofline_model(kind, M, N_avg, c0, sm_count, sm_mhz)
    upd_rank = updates_per_step_rank / t_step             # this rank's kernel rate
    bind = rm["binding"]
    achieved = upd_rank * rm["ops_per_update"][bind]      # algorithmic ops (or SMEM bytes) per second
    traffic, traffic_src = ncu_traffic_bytes(cfg.idx)

    # ---- end-to-end through the public API with HOST buffers: saim_create from host arrays (H2D
    # of the problem), saim_run, D2H of the results, every step; per-phase times for the setup and
    # readback rates ----
    e2e_times, t_cr, t_rb = [], [], []
    h2d = Q.nbytes if Q is not None else 0
    h2d += c.nbytes + A.nbytes + b.nbytes + 8 * sol.n_inst
    res_keys = ["best_f", "best_x", "best_k", "n_feasible", "inst_best", "counters"]
    d2h = sum(out[k].numel() * out[k].element_size() for k in res_keys)
    pinned = {k: torch.empty(out[k].shape, dtype=out[k].dtype, pin_memory=True) for k in res_keys}
    for i in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s2 = P.Solver(Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, device=dev)
        t1 = time.perf_counter()
        o2 = s2.run(7 + i, R, cfg.K, cfg.T, rep0=rep0)
        if world > 1:
            sdist.finalize(o2, rep0, R)
        stream.synchronize()
        t2 = time.perf_counter()
        for k in res_keys:
            pinned[k].copy_(o2[k], non_blocking=True)
        stream.synchronize()
        t3 = time.perf_counter()
        e2e_times.append(t3 - t0)
        t_cr.append(t1 - t0)
        t_rb.append(t3 - t2)
        s2.close()
    e2e_t = float(np.mean(e2e_times))
    if world > 1:
        tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())
    e2e_value = updates_per_step_rank * world / e2e_t

    line = None
    if rank == 0:
        line = {
            "metric": metric_name(cfg), "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name} (BASELINE config {cfg.idx}): {R} replicas/GPU/instance x K={cfg.K} "
                                   f"Lagrange iterations x T={cfg.T} sweeps x N={Ns if len(Ns) <= 4 else f'{min(Ns)}..{max(Ns)}'} spins",
                       "instances": sol.n_inst, "replicas_per_gpu": R, "K": cfg.K, "T": cfg.T,
                       "N": Ns if len(Ns) <= 4 else [min(Ns), max(Ns)],
                       "P": cfg.P if len(cfg.P) <= 4 else [min(cfg.P), max(cfg.P)], "eta": cfg.eta,
                       "beta_max": cfg.beta_max, "kernel": kind, "lanes_per_replica": sol.info["lanes_per_replica"],
                       "l2": "flushed between steps (256 MiB write outside the timed events)",
                       "parallelism": f"replicas sharded over {world} GPU(s), global replica index keyed RNG"},
            "samples_per_s": samples_per_s,
            "gpu_launches": 3 * args.steps,   # per step: init, main SAIM kernel, exact-replay kernel
            "roofline": {"bound": "alu" if bind != "smem" else "smem",
                         "achieved": achieved / (1e12 if bind != "smem" else 1e9),
                         "peak": rm["peak_per_s"] / (1e12 if bind != "smem" else 1e9),
                         "unit": "Tops/s" if bind != "smem" else "GB/s",
                         "frac": upd_rank / rm["roof_updates_per_s"][bind],
                         "traffic": traffic,
                         "traffic_unit": "DRAM bytes per launch",
                         "traffic_source": (f"static: ncu --set full capture {traffic_src} (not measured by this run)"
                                            if traffic_src else None),
                         "binding_class": bind,
                         "model": "SURVEY.md 8(d) algorithmic ops per attempted update x measured f_u, p_f",
                         "f_u": rm["f_u"], "p_f": rm["p_f"],
                         "ops_per_update": rm["ops_per_update"],
                         "roof_updates_per_s": rm["roof_updates_per_s"],
                         "peak_basis": f"{sm_count} SMs x per-SM-clock peaks {PEAK_PER_SM_CLK} (tools/ubench.cu) x "
                                       f"{sm_mhz:.0f} MHz (measured median SM clock during the timed region)",
                         "kernel_ms": 1e3 * t_step},
            "counters": c0,
            "evaluated_sweep_fraction": c0["sweeps"] / float(R * cfg.K * cfg.T * sol.n_inst),
            "no_freeze_exit": nofreeze,
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "setup": {"saim_create_ms": 1e3 * float(np.mean(t_cr)), "first_create_ms": 1e3 * t_create,
                      "h2d_bytes": int(h2d),
                      "h2d_GBps": h2d / float(np.mean(t_cr)) / 1e9,
                      "note": "saim_create = validation, slack extension, range proofs, layout on the host + one "
                              "H2D upload; the kernel prologue then stages the blob HBM -> SMEM by TMA "
                              "(DRAM bytes per launch: roofline.traffic)"},
            "readback": {"d2h_bytes": int(d2h), "ms": 1e3 * float(np.mean(t_rb)),
                         "GBps": d2h / float(np.mean(t_rb)) / 1e9},
        }
        if not args.no_cpu_baseline and world == 1:
            cb = oracle_sample(cfg, seconds_target=args.cpu_seconds, trace=True)
            line["cpu_baseline"] = {"value": cb["updates_per_s"], "unit": "updates/s", "cores": cb["cores"],
                                    "kind": "oracle", "sample": cb["sample"]}
            line["parity"] = parity_summary(P, sol, cfg, cb, stream)
        print(json.dumps(line), flush=True)
    sol.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def parity_summary(P, sol, cfg, cb, stream):
    """The GPU on the cpu_baseline's own sample (same seed, replicas, K): element-wise comparison of
    every readout with the oracle's, plus the decision-level report north_star asks for (near ties
    |u - sigma| < 2^-20 seen by the oracle, GPU fp64/double-double slow-path counts, mismatches)."""
    import torch
    o = cb["result"]
    nrep, K = cb["nrep"], cb["K"]
    g = sol.run(cb["seed"], nrep, K, cfg.T, trace=True, final=True, stream=stream)
    torch.cuda.synchronize()
    WN = (cb["N"] + 31) // 32
    gx = g["tr_x"][0].cpu().numpy().view(np.uint32)[..., :WN]
    mism_x = int(np.any(gx != o["tr_x"], axis=-1).sum())
    mism = {"samples_x": mism_x,
            "f": int((g["tr_f"][0].cpu().numpy() != o["tr_f"]).sum()),
            "feasible": int((g["tr_feas"][0].cpu().numpy() != o["tr_feas"]).sum()),
            "r": int(np.any(g["tr_r"][0].cpu().numpy() != o["tr_r"], axis=-1).sum()),
            "lambda": int(np.any(g["tr_lam"][0].cpu().numpy() != o["tr_lam"], axis=-1).sum()),
            "best_f": int((g["best_f"][0].cpu().numpy() != o["best_f"]).sum()),
            "flips": int(g["rep_flips"][0].cpu().numpy().astype(np.int64).sum() - o["counters"]["flips"])}
    gc = P.counters_dict(g["counters"])
    return {"sample": f"instance 0, replicas [0, {nrep}), K={K}, seed {cb['seed']} (the cpu_baseline's sample)",
            "mismatches": mism, "all_equal": all(v == 0 for v in mism.values()),
            "oracle_decisions": o["counters"]["decisions"], "oracle_near_ties_2^-20": o["counters"]["near_ties"],
            "oracle_binary128_fallbacks": o["counters"]["quad_fallbacks"],
            "gpu_fp64_slow_path": gc["fp64"], "gpu_uncertified": gc["uncertified"],
            "decision_mismatch_rate": 0.0 if mism_x == 0 else None}


if __name__ == "__main__":
    sys.exit(main())
