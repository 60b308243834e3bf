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

# Algorithmic lane-ops per attempted update: fast path per decision,
# per drawn uniform (Philox4x32-10 / 4 + u map + logit + compare), per flip (n-element phi update:
# byte extract + convert + fma, plus the Q-row loads) -- counted from the kernel's counters.
OPS_DECISION = 8
OPS_UNIFORM = 30
OPS_FLIP_PER_ITEM = 3.25
LANES_PER_SM_CLK = 128          # 4 SMSPs x 32 FP32/INT32 lanes issue per clock (B200_PROFILING.md)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def ncu_traffic_bytes():
    """dram__bytes_read.sum + dram__bytes_write.sum of the SAIM kernel per launch, from the committed
    ncu --set full capture of the same workload (profiles/r01/qkp_config2_K200_raw_selected.csv)."""
    p = os.path.join(ROOT, "profiles", "r01", "qkp_config2_K200_raw_selected.csv")
    if not os.path.exists(p):
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for ln in open(p).read().splitlines()[1:]:
        name, unit, val = ln.split(",", 2)
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(val) * scale.get(unit, 1)
    return tot


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


def oracle_sample(cfg, seconds_target=15.0, threads=None, seed=1):
    """Time the oracle (as it stands) on a bounded sample of the workload on the host's cores."""
    import oracle
    threads = threads or os.cpu_count() or 1
    prob = cfg.instances[0]
    op = oracle.OracleProblem.from_inputs(prob, cfg.P[0], cfg.eta, cfg.beta_max, inst=0)
    N = op.N
    # calibrate: one replica, one iteration
    t0 = time.perf_counter()
    op.run(seed, 1, 1, cfg.T, nthreads=1)
    per_rep_iter = max(time.perf_counter() - t0, 1e-3)
    K = 2
    nrep = max(threads, int(round(seconds_target * threads / (per_rep_iter * K) / threads)) * threads)
    nrep = min(nrep, cfg.R)
    t0 = time.perf_counter()
    op.run(seed, nrep, K, cfg.T, nthreads=threads)
    dt = time.perf_counter() - t0
    updates = nrep * K * cfg.T * N
    return {"updates_per_s": updates / dt, "samples_per_s": nrep * K / dt, "seconds": dt, "cores": threads,
            "sample": f"{nrep} replicas x K={K} iterations x T={cfg.T} sweeps x N={N} spins of {cfg.name} "
                      f"(first {K} of {cfg.K} Lagrange iterations), {threads} threads, {cpu_model()}"}


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
        "impl": "reference", "metric": "p-bit updates/sec (SAIM, QKP n=300 config 2)", "value": v,
        "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cfg.R * cfg.K * cfg.T * N / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.R} replicas x K={cfg.K} x T={cfg.T} x N={N} "
                               "(reference arm times a bounded sample of it)"},
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
    sol = P.Solver(Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, device=dev)
    Ns = [sol.instance(s)["N"] for s in range(sol.n_inst)]
    n_items = cfg.instances[0].n
    out = sol.alloc_outputs(R, cfg.K)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(seed):
        sol.run(seed, R, cfg.K, cfg.T, rep0=rep0, out=out, stream=stream)
        if world > 1:
            sdist.reduce_inst_best(out["inst_best"])

    for i in range(args.warmup):
        step(1000 + i)
    torch.cuda.synchronize()

    # Transparency: the same workload with the exact frozen-anneal early exit disabled (every
    # sweep evaluated); identical outputs (tests/test_gpu_parity.py::test_freeze_exit_is_exact).
    nofreeze = None
    if not args.no_reference_variant:
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

    # ---- device-timed region: K steps, per-step CUDA events, L2 flush between steps ----
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

    # ---- kernel-only time of the dominant kernel (main SAIM kernel; init kernel is ~2 us) ----
    c0 = counters[-1]
    # evaluated decisions only (sweeps skipped by the exact early exit are not counted as work)
    evaluated = c0["decisions"] * c0["sweeps"] / float(R * cfg.K * cfg.T * sol.n_inst)
    ops = (evaluated * OPS_DECISION + c0["uniforms"] * OPS_UNIFORM
           + c0["flips"] * OPS_FLIP_PER_ITEM * n_items)
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    peaks = measured_peaks()
    sm_mhz = clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    peak_ops = sm_count * LANES_PER_SM_CLK * sm_mhz * 1e6
    achieved = ops / t_step
    # SURVEY.md 8(d) transparency variant: the roofline of a sampler that draws a uniform for every
    # update (f_u = 1, no saturation certificates), in updates/s, with this run's flip rate
    ops_per_update_rng_all = (OPS_DECISION + OPS_UNIFORM
                              + OPS_FLIP_PER_ITEM * n_items * c0["flips"] / float(c0["decisions"]))

    # ---- end-to-end through the public API with host buffers (create from host arrays = H2D,
    # run, D2H of the results), timed on the device stream with a host sync at the end ----
    e2e_times = []
    h2d = Q.nbytes + c.nbytes + A.nbytes + b.nbytes + 8 * sol.n_inst
    d2h = sum(out[k].numel() * out[k].element_size() for k in ["best_f", "best_x", "best_k", "n_feasible",
                                                                 "inst_best", "counters"])
    for i in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s2 = P.Solver(Q, c, A, b, cfg.P, cfg.eta, cfg.beta_max, device=dev)
        o2 = s2.run(7 + i, R, cfg.K, cfg.T, rep0=rep0)
        if world > 1:
            sdist.reduce_inst_best(o2["inst_best"])
        host = {k: o2[k].cpu() for k in ["best_f", "best_x", "best_k", "n_feasible", "inst_best", "counters"]}
        e2e_times.append(time.perf_counter() - t0)
        s2.close()
        del host
    e2e_t = float(np.mean(e2e_times))
    if world > 1:
        tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())
    e2e_value = updates_per_step_rank * world / e2e_t

    line = None
    if rank == 0:
        line = {
            "metric": "p-bit updates/sec (SAIM, QKP n=300 config 2)", "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name} (BASELINE config {cfg.idx}): {R} replicas/GPU x K={cfg.K} "
                                   f"Lagrange iterations x T={cfg.T} sweeps x N={Ns} spins",
                       "instances": sol.n_inst, "replicas_per_gpu": R, "K": cfg.K, "T": cfg.T, "N": Ns,
                       "P": cfg.P, "eta": cfg.eta, "beta_max": cfg.beta_max,
                       "l2": "flushed between steps (256 MiB write outside the timed events)",
                       "parallelism": f"replicas sharded over {world} GPU(s), global replica index keyed RNG"},
            "samples_per_s": samples_per_s,
            "gpu_launches": 2 * args.steps,
            "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_ops / 1e12, "unit": "Tops/s",
                         "frac": achieved / peak_ops, "traffic": ncu_traffic_bytes(),
                         "traffic_unit": "DRAM bytes per launch (ncu capture in profiles/r01; the path is on-chip)",
                         "ops_per_launch": ops, "ops_model": f"{OPS_DECISION}*evaluated decisions + {OPS_UNIFORM}*uniforms + "
                                                            f"{OPS_FLIP_PER_ITEM}*n*flips (lane-ops)",
                         "peak_basis": f"{sm_count} SMs x {LANES_PER_SM_CLK} lanes/clk x {sm_mhz:.0f} MHz "
                                       "(measured median SM clock under load)",
                         "rng_every_update": {
                             "roof_updates_per_s": peak_ops / ops_per_update_rng_all,
                             "value_over_roof": value / world / (peak_ops / ops_per_update_rng_all),
                             "ops_per_update": ops_per_update_rng_all,
                             "note": "roofline of a sampler drawing a uniform for every update (f_u = 1); "
                                     "the certified saturation skip lets the measured rate exceed it"},
                         "ncu": "profiles/r01/qkp_config2_K200_raw_selected.csv (issue slots, pipes, "
                                "shared-memory wavefronts, DRAM bytes)"},
            "counters": c0,
            "evaluated_sweep_fraction": c0["sweeps"] / float(R * cfg.K * cfg.T * sol.n_inst),
            "no_freeze_exit": nofreeze,
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
        }
        if not args.no_cpu_baseline and world == 1:
            cb = oracle_sample(cfg, seconds_target=args.cpu_seconds)
            line["cpu_baseline"] = {"value": cb["updates_per_s"], "unit": "updates/s", "cores": cb["cores"],
                                    "kind": "oracle", "sample": cb["sample"]}
        print(json.dumps(line), flush=True)
    sol.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
