"""Host-side logic on CPU: bench.py's roofline model and the multi-GPU exchange's
edge cases (dist.finalize with instances that have no feasible sample)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2501_04971_b200 import dist as sdist  # noqa: E402


def _counters(decisions, uniforms, flips):
    return {"decisions": decisions, "uniforms": uniforms, "flips": flips}


def test_roofline_model_qkp_config2_numbers():
    """The round-1 review's recomputation of config 2 on 8(d)'s model: f_u = 0.0223, p_f = 0.00226,
    N = 312, M = 1 -> INT 4.93, FP32 5.07, MUFU 0.02 lane-ops, issue-bound at 148 x 128 x 1965 MHz /
    10.02 = 3.71e12 updates/s."""
    d = 255590400000
    c = _counters(d, int(0.0223 * d), int(0.00226 * d))
    rm = bench.roofline_model("qkp", 1, 312.0, c, 148, 1965.0)
    ops = rm["ops_per_update"]
    assert abs(ops["int"] - (4 + 18 * 0.0223 + 0.00226 * (0.75 * 312 + 1))) < 1e-3
    assert abs(ops["fp32"] - (5 + 3 * 0.0223)) < 1e-3
    assert abs(ops["issue"] - 10.02) < 0.01
    assert rm["binding"] == "issue"
    assert abs(rm["roof_updates_per_s"]["issue"] - 3.71e12) / 3.71e12 < 0.003
    # the INT roof (64 lanes/clk) is the runner-up
    assert rm["roof_updates_per_s"]["int"] > rm["roof_updates_per_s"]["issue"]


def test_roofline_model_mkp_and_smem():
    """MKP (M = 30, f_u = 0.9, p_f = 0.25): INT = 2M + 18 f_u + p_f M binds (64 lanes/clk); the
    SMEM class (2M + 2M p_f bytes at 128 B/clk) is looser."""
    d = 10 ** 12
    c = _counters(d, int(0.9 * d), int(0.25 * d))
    rm = bench.roofline_model("mkp", 30, 1011.0, c, 148, 1965.0)
    assert abs(rm["ops_per_update"]["int"] - (60 + 16.2 + 7.5)) < 1e-6
    assert abs(rm["ops_per_update"]["smem"] - (60 + 15.0)) < 1e-6
    assert rm["binding"] == "int"
    assert rm["peak_per_s"] == 148 * 64 * 1965e6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_finalize_single_rank_and_no_feasible_instance():
    """dist.finalize on a one-rank gloo group: an instance without a feasible sample (key INT64_MAX)
    gets an all-zero winning bitset; the other instance's winner is its own best_x row."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        best_x = torch.tensor([[[1, 2], [3, 4], [5, 6]], [[7, 8], [9, 10], [11, 12]]], dtype=torch.int32)
        inst_best = torch.tensor([sdist.I64_MAX, sdist.pack_best(-42, 2)], dtype=torch.int64)
        out = {"inst_best": inst_best, "best_x": best_x}
        win = sdist.finalize(out, rep0=0, R=3)
        assert win.tolist() == [[0, 0], [11, 12]]
        assert sdist.unpack_best(int(out["inst_best"][1])) == (-42, 2)
        # a rank whose range does not hold the winner contributes zeros
        win2 = sdist.finalize({"inst_best": inst_best.clone(), "best_x": best_x}, rep0=100, R=3)
        assert win2.tolist() == [[0, 0], [0, 0]]
    finally:
        dist.destroy_process_group()
