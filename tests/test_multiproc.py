"""The N > 1 path on CPU: world_size-2 gloo processes shard the replicas by global index, run their
shard (through the oracle -- the CUDA kernels need a GPU), and all-reduce(MIN) the packed
per-instance best.  The result must equal one process running every replica."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import saim_inputs as si
from paper_2501_04971_b200 import dist as sdist

R_PER_RANK, K, T, SEED = 12, 20, 100, 21


def _instances():
    """Two small QKP instances (config-0 shape) that reach feasible samples within K iterations."""
    probs = [si.qkp(20, 0.5, [0, 0, 0]), si.qkp(20, 0.5, [5, 1, 0])]
    return probs, [si.paper_P(p, 2.0) for p in probs], 20.0, 10.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    probs, Ps, eta, bmax = _instances()
    rep0, R = sdist.shard_range(rank, world, R_PER_RANK)
    keys = []
    for s, prob in enumerate(probs):
        op = oracle.OracleProblem.from_inputs(prob, Ps[s], eta, bmax, inst=s)
        res = op.run(SEED, R, K, T, rep0=rep0, nthreads=2)
        best = sdist.I64_MAX
        for j in range(R):
            if res["best_k"][j] >= 0:
                best = min(best, sdist.pack_best(res["best_f"][j], rep0 + j))
        keys.append(best)
    t = torch.tensor(keys, dtype=torch.int64)
    sdist.reduce_inst_best(t)
    if rank == 0:
        np.save(out_path, t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_equals_single_run(tmp_path):
    out = str(tmp_path / "keys.npy")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    probs, Ps, eta, bmax = _instances()
    for s, prob in enumerate(probs):
        op = oracle.OracleProblem.from_inputs(prob, Ps[s], eta, bmax, inst=s)
        res = op.run(SEED, 2 * R_PER_RANK, K, T, nthreads=4)
        want = sdist.I64_MAX
        for j in range(2 * R_PER_RANK):
            if res["best_k"][j] >= 0:
                want = min(want, sdist.pack_best(res["best_f"][j], j))
        assert int(got[s]) == want
    assert all(int(k) != sdist.I64_MAX for k in got)   # both instances reach feasible samples


def test_shard_range_and_packing():
    assert sdist.shard_range(0, 4, 4096) == (0, 4096)
    assert sdist.shard_range(3, 4, 4096) == (12288, 4096)
    with pytest.raises(ValueError):
        sdist.shard_range(4, 4, 8)
    with pytest.raises(ValueError):
        sdist.shard_range(255, 256, 8192)
    k = sdist.pack_best(-123456, 777)
    assert sdist.unpack_best(k) == (-123456, 777)
    assert sdist.pack_best(-5, 9) < sdist.pack_best(-5, 10) < sdist.pack_best(-4, 0)
    assert sdist.unpack_best(sdist.I64_MAX) == (None, None)
