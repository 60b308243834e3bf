"""The N > 1 path on CPU: world_size-2 gloo processes shard the replicas by global index, compute
their shard (through the oracle -- the CUDA kernels need a GPU -- written into the same output dict
saim_run fills: inst_best keys and per-replica best_x), and run the end-of-run exchange with the
function bench.py calls (dist.finalize: all-reduce(MIN) of the packed per-instance best, then the
winning replica's bitset from its owner).  The result must equal one process running every replica
(DESIGN.md section 8)."""
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


def _shard_outputs(rep0, R):
    """What saim_run returns for replicas [rep0, rep0 + R) of every instance (inst_best = min packed
    key over the shard, best_x per replica), computed by the oracle."""
    probs, Ps, eta, bmax = _instances()
    keys, bx = [], []
    for s, prob in enumerate(probs):
        op = oracle.OracleProblem.from_inputs(prob, Ps[s], eta, bmax, inst=s)
        res = op.run(SEED, R, K, T, rep0=rep0, nthreads=2)
        best = sdist.I64_MAX
        for j in range(R):
            if res["best_k"][j] >= 0:
                best = min(best, sdist.pack_best(res["best_f"][j], rep0 + j))
        keys.append(best)
        bx.append(res["best_x"].view(np.int32))
    return {"inst_best": torch.tensor(keys, dtype=torch.int64), "best_x": torch.from_numpy(np.stack(bx))}


def _worker(rank, world, port, out_path, reverse):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # reverse: rank r owns the range of rank world-1-r, so the winners (lowest replica index on
    # ties) live on the last rank and the bitset must travel to rank 0
    rep0, R = sdist.shard_range(world - 1 - rank if reverse else rank, world, R_PER_RANK)
    out = _shard_outputs(rep0, R)
    win_x = sdist.finalize(out, rep0, R)          # the exchange bench.py runs after every step
    np.save(out_path + f".{rank}.npy", np.concatenate([out["inst_best"].numpy(), win_x.numpy().ravel()]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("reverse", [False, True])
def test_two_rank_sharding_equals_single_run(tmp_path, reverse):
    out = str(tmp_path / "keys")
    mp.start_processes(_worker, args=(2, _free_port(), out, reverse), nprocs=2, join=True, start_method="spawn")
    ranks = [np.load(out + f".{r}.npy") for r in range(2)]
    assert np.array_equal(ranks[0], ranks[1])          # every rank holds the same result
    probs, Ps, eta, bmax = _instances()
    S = len(probs)
    got_keys, got_x = ranks[0][:S], ranks[0][S:].reshape(S, -1)
    for s, prob in enumerate(probs):
        op = oracle.OracleProblem.from_inputs(prob, Ps[s], eta, bmax, inst=s)
        res = op.run(SEED, 2 * R_PER_RANK, K, T, nthreads=4)
        want, wj = sdist.I64_MAX, None
        for j in range(2 * R_PER_RANK):
            if res["best_k"][j] >= 0 and sdist.pack_best(res["best_f"][j], j) < want:
                want, wj = sdist.pack_best(res["best_f"][j], j), j
        assert int(got_keys[s]) == want
        assert np.array_equal(got_x[s].astype(np.int32).view(np.uint32), res["best_x"][wj])
        f, rho = sdist.unpack_best(int(got_keys[s]))
        assert rho == wj and f == res["best_f"][wj]
    assert all(int(k) != sdist.I64_MAX for k in got_keys)   # both instances reach feasible samples


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
