"""Multi-GPU sharding of the SAIM hot path.

Replicas are independent chains, so the path shards by GLOBAL replica index with no data-path
collective: rank r runs replicas [rep0, rep0 + R) of every instance (`saim_run(..., rep0, R, ...)`),
and because the uniforms are keyed on the global index the union of the shards is bit-identical to
one GPU running all replicas.  The exchange at the end of a run is the
per-instance best, packed as the int64 key (f << 20) | replica (INT64_MAX = none), reduced with MIN
over the process group, plus the winning replica's item bitset (ceil(n/32) words per instance)
from the rank that owns it: ~8 + 4 ceil(n/32) bytes per instance over NCCL (NVLink/NVSwitch) in
production, gloo in the CPU tests.  `finalize` is that exchange; bench.py and the multi-process
test call it on saim_run's output dict.
"""
from __future__ import annotations

from typing import Tuple

I64_MAX = (1 << 63) - 1


def shard_range(rank: int, world: int, R_per_rank: int) -> Tuple[int, int]:
    """Weak scaling: every rank runs R_per_rank replicas; rank r owns [r*R, (r+1)*R)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    if (rank + 1) * R_per_rank > (1 << 20):
        raise ValueError("global replica index exceeds the RNG counter field (2^20)")
    return rank * R_per_rank, R_per_rank


def pack_best(f: int, replica: int) -> int:
    return (int(f) << 20) | int(replica)


def unpack_best(key: int) -> Tuple[int, int]:
    if key == I64_MAX:
        return None, None
    return key >> 20, key & ((1 << 20) - 1)


def finalize(out, rep0: int, R: int, group=None):
    """End-of-run exchange on saim_run's outputs (torch tensors; device or CPU): all-reduce(MIN) of
    out["inst_best"] in place, then the winning replica's best_x row of every instance, contributed
    by the rank whose global range [rep0, rep0 + R) holds it and summed (zeros elsewhere) so every
    rank receives it.  Returns win_x [n_inst, Wn] int32 (zeros for an instance with no feasible
    sample)."""
    import torch
    import torch.distributed as dist
    inst_best, best_x = out["inst_best"], out["best_x"]
    dist.all_reduce(inst_best, op=dist.ReduceOp.MIN, group=group)
    valid = inst_best != I64_MAX
    loc = (inst_best & ((1 << 20) - 1)) - rep0
    mine = valid & (loc >= 0) & (loc < R)
    idx = loc.clamp(0, R - 1)
    sel = best_x[torch.arange(best_x.shape[0], device=best_x.device), idx]
    win_x = torch.where(mine[:, None], sel, torch.zeros_like(sel))
    dist.all_reduce(win_x, op=dist.ReduceOp.SUM, group=group)
    return win_x


def reduce_inst_best(inst_best, group=None):
    """All-reduce(MIN) of the packed per-instance best keys (a torch int64 tensor), in place."""
    import torch.distributed as dist
    dist.all_reduce(inst_best, op=dist.ReduceOp.MIN, group=group)
    return inst_best
