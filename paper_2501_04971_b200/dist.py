"""Multi-GPU sharding of the SAIM hot path.

Replicas are independent chains, so the path shards by GLOBAL replica index with no data-path
collective: rank r runs replicas [rep0, rep0 + R) of every instance (`saim_run(..., rep0, R, ...)`),
and because the uniforms are keyed on the global index the union of the shards is bit-identical to
one GPU running all replicas.  The single exchange is the per-instance best, packed as the int64
key (f << 20) | replica (INT64_MAX = none), reduced with MIN over the process group (NCCL on
NVLink/NVSwitch in production, gloo in the CPU tests).
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


def reduce_inst_best(inst_best, group=None):
    """All-reduce(MIN) of the packed per-instance best keys (a torch int64 tensor), in place."""
    import torch.distributed as dist
    dist.all_reduce(inst_best, op=dist.ReduceOp.MIN, group=group)
    return inst_best
