"""Multi-GPU plumbing for pm4g: case-range sharding and communicator bootstrap.

The log is sharded by contiguous case-code ranges (SPEC.md S:228-231
"segments are disjoint, ordered, and cover all cases; no case is split across
segments"; reading R19), so every per-case quantity is computed
locally and only the A x A / A tables (allreduce) and the variant tables
(allgather + merge) cross GPUs -- inside libpm4g, over NCCL.  torch.distributed
is used only to carry the NCCL unique id from rank 0 to the other ranks.
"""
from __future__ import annotations


def shard_range(n_cases: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) case codes of `rank`: floor(r C / R) .. floor((r+1) C / R)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return (n_cases * rank) // world, (n_cases * (rank + 1)) // world


def shard_ranges(n_cases: int, world: int) -> list[tuple[int, int]]:
    return [shard_range(n_cases, r, world) for r in range(world)]


def broadcast_unique_id(uid: bytes | None, rank: int, src: int = 0, group=None) -> bytes:
    """Send the NCCL unique id (opaque bytes) from `src` to every rank."""
    import torch.distributed as dist
    obj = [uid if rank == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def make_comm(rank: int, world: int, group=None):
    """Create the library-owned NCCL communicator (torch.distributed must be initialised)."""
    from . import pm4g
    if world == 1:
        return pm4g.pm4g_comm_create(b"\0" * 128, 1, 0)
    uid = pm4g.pm4g_comm_unique_id() if rank == 0 else None
    uid = broadcast_unique_id(uid, rank, 0, group)
    return pm4g.pm4g_comm_create(uid, world, rank)
