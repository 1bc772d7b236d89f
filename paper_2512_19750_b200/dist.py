"""Host-side multi-GPU plumbing: contiguous row shards, one
process per GPU, NCCL unique-id broadcast over torch.distributed.  The merge
itself (all-reduce sum over counts, max over HLL registers) runs inside
gace_probe on the table's stream."""
from __future__ import annotations

import torch.distributed as dist


def shard_range(g: int, G: int, n: int) -> tuple[int, int]:
    """Rows [floor(gN/G), floor((g+1)N/G)) of shard g out of G."""
    return (g * n) // G, ((g + 1) * n) // G


def broadcast_unique_id(uid: bytes | None, src: int = 0) -> bytes:
    """Rank `src` passes its 128-byte ncclUniqueId; every rank returns it."""
    obj = [uid if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def dist_info(nrows_total: int):
    """DistInfo for this rank of the default process group (creates the NCCL id on rank 0)."""
    from .gace import DistInfo, nccl_unique_id
    rank, world = dist.get_rank(), dist.get_world_size()
    r0, _ = shard_range(rank, world, nrows_total)
    uid = broadcast_unique_id(nccl_unique_id() if rank == 0 else None) if world > 1 else None
    return DistInfo(rank, world, r0, nrows_total, uid)
