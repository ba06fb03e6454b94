"""Multi-GPU plumbing: one process per GPU, torch.distributed only for the bootstrap.

The library creates its own NCCL communicator (ams_pool_create with world > 1) from a
128-byte ncclUniqueId.  Rank 0 draws the id through the C ABI and this module
broadcasts the bytes over an existing torch.distributed process group (nccl on the GPU
box, gloo in the CPU tests).  Rows are sharded by the library's block-cyclic map
(ams_shard_locate); queries are replicated; per-shard top-k lists are merged inside
ams_match by an NCCL all-gather and a k-way merge kernel.
"""
from __future__ import annotations

from typing import Optional

from . import Pool, ams_get_nccl_unique_id, ams_shard_locate


def bootstrap_nccl_id(group=None) -> Optional[bytes]:
    """Rank 0's ncclUniqueId, identical on every rank of `group` (None if world == 1)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    obj = [ams_get_nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    assert isinstance(obj[0], (bytes, bytearray)) and len(obj[0]) == 128
    return bytes(obj[0])


def create_pool(dim, joint_dim, capacity, max_queries, max_k, dtype="bf16", shard_block=0, group=None,
                device: Optional[int] = None, force_collective: bool = False) -> Pool:
    """Collective: every rank of the torch.distributed group creates its shard.
    force_collective (world 1 only): build a 1-rank NCCL communicator so the world > 1 code
    path (shard merge, all-gather, final merge, peer exchange) runs on one GPU."""
    import torch
    import torch.distributed as dist
    rank, world = (dist.get_rank(group), dist.get_world_size(group)) if dist.is_initialized() else (0, 1)
    dev = torch.cuda.current_device() if device is None else device
    nid = bootstrap_nccl_id(group)
    if nid is None and force_collective:
        nid = ams_get_nccl_unique_id()
    return Pool(dim, joint_dim, capacity, max_queries, max_k, dtype=dtype, device=dev, rank=rank, world=world,
                nccl_id=nid, shard_block=shard_block)


def owned_range_overlaps(capacity: int, world: int, shard_block: int, rank: int, lo: int, hi: int) -> bool:
    """Does `rank` own any global row in [lo, hi)?  (host-side shard map query)"""
    if world == 1:
        return hi > lo
    B = shard_block if shard_block > 0 else -(-capacity // world)
    first_block, last_block = lo // B, (hi - 1) // B
    if last_block - first_block + 1 >= world:
        return True
    for b in range(first_block, last_block + 1):
        if ams_shard_locate(capacity, world, shard_block, min(b * B, capacity - 1))[0] == rank:
            return True
    return False
