"""Data-parallel plumbing: one process per GPU, rays sharded by pixel row.

Rank r keeps the rays of pixel rows v % world == r of every frame (the C library applies the
rule inside mrf_add_frame); the only exchange is the per-iteration int64 sum all-reduce of the
voxel beliefs, done by NCCL inside mrf_bp_iterate.  torch.distributed is used only to agree on
the NCCL unique id.
"""

from __future__ import annotations

from . import MRFMap, MRF_COMM_NCCL, nccl_unique_id


def owned_rows(height: int, rank: int, world: int):
    """Pixel rows a rank traces (mirrors FrameDesc.rows_owned in the library)."""
    return list(range(rank, height, world))


def bootstrap_nccl_id(group=None, id_fn=nccl_unique_id) -> bytes:
    """Rank 0 creates the 128-byte ncclUniqueId and broadcasts it over `group`."""
    import torch.distributed as dist
    obj = [id_fn() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    nid = obj[0]
    assert isinstance(nid, (bytes, bytearray)) and len(nid) == 128
    return bytes(nid)


def make_sharded_map(workload, group=None, **kw) -> MRFMap:
    """MRFMap for this process's rank of the default (or given) process group."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return MRFMap.from_workload(workload, **kw)
    nid = bootstrap_nccl_id(group)
    return MRFMap.from_workload(workload, rank=rank, world=world, comm=MRF_COMM_NCCL, nccl_id=nid, **kw)
