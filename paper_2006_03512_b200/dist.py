"""Data-parallel plumbing: one process per GPU, rays sharded by pixel row.

Rank r keeps the rays of pixel rows v % world == r of every frame (the C library applies the
rule inside mrf_add_frame); the only exchange is the per-iteration int64 sum all-reduce of the
voxel beliefs, done by NCCL inside mrf_bp_iterate.  torch.distributed is used only to agree on
the NCCL unique id.
"""

from __future__ import annotations

from . import MRFMap, MRF_COMM_EXTERNAL, MRF_COMM_NCCL, nccl_unique_id


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


class EmulatedRanks:
    """`world` ranks of one workload on ONE GPU: one MRF_COMM_EXTERNAL ctx per rank, each
    holding the pixel rows v % world == rank.  Every iteration each rank runs its ray kernels
    and K6 into its own int64 partial (mrf_bp_partial), the partials are summed on the device
    (a torch int64 add standing in for the NCCL all-reduce of the real multi-GPU path) and
    every rank takes the total (mrf_bp_finish).  Used where one ctx cannot hold a config's
    incidences (< 2^31 slots per ctx: the 0.02 m configs) and to test the sharded path."""

    def __init__(self, workload, world: int, stream_ptr=None):
        import torch
        self.world = world
        self.maps = [MRFMap.from_workload(workload, rank=r, world=world, comm=MRF_COMM_EXTERNAL)
                     for r in range(world)]
        if stream_ptr is None:
            stream_ptr = torch.cuda.current_stream().cuda_stream
        for m in self.maps:
            m.set_stream(stream_ptr)
        self.parts = None

    def add_frame(self, depth, K, T_wc):
        for m in self.maps:
            m.add_frame(depth, K, T_wc)

    def bp_iterate(self, n: int):
        import torch
        if self.parts is None:
            S = self.maps[0].belief_slots()
            self.parts = torch.empty((self.world, S), dtype=torch.int64, device="cuda")
        for _ in range(n):
            for m, part in zip(self.maps, self.parts):
                m.bp_partial(part, iterate=True)
            total = self.parts.sum(0)
            for m in self.maps:
                m.bp_finish(total)

    def reset(self):
        for m in self.maps:
            m.reset()

    def marginals(self, out=None):
        return self.maps[0].marginals(out)

    def graph_sizes(self):
        s = [m.graph_sizes(active=False) for m in self.maps]
        return dict(E=sum(x["E"] for x in s), n_rays=sum(x["n_rays"] for x in s))

    def layout_sizes(self):
        s = [m.layout_sizes() for m in self.maps]
        return dict(n_slots=sum(x["n_slots"] for x in s), n_runs=sum(x["n_runs"] for x in s),
                    n_belief_slots=s[0]["n_belief_slots"])

    def k6_path(self):
        paths = {m.k6_path() for m in self.maps}
        return paths.pop() if len(paths) == 1 else "mixed"

    def set_profiling(self, on=True):
        for m in self.maps:
            m.set_profiling(on)

    def profile_read(self):
        out = {}
        for m in self.maps:
            for k, (n, ms) in m.profile_read().items():
                a = out.setdefault(k, [0, 0.0])
                a[0] += n
                a[1] += ms
        return {k: tuple(v) for k, v in out.items()}

    def launch_count(self):
        return sum(m.launch_count() for m in self.maps)

    def close(self):
        for m in self.maps:
            m.close()
        self.maps = []
