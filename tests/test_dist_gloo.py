"""World-size-2 CPU tests (gloo) of the N>1 host logic.

The product's multi-GPU path (row sharding v % world == rank, one int64 sum all-reduce of the
voxel beliefs per iteration, NCCL id agreed over torch.distributed) cannot run here without
GPUs; these tests cover its host-side pieces with two CPU processes:
  * the NCCL-id bootstrap helper broadcasts one 128-byte id to every rank;
  * the decomposition itself: with each rank tracing only its rows (oracle graph build, the same
    rule the library applies) and the per-iteration exchange being an int64 all-reduce of
    fixed-point message sums, every rank ends with beliefs bit-identical to world = 1.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

Q = 2.0 ** 23


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _quantise(lam):
    return np.rint(np.clip(lam, -256, 256) * Q).astype(np.int64)


def _fixed_point_bp(p, g, n_iter, reduce_fn):
    """Flooding BP where T is the int64 sum of quantised messages, reduced by reduce_fn."""
    lam = np.zeros(g.E)
    T = np.zeros(p.V, np.int64)
    for _ in range(n_iter):
        oracle.ray_pass(p, g, T.astype(np.float64) / Q, lam)
        q = _quantise(lam)
        lam = q.astype(np.float64) / Q
        part = np.zeros(p.V, np.int64)
        np.add.at(part, g.vid, q)
        T = reduce_fn(part)
    return T


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2006_03512_b200.dist import bootstrap_nccl_id, owned_rows
        nid = bootstrap_nccl_id(id_fn=lambda: bytes(np.random.default_rng(7).integers(0, 256, 128, dtype=np.uint8)))
        w = synth.frames30(n_frames=2)
        p = oracle.Params.from_workload(w)
        g = oracle.build_graph(p, w.frames, rank=rank, world=world)
        rows = set(int(x) // w.frames[0].width for x in g.pixel)
        assert rows <= set(owned_rows(w.frames[0].height, rank, world))

        def allreduce(part):
            t = torch.from_numpy(part.copy())
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            return t.numpy()

        T = _fixed_point_bp(p, g, 3, allreduce)
        out[rank] = (nid, T, g.E, g.n_rays)
    finally:
        dist.destroy_process_group()


@pytest.mark.slow
def test_row_sharding_with_int64_allreduce_is_bit_identical():
    world = 2
    port = _free_port()
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] and len(res[0][0]) == 128      # one NCCL id on all ranks
    w = synth.frames30(n_frames=2)
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    T1 = _fixed_point_bp(p, g, 3, lambda part: part)
    assert res[0][2] + res[1][2] == g.E and res[0][3] + res[1][3] == g.n_rays
    assert np.array_equal(res[0][1], T1) and np.array_equal(res[1][1], T1)


def test_owned_rows_partition():
    from paper_2006_03512_b200.dist import owned_rows
    for world in (1, 2, 3, 8):
        rows = sorted(r for k in range(world) for r in owned_rows(480, k, world))
        assert rows == list(range(480))
