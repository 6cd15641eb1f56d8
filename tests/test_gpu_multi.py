"""The multi-GPU data plane through the C ABI.

  * On one GPU: the compacted reduction (K6 writes the touched tiles in compact order, a scatter
    puts the sums back) forced at world = 1 (MRF_COMPACT=1) gives beliefs and messages
    bit-identical to the plain path -- the kernels the NCCL path runs around its all-reduce.
  * On >= 2 GPUs (skipped below): real NCCL ranks, rows sharded v % world == rank, the
    all-reduce over the touched tiles every iteration; T bit-identical to world = 1 on every
    rank (integer sums: exact for any rank count and reduction order).
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synth  # noqa: E402
import paper_2006_03512_b200 as pkg  # noqa: E402

pytestmark = pytest.mark.gpu


def _run(w, n_iter, **kw):
    m = pkg.MRFMap.from_workload(w, **kw)
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    with m:
        for fr in w.frames:
            m.add_frame(fr.depth, fr.K, fr.T_wc)
        m.bp_iterate(n_iter)
        return m.export_beliefs(), m.export_messages(), m.marginals()


def test_compacted_reduction_bit_identical_one_gpu(monkeypatch):
    w = synth.frames30(n_frames=3)
    a = _run(w, 3)
    monkeypatch.setenv("MRF_COMPACT", "1")
    b = _run(w, 3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_nccl_data_plane_one_rank(monkeypatch):
    """The NCCL data plane on one GPU (MRF_NCCL_WORLD1=1: a one-rank communicator): the ncclMax
    of the touched-tile mask, the in-place ncclAllReduce of the compacted sums, the scatter and
    the async-error polling all run, through the C ABI; beliefs, messages and marginals
    bit-identical to the plain path, warm start included."""
    w = synth.frames30(n_frames=3)
    a = _run(w, 3)
    monkeypatch.setenv("MRF_NCCL_WORLD1", "1")
    b = _run(w, 3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    m = pkg.MRFMap.from_workload(w)
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    with m:
        m.set_profiling(True)
        for fr in w.frames[:2]:
            m.add_frame(fr.depth, fr.K, fr.T_wc)
        m.bp_iterate(1)
        m.add_frame(w.frames[2].depth, w.frames[2].K, w.frames[2].T_wc)  # the touched tiles change
        m.bp_iterate(2)
        prof = m.profile_read()
        assert prof["allreduce"][0] >= 3  # the NCCL all-reduce ran every iteration
        T = m.export_beliefs()
    monkeypatch.delenv("MRF_NCCL_WORLD1")
    m = pkg.MRFMap.from_workload(w)
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    with m:
        for fr in w.frames[:2]:
            m.add_frame(fr.depth, fr.K, fr.T_wc)
        m.bp_iterate(1)
        m.add_frame(w.frames[2].depth, w.frames[2].K, w.frames[2].T_wc)
        m.bp_iterate(2)
        assert np.array_equal(m.export_beliefs(), T)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2006_03512_b200.dist import make_sharded_map
        w = synth.frames30(n_frames=3)
        m = make_sharded_map(w)
        with m:
            m.set_stream(torch.cuda.current_stream().cuda_stream)
            for fr in w.frames:
                m.add_frame(fr.depth, fr.K, fr.T_wc)
            m.bp_iterate(3)
            out[rank] = (m.export_beliefs(), m.marginals(), m.graph_sizes(active=False)["E"])
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_nccl_ranks_bit_identical_to_one_gpu():
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    w = synth.frames30(n_frames=3)
    T1, marg1, _ = _run(w, 3)
    E1 = pkg.MRFMap.from_workload(w)
    with E1:
        for fr in w.frames:
            E1.add_frame(fr.depth, fr.K, fr.T_wc)
        e_total = E1.graph_sizes(active=False)["E"]
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_rank, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    assert sum(res[r][2] for r in range(world)) == e_total
    for r in range(world):
        assert np.array_equal(res[r][0], T1) and np.array_equal(res[r][1], marg1)
