"""GPU parity of the sparse-brick variant (DESIGN.md
reading R23) against the oracle, through the C ABI: the brick allocation mask and the empty-skip
graph bit-exact (integer work), messages 1e-3 relative and marginals 1e-4 (the per-ray bars)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2006_03512_b200 as pkg  # noqa: E402

pytestmark = pytest.mark.gpu

MSG_TOL = 1e-3
MARG_TOL = 1e-4


def _sparse_map(w, frames=None, brick=8):
    m = pkg.MRFMap.from_workload(w)
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    m.set_sparse_bricks(brick)
    for fr in (w.frames if frames is None else frames):
        m.add_frame(fr.depth, fr.K, fr.T_wc)
    return m


def _msg_err(lam, ref):
    return float(np.max(np.abs(lam.astype(np.float64) - ref) / np.maximum(1.0, np.abs(ref)))) if len(ref) else 0.0


@pytest.mark.parametrize("name", ["tiny", "tiny_frames", "frame1"])
def test_sparse_graph_bitexact_and_bp(name):
    w = {"tiny": synth.tiny, "tiny_frames": synth.tiny_frames, "frame1": synth.single_frame}[name]()
    p = oracle.Params.from_workload(w)
    bk = oracle.alloc_bricks(p, w.frames)
    g = oracle.build_graph(p, w.frames, bricks=bk)
    n_iter = 2 if name == "frame1" else 5
    lam_ref, T_ref = oracle.bp(p, g, n_iter)
    with _sparse_map(w) as m:
        assert np.array_equal(m.export_bricks(), bk.mask)
        gg = m.export_graph()
        for k in ("row_ptr", "vid", "off_q", "pixel"):
            assert np.array_equal(gg[k], getattr(g, k)), k
        assert g.E < oracle.build_graph(p, w.frames[:1]).E * len(w.frames)  # cells were skipped
        m.bp_iterate(n_iter)
        lam = m.export_messages()
        marg = m.marginals()
    assert _msg_err(lam, lam_ref) <= MSG_TOL
    assert np.max(np.abs(marg - oracle.marginals(p, T_ref))) <= MARG_TOL
    assert np.all(marg[~bk.cell_mask(p)] == np.float32(p.prior))  # unallocated space keeps the prior


def test_sparse_frames30_sampled_rays():
    """30 frames: the allocation over all frames bit-exact, and 3000 sampled pixels traced one by
    one by the oracle's empty-skip walk bit-exact against mrf_export_rays."""
    w = synth.frames30()
    p = oracle.Params.from_workload(w)
    bk = oracle.alloc_bricks(p, w.frames)
    with _sparse_map(w) as m:
        mask = m.export_bricks()
        sizes = m.graph_sizes()
        H, W = w.frames[0].depth.shape
        rng = np.random.default_rng(5)
        key = np.unique(rng.integers(0, len(w.frames) * H * W, 3000))
        fsel, psel = (key // (H * W)).astype(np.int32), (key % (H * W)).astype(np.int64)
        got = m.export_rays(fsel, psel)
    assert np.array_equal(mask, bk.mask)
    assert sizes["E"] < 846709585  # the dense frames30 graph
    lens = np.diff(got["row_ptr"])
    for fi in np.unique(fsel):
        idx = np.nonzero(fsel == fi)[0]
        sub = oracle.trace_pixels(p, w.frames[fi], psel[idx], int(fi), bricks=bk)
        order = {int(px): k for k, px in enumerate(sub.pixel)}
        for i in idx:
            k = order.get(int(psel[i]))
            s0, s1 = got["row_ptr"][i], got["row_ptr"][i + 1]
            if k is None:
                assert lens[i] == 0
                continue
            e0, e1 = sub.row_ptr[k], sub.row_ptr[k + 1]
            assert np.array_equal(got["vid"][s0:s1], sub.vid[e0:e1])
            assert np.array_equal(got["off_q"][s0:s1], sub.off_q[e0:e1])


def test_sparse_mode_rules():
    w = synth.tiny_frames(n_frames=3)
    m = pkg.MRFMap.from_workload(w)
    with m:
        with pytest.raises(pkg.MrfError) as e:
            m.set_sparse_bricks(6)  # not a power of two
        assert e.value.status == 1
        with pytest.raises(pkg.MrfError):
            m.export_bricks()  # dense
        m.set_sparse_bricks(8)
        m.add_frame(w.frames[0].depth, w.frames[0].K, w.frames[0].T_wc)
        with pytest.raises(pkg.MrfError) as e:
            m.set_sparse_bricks(4)  # frames already added
        assert e.value.status == 6
        m.add_frame(w.frames[1].depth, w.frames[1].K, w.frames[1].T_wc)
        m.bp_iterate(1)
        m.add_frame(w.frames[2].depth, w.frames[2].K, w.frames[2].T_wc)  # after use: re-walk (R24)
        m.bp_iterate(1)
        mf = pkg.MRFMap.from_workload(w)
        with mf:  # sparse + matrix-free: the allocation is fixed once the graph is used
            mf.set_sparse_bricks(8)
            mf.set_matrix_free(1)
            mf.add_frame(w.frames[0].depth, w.frames[0].K, w.frames[0].T_wc)
            mf.bp_iterate(1)
            with pytest.raises(pkg.MrfError) as e:
                mf.add_frame(w.frames[1].depth, w.frames[1].K, w.frames[1].T_wc)
            assert e.value.status == 6
        m.reset()  # clears the allocation, keeps the mode
        assert m.export_bricks().sum() == 0
        m.add_frame(w.frames[2].depth, w.frames[2].K, w.frames[2].T_wc)
        p = oracle.Params.from_workload(w)
        assert np.array_equal(m.export_bricks(), oracle.alloc_bricks(p, [w.frames[2]]).mask)


def test_sparse_bricks_with_keyframe_averages():
    """The two paper-model modes compose: keyframe-average messages over the empty-skip graph
    of a sparse-brick map, against oracle.kf_bp on the oracle's sparse graph."""
    w = synth.tiny_frames(n_frames=4)
    p = oracle.Params.from_workload(w)
    bk = oracle.alloc_bricks(p, w.frames)
    g = oracle.build_graph(p, w.frames, bricks=bk)
    lam_ref, lbar_ref, T_ref = oracle.kf_bp(p, g, 5, F=len(w.frames))
    m = pkg.MRFMap.from_workload(w)
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    m.set_sparse_bricks(8)
    m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
    for fr in w.frames:
        m.add_frame(fr.depth, fr.K, fr.T_wc)
    with m:
        assert np.array_equal(m.export_graph()["vid"], g.vid)
        m.bp_iterate(5)
        lam = m.export_messages()
        marg = m.marginals()
    assert _msg_err(lam, lam_ref) <= MSG_TOL
    assert np.max(np.abs(marg - oracle.marginals(p, T_ref))) <= MARG_TOL


def _carry_messages(g_old, lam_old, g_new, V):
    """Warm start across a re-walk (reading R24): each incidence of the new graph takes the message
    of the same (frame, pixel, voxel) in the old graph, 0 if it is new (host-side reference)."""
    def keys(g):
        ray = np.repeat(np.arange(g.n_rays), np.diff(g.row_ptr))
        return (g.frame[ray].astype(np.int64) << 52) | (g.pixel[ray].astype(np.int64) << 32) | g.vid.astype(np.int64)
    ko, kn = keys(g_old), keys(g_new)
    order = np.argsort(ko)
    pos = np.searchsorted(ko[order], kn)
    pos = np.minimum(pos, len(ko) - 1)
    hit = ko[order][pos] == kn
    out = np.zeros(g_new.E, np.float64)
    out[hit] = np.asarray(lam_old, np.float64)[order][pos[hit]]
    assert hit.sum() == g_old.E  # every old incidence survives (the allocation only grows)
    return out


@pytest.mark.parametrize("name,k,n_after", [("tiny_frames", 2, 2), ("frames30_3", 1, 1)])
def test_sparse_keyframes_after_use(name, k, n_after):
    """P:205 "When adding new depth images, new bricks are allocated" (reading R24): keyframes added
    after iterating grow the allocation under rays already walked.  Every frame is walked again
    against the grown allocation: the graph equals the oracle's empty-skip graph over all frames
    (bit-exact); every old incidence keeps its message and the new ones start at 0 (the host-side
    (frame, pixel, voxel) mapping, exact); the beliefs are unchanged by the re-walk; the next
    iterations match the oracle continued from that state."""
    w = synth.tiny_frames(n_frames=4) if name == "tiny_frames" else synth.frames30(n_frames=3)
    p = oracle.Params.from_workload(w)
    g_old = oracle.build_graph(p, w.frames[:k], bricks=oracle.alloc_bricks(p, w.frames[:k]))
    bk = oracle.alloc_bricks(p, w.frames)
    g_new = oracle.build_graph(p, w.frames, bricks=bk)
    assert g_new.E > g_old.E
    with _sparse_map(w, frames=w.frames[:k]) as m:
        m.bp_iterate(3)
        lam_old = m.export_messages()
        T_old = m.export_beliefs()
        for fr in w.frames[k:]:
            m.add_frame(fr.depth, fr.K, fr.T_wc)
        assert np.array_equal(m.export_bricks(), bk.mask)
        gg = m.export_graph()
        for key in ("row_ptr", "vid", "off_q", "pixel", "frame"):
            assert np.array_equal(gg[key], getattr(g_new, key)), key
        lam_start = m.export_messages()
        assert np.array_equal(lam_start.astype(np.float64), _carry_messages(g_old, lam_old, g_new, p.V))
        assert np.array_equal(m.export_beliefs(), T_old)
        m.bp_iterate(n_after)
        lam = m.export_messages()
        marg = m.marginals()
    lam_ref, T_ref = oracle.bp(p, g_new, n_after, lam=lam_start.astype(np.float64))
    assert _msg_err(lam, lam_ref) <= MSG_TOL
    assert np.max(np.abs(marg - oracle.marginals(p, T_ref))) <= MARG_TOL
