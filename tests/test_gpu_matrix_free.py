"""Matrix-free iteration (the paper re-traces every keyframe each pass,
P:200): only the messages and the tile runs persist, the rays are walked again per chunk of
frames.  The walk is the same integer DDA and the reductions are exact integer sums, so the
results must be BIT-IDENTICAL to the stored-graph path (itself parity-tested against the oracle
in test_gpu_parity.py) -- in the per-ray, keyframe-average and sparse-brick modes."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2006_03512_b200 as pkg  # noqa: E402

pytestmark = pytest.mark.gpu


def _run(w, n_iter, mf=0, kf=False, bricks=0, frames=None):
    m = pkg.MRFMap.from_workload(w)
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    if mf:
        m.set_matrix_free(mf)
    if kf:
        m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
    if bricks:
        m.set_sparse_bricks(bricks)
    for fr in (w.frames if frames is None else frames):
        m.add_frame(fr.depth, fr.K, fr.T_wc)
    with m:
        m.bp_iterate(n_iter)
        sizes = m.graph_sizes(active=not mf)
        if kf:  # keyframe averages: the state (with matrix-free walks no messages are kept)
            lam = np.stack([m.export_keyframe_average(f) for f in range(len(frames or w.frames))])
        else:
            lam = m.export_messages()
        return lam, m.export_beliefs(), m.marginals(), sizes


@pytest.mark.parametrize("mf", [1, 2, 3])
def test_matrix_free_bit_identical(mf):
    w = synth.tiny_frames(n_frames=4)
    lam0, T0, m0, s0 = _run(w, 6)
    lam1, T1, m1, s1 = _run(w, 6, mf=mf)
    assert np.array_equal(lam0, lam1) and np.array_equal(T0, T1) and np.array_equal(m0, m1)
    assert s1["E"] == s0["E"] and s1["n_rays"] == s0["n_rays"]


def test_matrix_free_frame1_and_modes():
    w = synth.single_frame()
    a = _run(w, 3)
    b = _run(w, 3, mf=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    t = synth.tiny_frames(n_frames=4)
    for kw in (dict(kf=True), dict(bricks=8), dict(kf=True, bricks=8)):
        x = _run(t, 4, **kw)
        y = _run(t, 4, mf=2, **kw)
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1]), kw


def test_matrix_free_warm_start_and_rules():
    """Frames added after iterations (warm start) are walked and counted like the others; the
    stored-graph exports are refused."""
    w = synth.tiny_frames(n_frames=4)
    res = []
    for mf in (0, 2):
        m = pkg.MRFMap.from_workload(w)
        m.set_stream(torch.cuda.current_stream().cuda_stream)
        if mf:
            m.set_matrix_free(mf)
        with m:
            for fr in w.frames[:3]:
                m.add_frame(fr.depth, fr.K, fr.T_wc)
            m.bp_iterate(3)
            m.add_frame(w.frames[3].depth, w.frames[3].K, w.frames[3].T_wc)
            m.bp_iterate(2)
            res.append((m.export_messages(), m.export_beliefs()))
            if mf:
                with pytest.raises(pkg.MrfError) as e:
                    m.export_graph()
                assert e.value.status == 6
                with pytest.raises(pkg.MrfError):
                    m.export_rays(np.zeros(1, np.int32), np.zeros(1, np.int64))
                assert m.graph_sizes()["n_active"] == -1
                with pytest.raises(pkg.MrfError):
                    m.set_matrix_free(1)  # frames already added
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


def _oracle_leg(w, n_iter, mf):
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    lam_ref, T_ref = oracle.bp(p, g, n_iter)
    lam, _, marg, sizes = _run(w, n_iter, mf=mf)
    assert sizes["E"] == g.E and sizes["n_rays"] == g.n_rays
    rel = np.abs(lam.astype(np.float64) - lam_ref) / np.maximum(1.0, np.abs(lam_ref))
    assert rel.max() <= 1e-3, f"max rel msg err {rel.max():.3e}"
    d = np.abs(marg - oracle.marginals(p, T_ref))
    assert d.max() <= 1e-4, f"max marginal err {d.max():.3e}"


@pytest.mark.parametrize("mf,n_iter", [(1, 1), (2, 3), (3, 10)])
def test_matrix_free_matches_oracle_tiny_frames(mf, n_iter):
    """Matrix-free against the fp64 oracle directly (not only against the stored graph): the
    tiny scene seen from 4 keyframes, full trajectory."""
    _oracle_leg(synth.tiny_frames(n_frames=4), n_iter, mf)


def test_matrix_free_matches_oracle_frame1():
    """The single-frame room (26 M incidences), full trajectory over 2 iterations (where the
    loopy graph is still well conditioned)."""
    _oracle_leg(synth.single_frame(), 2, 1)


@pytest.mark.parametrize("mf", [1, 3])
def test_keyframe_average_matrix_free_storage_and_parity(mf):
    """The paper's own storage (keyframes re-traced every pass, "an auxiliary buffer that
    stores the average outgoing message"): keyframe averages with fused matrix-free walks keep no
    per-incidence messages -- only a one-chunk scratch between K5 and K6' -- and give keyframe
    averages and beliefs bit-identical to the stored keyframe-average path, which matches the
    oracle's kf_bp; warm start (a keyframe added after iterating) included."""
    w = synth.tiny_frames(n_frames=4)
    F = len(w.frames)
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    _, lbar_ref, T_ref = oracle.kf_bp(p, g, 5, F=F)
    outs = []
    for m_f in (0, mf):
        m = pkg.MRFMap.from_workload(w)
        m.set_stream(torch.cuda.current_stream().cuda_stream)
        m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
        if m_f:
            m.set_matrix_free(m_f)
        with m:
            for fr in w.frames:
                m.add_frame(fr.depth, fr.K, fr.T_wc)
            m.bp_iterate(5)
            lbar = np.stack([m.export_keyframe_average(f) for f in range(F)])
            outs.append((lbar, m.export_beliefs(), m.marginals()))
            if m_f:
                with pytest.raises(pkg.MrfError) as e:
                    m.export_messages()
                assert e.value.status == 6
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    err = np.abs(outs[1][0].astype(np.float64).reshape(-1) - lbar_ref.reshape(-1)) / np.maximum(1.0, np.abs(lbar_ref.reshape(-1)))
    assert err.max() <= 1e-3
    assert np.max(np.abs(outs[1][2] - oracle.marginals(p, T_ref))) <= 1e-4
    # warm start: 3 keyframes, iterate, add the 4th, iterate -- equal to the stored path
    res = []
    for m_f in (0, mf):
        m = pkg.MRFMap.from_workload(w)
        m.set_stream(torch.cuda.current_stream().cuda_stream)
        m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
        if m_f:
            m.set_matrix_free(m_f)
        with m:
            for fr in w.frames[:3]:
                m.add_frame(fr.depth, fr.K, fr.T_wc)
            m.bp_iterate(3)
            m.add_frame(w.frames[3].depth, w.frames[3].K, w.frames[3].T_wc)
            m.bp_iterate(2)
            res.append((np.stack([m.export_keyframe_average(f) for f in range(F)]), m.export_beliefs()))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
