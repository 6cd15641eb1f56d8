"""GPU parity of the keyframe-average message variant (PAPER.md P:200,
DESIGN.md reading R22) against the oracle's kf_* functions, through the C ABI.

Bars: per-incidence messages and keyframe averages |d| <= 1e-3 max(1, |x|), marginals within
1e-4 -- the per-ray path's bars (the averages are means of the messages)."""

import dataclasses

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2006_03512_b200 as pkg  # noqa: E402

pytestmark = pytest.mark.gpu

MSG_TOL = 1e-3
MARG_TOL = 1e-4
LBAR_TOL = 1e-3


def _kf_map(w):
    m = pkg.MRFMap.from_workload(w)
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
    for fr in w.frames:
        m.add_frame(fr.depth, fr.K, fr.T_wc)
    return m


def _msg_err(lam, ref):
    return float(np.max(np.abs(lam.astype(np.float64) - ref) / np.maximum(1.0, np.abs(ref)))) if len(ref) else 0.0


def _lbar_err(lbar, ref):
    return _msg_err(lbar.reshape(-1), ref.reshape(-1))


@pytest.fixture(scope="module")
def tf4():
    return synth.tiny_frames(n_frames=4)


@pytest.mark.parametrize("n_iter", [1, 2, 5, 10])
def test_kfavg_trajectory(tf4, n_iter):
    """Full trajectory from zero messages on four overlapping keyframes."""
    w = tf4
    F = len(w.frames)
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    lam_ref, lbar_ref, T_ref = oracle.kf_bp(p, g, n_iter, F=F)
    with _kf_map(w) as m:
        m.bp_iterate(n_iter)
        lam = m.export_messages()
        marg = m.marginals()
        lbar = np.stack([m.export_keyframe_average(f) for f in range(F)])
    assert _msg_err(lam, lam_ref) <= MSG_TOL
    assert _lbar_err(lbar, lbar_ref) <= LBAR_TOL
    assert np.max(np.abs(marg - oracle.marginals(p, T_ref))) <= MARG_TOL
    if n_iter >= 2:  # the variant is really in effect (not the per-ray iteration)
        lam_ray, _ = oracle.bp(p, g, n_iter)
        assert np.max(np.abs(lam_ray - lam_ref)) > 1e-2


def test_kfavg_one_step_from_gpu_state(tf4):
    """T3-style: from the GPU's own keyframe averages after 6 iterations, one more iteration on
    each side (oracle kf_pass + kf_average from the exported averages)."""
    w = tf4
    F = len(w.frames)
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    with _kf_map(w) as m:
        m.bp_iterate(6)
        lbar0 = np.stack([m.export_keyframe_average(f) for f in range(F)]).astype(np.float64)
        m.bp_iterate(1)
        lam = m.export_messages()
        lbar1 = np.stack([m.export_keyframe_average(f) for f in range(F)])
        marg = m.marginals()
    lam_ref = oracle.kf_pass(p, g, lbar0)
    lbar_ref = oracle.kf_average(g, lam_ref, F, p.V)
    assert _msg_err(lam, lam_ref) <= MSG_TOL
    assert _lbar_err(lbar1, lbar_ref) <= LBAR_TOL
    assert np.max(np.abs(marg - oracle.marginals(p, oracle.kf_beliefs(lbar_ref)))) <= MARG_TOL


def test_kfavg_single_keyframe_rays_equal_per_ray_path():
    """Frames of one valid pixel each: no keyframe has two rays through a voxel, so the variant
    must give the per-ray path's messages (the oracle pin of the same reduction, on the GPU)."""
    w = synth.tiny_frames(n_frames=6)
    frames = []
    for k, fr in enumerate(w.frames):
        d = np.zeros_like(fr.depth)
        v, u = 10 + 5 * k, 12 + 7 * k
        d[v, u] = fr.depth[v, u] if fr.depth[v, u] > 0 else 1.0
        frames.append(synth.Frame(d, fr.K, fr.T_wc))
    w1 = dataclasses.replace(w, frames=frames)
    with _kf_map(w1) as a:
        a.bp_iterate(5)
        lam_a, marg_a = a.export_messages(), a.marginals()
    m = pkg.MRFMap.from_workload(w1)
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    for fr in frames:
        m.add_frame(fr.depth, fr.K, fr.T_wc)
    with m:
        m.bp_iterate(5)
        lam_b, marg_b = m.export_messages(), m.marginals()
    assert len(lam_a) == len(lam_b) > 0
    assert np.max(np.abs(lam_a - lam_b)) <= 1e-5 * max(1.0, float(np.max(np.abs(lam_b))))
    assert np.max(np.abs(marg_a - marg_b)) <= 1e-6


def test_kfavg_mode_errors(tf4):
    w = tf4
    m = pkg.MRFMap.from_workload(w)
    with m:
        m.add_frame(w.frames[0].depth, w.frames[0].K, w.frames[0].T_wc)
        with pytest.raises(pkg.MrfError) as e:
            m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)  # frames already added
        assert e.value.status == 6
        with pytest.raises(pkg.MrfError):
            m.export_keyframe_average(0)  # per-ray mode
        with pytest.raises(pkg.MrfError):
            m.set_message_mode(7)
    with _kf_map(w) as m:
        with pytest.raises(pkg.MrfError):
            m.export_keyframe_average(len(w.frames))
        m.bp_iterate(2)
        m.reset()  # back to no frames: averages start uniform again
        m.add_frame(w.frames[1].depth, w.frames[1].K, w.frames[1].T_wc)
        assert np.all(m.export_keyframe_average(0) == 0.0)


def test_kfavg_import_and_warm_start(tf4):
    """mrf_import_messages in keyframe-average mode rebuilds the averages from the messages
    (the same K6' + finalize as an iteration); a frame added after iterations starts uniform
    and the earlier keyframes keep their averages (warm start, as in the per-ray mode)."""
    w = tf4
    F = len(w.frames)
    with _kf_map(w) as m:
        m.bp_iterate(4)
        lam = m.export_messages()
        lbar = np.stack([m.export_keyframe_average(f) for f in range(F)])
        marg = m.marginals()
        m.import_messages(lam)
        lbar2 = np.stack([m.export_keyframe_average(f) for f in range(F)])
        assert np.array_equal(lbar, lbar2)
        assert np.array_equal(marg, m.marginals())
    p = oracle.Params.from_workload(w)
    with _kf_map(dataclasses.replace(w, frames=w.frames[:3])) as m:
        m.bp_iterate(3)
        lbar3 = np.stack([m.export_keyframe_average(f) for f in range(3)])
        fr = w.frames[3]
        m.add_frame(fr.depth, fr.K, fr.T_wc)
        assert np.all(m.export_keyframe_average(3) == 0.0)
        assert np.array_equal(np.stack([m.export_keyframe_average(f) for f in range(3)]), lbar3)
        m.bp_iterate(2)
        lam = m.export_messages()
        marg = m.marginals()
    g = oracle.build_graph(p, w.frames)
    lb0 = np.zeros((F, p.V))
    lb0[:3] = lbar3.astype(np.float64)
    lam_ref, lbar_ref, T_ref = oracle.kf_bp(p, g, 2, F=F, lbar=lb0)
    assert _msg_err(lam, lam_ref) <= MSG_TOL
    assert np.max(np.abs(marg - oracle.marginals(p, T_ref))) <= MARG_TOL


@pytest.mark.parametrize("mf", [0, 1])
def test_kfavg_deterministic(tf4, mf):
    """The keyframe averages are exact integer sums (counts, min |q|, fixed-point small
    probabilities): byte-identical averages and beliefs across runs, every iteration, with the
    stored graph and with matrix-free walks (chunked, no per-incidence messages)."""
    F = len(tf4.frames)
    runs = []
    for _ in range(3):
        m = pkg.MRFMap.from_workload(tf4)
        m.set_stream(torch.cuda.current_stream().cuda_stream)
        m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
        if mf:
            m.set_matrix_free(mf)
        out = []
        with m:
            for fr in tf4.frames:
                m.add_frame(fr.depth, fr.K, fr.T_wc)
            for _ in range(4):
                m.bp_iterate(1)
                out.append((np.stack([m.export_keyframe_average(f) for f in range(F)]), m.export_beliefs()))
        runs.append(out)
    for other in runs[1:]:
        for (a, ta), (b, tb) in zip(runs[0], other):
            assert np.array_equal(a, b) and np.array_equal(ta, tb)


@pytest.mark.parametrize("scene", ["tiny4", "room3"])
def test_kfavg_block_passes_bit_identical(scene, monkeypatch):
    """The keyframe-average sums over pixel blocks (K6b passes: MRF_K6=block + MRF_KF_BLOCK=1, an
    option -- slower than the runs at frames30) against the passes over (frame, tile) runs (MRF_K6=tile):
    keyframe averages, messages and beliefs bit-identical (integer counts, minima and fixed-point
    sums in any order), with a frame added after iterating (warm start)."""
    w = synth.tiny_frames(n_frames=4) if scene == "tiny4" else synth.frames30(n_frames=3)
    monkeypatch.setenv("MRF_KF_BLOCK", "1")
    outs = {}
    for k6 in ("tile", "block"):
        monkeypatch.setenv("MRF_K6", k6)
        m = pkg.MRFMap.from_workload(w)
        m.set_stream(torch.cuda.current_stream().cuda_stream)
        m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
        with m:
            for fr in w.frames[:-1]:
                m.add_frame(fr.depth, fr.K, fr.T_wc)
            m.bp_iterate(2)
            fr = w.frames[-1]
            m.add_frame(fr.depth, fr.K, fr.T_wc)
            m.bp_iterate(2)
            assert m.k6_path() == k6
            outs[k6] = [m.export_keyframe_average(f) for f in range(len(w.frames))] + [m.export_messages(),
                                                                                      m.export_beliefs()]
    for a, b in zip(outs["tile"], outs["block"]):
        assert np.array_equal(a, b)
