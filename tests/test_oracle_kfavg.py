"""Pins of the oracle's keyframe-average variant ("all rays
going through a voxel from a single keyframe send the same average message"; DESIGN.md reading
R22): SPEC's worked examples for accumulate_outgoing and incoming_product, permutation
invariance, and the reduction to the per-ray iteration (B5) when a keyframe has at most one ray
per voxel -- none of which re-types the oracle's formulas."""

import math

import numpy as np

import oracle
import synth


def _graph(rays, frames):
    """Hand-made CSR: rays = list of voxel-id lists, frames = keyframe of each ray."""
    row_ptr = np.concatenate([[0], np.cumsum([len(r) for r in rays])]).astype(np.int64)
    vid = np.concatenate([np.asarray(r, np.int32) for r in rays]) if rays else np.zeros(0, np.int32)
    E = len(vid)
    return oracle.Graph(row_ptr, vid, np.zeros(E, np.int16), np.full(len(rays), 1.0),
                        np.asarray(frames, np.int32), np.arange(len(rays), dtype=np.int64), 0, 0)


def test_accumulate_outgoing_spec_examples():
    """SPEC accumulate_outgoing: two accumulations (0.3, 0.7) and (0.5, 0.5) -> average
    (0.4, 0.6); zero accumulations -> the uniform pair (log-odds 0)."""
    g = _graph([[0, 1], [0]], [0, 0])
    lam = np.array([math.log(0.7 / 0.3), 2.0, 0.0])  # ray 0: v0 (0.3, 0.7), v1 anything; ray 1: v0 (0.5, 0.5)
    lbar = oracle.kf_average(g, lam, F=1, V=3)
    assert abs(lbar[0, 0] - math.log(0.6 / 0.4)) < 1e-12
    assert abs(lbar[0, 1] - 2.0) < 1e-12   # a single message averages to itself
    assert lbar[0, 2] == 0.0                # no ray of the keyframe reaches v2


def test_average_permutation_and_identical_messages():
    """SPEC: the average does not depend on the accumulation order; identical messages average
    to themselves; keyframes never mix."""
    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(1, 40))
        lam = rng.uniform(-30, 30, n)
        frames = rng.integers(0, 3, n)
        g = _graph([[0]] * n, frames)
        a = oracle.kf_average(g, lam, F=3, V=1)
        perm = rng.permutation(n)
        b = oracle.kf_average(_graph([[0]] * n, frames[perm]), lam[perm], F=3, V=1)
        assert np.allclose(a, b, rtol=0, atol=1e-12)
        for f in range(3):
            if not np.any(frames == f):
                assert a[f, 0] == 0.0
        x = float(rng.uniform(-40, 40))
        c = oracle.kf_average(_graph([[0]] * n, np.zeros(n)), np.full(n, x), F=1, V=1)
        assert abs(c[0, 0] - x) < 1e-9


def test_incoming_product_spec_example():
    """SPEC incoming_product: with gamma = 0.1 and one OTHER keyframe whose average into v is
    (0.2, 0.8), the incoming pair is normalize(0.9 * 0.2, 0.1 * 0.8) = (0.6923.., 0.3076..).
    The ray's own keyframe average is excluded whatever it holds; the messages are then B5's
    (pinned by enumeration) for that cavity."""
    w = synth.tiny()
    p = oracle.Params.from_workload(w)
    p.L0 = math.log(0.1 / 0.9)  # gamma = 0.1 (SPEC's example)
    g = _graph([[0, 1]], [0])
    g.off_q = np.array([-200, 300], np.int16)
    lbar = np.zeros((2, p.V))
    lbar[1, 0] = math.log(0.8 / 0.2)   # keyframe 1 -> v0: (0.2, 0.8)
    lbar[0, 0] = 5.0                   # the ray's own keyframe: must be excluded
    lbar[0, 1] = -3.0
    lam = oracle.kf_pass(p, g, lbar)
    c = np.array([math.log((0.1 * 0.8) / (0.9 * 0.2)), math.log(0.1 / 0.9)])
    assert abs(1 / (1 + math.exp(-c[0])) - 0.3076923) < 1e-7
    lnu = np.array([oracle.log_nu(p, 1.0, -200), oracle.log_nu(p, 1.0, 300)])
    lpos, lneg = oracle.ray_messages(c, lnu)
    assert np.allclose(lam, np.clip(lpos - lneg, -256, 256), rtol=0, atol=1e-12)


def test_one_ray_per_keyframe_equals_per_ray_bp():
    """When no keyframe has two rays through one voxel, the keyframe average of (f, v) IS the
    one ray's message and excluding the keyframe excludes exactly that message: the variant
    must reproduce the per-ray iteration (B5, pinned on trees) on a loopy graph."""
    w = synth.tiny()
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    n = 150
    sub = oracle.Graph(g.row_ptr[:n + 1].copy(), g.vid[:g.row_ptr[n]].copy(), g.off_q[:g.row_ptr[n]].copy(),
                       g.Z[:n].copy(), np.arange(n, dtype=np.int32), g.pixel[:n].copy(), 0, 0)
    for it in (1, 3, 8):
        lam_ref, T_ref = oracle.bp(p, sub, it)
        lam, lbar, T = oracle.kf_bp(p, sub, it, F=n)
        assert np.max(np.abs(lam - lam_ref)) < 1e-8
        assert np.max(np.abs(T - T_ref)) < 1e-8


def test_first_iteration_and_unseen_voxels():
    """From zero messages both variants see the prior everywhere, so iteration 1's messages
    coincide; voxels no ray reaches keep T = 0 (the prior); marginals lie in [0, 1]."""
    w = synth.tiny()
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    lam_ref, _ = oracle.bp(p, g, 1)
    lam, lbar, T = oracle.kf_bp(p, g, 1, F=len(w.frames))
    assert np.array_equal(lam, lam_ref)
    seen = np.zeros(p.V, bool)
    seen[g.vid] = True
    lam5, lbar5, T5 = oracle.kf_bp(p, g, 5, F=len(w.frames))
    assert np.all(T5[~seen] == 0.0) and np.all(lbar5[:, ~seen] == 0.0)
    m = oracle.marginals(p, T5)
    assert np.all((m >= 0) & (m <= 1))
    # several rays of the one keyframe share voxels: the variant is not the per-ray iteration
    lam_ref5, _ = oracle.bp(p, g, 5)
    assert np.max(np.abs(lam5 - lam_ref5)) > 1e-3
