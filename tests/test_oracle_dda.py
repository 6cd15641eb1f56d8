"""Pins for oracle B1 (pixel -> segment) and B2/B3 (fixed-point DDA + offsets).

B2 is pinned against an exact rational brute force (tests/exact.py): all cells
whose intersection with the segment has positive length, sorted by entry.  The
oracle's incremental walk must equal it bit for bit, t_in/t_out included (both
are correctly rounded num/den).  B1 is pinned by closed-form rays and
a pixel -> point -> pixel round trip.
"""

import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests.exact import dda_bruteforce, ONE


def _check(dims, G0, G1):
    vid, off, tin, tout = oracle.dda(dims, G0, G1)
    ref = dda_bruteforce(dims, [int(x) for x in G0], [int(x) for x in G1])
    assert [r[0] for r in ref] == vid.tolist(), (dims, G0, G1)
    assert [float(r[1]) for r in ref] == tin.tolist()
    assert [float(r[2]) for r in ref] == tout.tolist()
    return ref


def _random_segments(rng, n, dims):
    segs = []
    for i in range(n):
        kind = i % 8
        d = np.array(dims)
        if kind == 0:      # generic
            G0 = rng.integers(0, d * ONE)
            G1 = G0 + rng.integers(-5 * ONE, 5 * ONE, 3)
        elif kind == 1:    # start on a face / edge / corner
            G0 = rng.integers(0, d) * ONE
            G0[rng.integers(0, 3)] += rng.integers(0, ONE)
            G1 = G0 + rng.integers(-4 * ONE, 4 * ONE, 3)
        elif kind == 2:    # axis-aligned
            G0 = rng.integers(0, d * ONE)
            G1 = G0.copy()
            G1[rng.integers(0, 3)] += rng.integers(-5 * ONE, 5 * ONE)
        elif kind == 3:    # axis-aligned along a voxel edge
            G0 = rng.integers(0, d) * ONE
            G1 = G0.copy()
            G1[rng.integers(0, 3)] += rng.integers(-5 * ONE, 5 * ONE)
        elif kind == 4:    # 45 degrees in two axes through edges
            G0 = rng.integers(0, d) * ONE + rng.choice([0, ONE // 2], 3)
            s = rng.integers(1, 5) * ONE // rng.choice([1, 2, 4])
            G1 = G0 + np.array([s * rng.choice([-1, 1]), s * rng.choice([-1, 1]), 0])[rng.permutation(3)]
        elif kind == 5:    # body diagonal through corners
            G0 = rng.integers(0, d) * ONE
            s = rng.integers(1, 5) * ONE
            G1 = G0 + s * rng.choice([-1, 1], 3)
        elif kind == 6:    # end exactly on faces / corners
            G0 = rng.integers(0, d * ONE)
            G1 = rng.integers(0, d) * ONE
            G1[rng.integers(0, 3)] += rng.integers(0, ONE)
        else:              # leaves the grid (margin past the far face)
            G0 = rng.integers(0, d * ONE)
            G1 = G0 + rng.integers(-12 * ONE, 12 * ONE, 3)
        if np.all(G1 == G0):
            G1 = G0 + np.array([1, 0, 0])
        segs.append((G0.astype(np.int64), G1.astype(np.int64)))
    return segs


def test_dda_matches_rational_bruteforce_random():
    rng = np.random.default_rng(1234)
    n = 0
    for dims in ([16, 16, 16], [5, 9, 7], [12, 3, 16], [1, 1, 16]):
        for G0, G1 in _random_segments(rng, 2600, dims):
            _check(dims, G0, G1)
            n += 1
    assert n >= 10_000


@pytest.mark.parametrize("G0,G1,expect", [
    # principal ray of Tiny: along +x exactly on the y=16 / z=16 voxel edges (half-open -> upper cells)
    ([16 * ONE, 16 * ONE, 16 * ONE], [20 * ONE + 123, 16 * ONE, 16 * ONE], [(16, 16, 16), (17, 16, 16), (18, 16, 16), (19, 16, 16), (20, 16, 16)]),
    # same, moving -x from a face: start cell is the one below the face
    ([16 * ONE, 16 * ONE, 16 * ONE], [14 * ONE, 16 * ONE, 16 * ONE], [(15, 16, 16), (14, 16, 16)]),
    # body diagonal through corners: corner-touching cells have zero length
    ([2 * ONE, 2 * ONE, 2 * ONE], [5 * ONE, 5 * ONE, 5 * ONE], [(2, 2, 2), (3, 3, 3), (4, 4, 4)]),
    # start on the low grid face moving out: nothing inside
    ([0, 3 * ONE, 3 * ONE], [-2 * ONE, 3 * ONE + 5, 3 * ONE], []),
])
def test_dda_special_cases(G0, G1, expect):
    dims = [32, 32, 32]
    vid, *_ = oracle.dda(dims, np.array(G0), np.array(G1))
    got = [(v % 32, (v // 32) % 32, v // 1024) for v in vid.tolist()]
    assert got == expect
    _check(dims, np.array(G0), np.array(G1))


def test_dda_axis_aligned_from_voxel_centre():
    """+x ray from a voxel centre, s_max = 4 voxels -> 5 cells, first/last half."""
    dims = [16, 16, 16]
    G0 = np.array([3 * ONE + ONE // 2, 5 * ONE + ONE // 2, 5 * ONE + ONE // 2])
    G1 = G0 + np.array([4 * ONE, 0, 0])
    vid, _, tin, tout = oracle.dda(dims, G0, G1)
    assert (vid % 16).tolist() == [3, 4, 5, 6, 7]
    assert np.allclose(tout - tin, [0.125, 0.25, 0.25, 0.25, 0.125], rtol=0, atol=0)


def test_dda_length_conservation():
    """the traversed spans tile [0, t_exit] without gaps (t_out_k == t_in_{k+1})."""
    rng = np.random.default_rng(7)
    dims = [16, 16, 16]
    for G0, G1 in _random_segments(rng, 400, dims):
        vid, _, tin, tout = oracle.dda(dims, G0, G1)
        if len(vid) == 0:
            continue
        assert tin[0] == 0.0
        assert np.all(tout[:-1] == tin[1:])
        # exit parameter of the segment from the grid box, exactly
        t_exit = Fraction(1)
        for k in range(3):
            d = int(G1[k] - G0[k])
            if d > 0:
                t_exit = min(t_exit, Fraction(dims[k] * ONE - int(G0[k]), d))
            elif d < 0:
                t_exit = min(t_exit, Fraction(-int(G0[k]), d))
        assert tout[-1] == float(t_exit)


def test_dda_offsets_are_span_midpoints():
    """B3: off_q = llrint((0.5 (t_in + t_out) L - Z) * 32768), clamped to +-32767."""
    dims = [16, 16, 16]
    G0 = np.array([1 * ONE + 100, 2 * ONE + 7, 3 * ONE + 99])
    G1 = np.array([13 * ONE + 5, 9 * ONE + 1, 4 * ONE + 3])
    Z, L = 0.31, 0.42
    vid, off, tin, tout = oracle.dda(dims, G0, G1, Z, L)
    ref = [int(np.clip(np.rint((0.5 * (a + b) * L - Z) * 32768), -32767, 32767)) for a, b in zip(tin, tout)]
    assert off.tolist() == ref
    # far-in-front offsets clamp to -1 m
    vid, off, *_ = oracle.dda(dims, G0, G1, 5.0, 6.0)
    assert off.min() == -32767


def _params(dims=(32, 32, 32), res=0.05):
    lut = np.zeros((4, 4), np.float32)
    return oracle.Params(dims, res, (0, 0, 0), 0.5, lut, 0, 2, -0.2, 0.2, 0.1, 3.0, (0, 0, 0.0012))


def test_ray_setup_closed_forms():
    """principal ray has range z; u = cx + fx has range z*sqrt(2)."""
    p = _params()
    T = np.array([1, 0, 0, 0.8, 0, 1, 0, 0.8, 0, 0, 1, 0.3])  # identity rotation, camera at (0.8,0.8,0.3)
    K = [60.0, 60.0, 32.0, 24.0]
    s, G0, G1, Z, L = oracle.ray_setup(p, K, T, 32, 24, 1.0)
    assert s == 0 and Z == 1.0 and L == 1.1
    assert G0.tolist() == [16 * ONE, 16 * ONE, 6 * ONE]
    assert G1[0] == G0[0] and G1[1] == G0[1] and G1[2] == round((0.3 + 1.1) / 0.05 * ONE)
    s, G0, G1, Z, L = oracle.ray_setup(p, K, T, 92, 24, 0.5)
    assert s == 0 and abs(Z - 0.5 * math.sqrt(2.0)) < 1e-15
    d = (G1 - G0).astype(np.float64)
    assert abs(d[0] - d[2]) <= 2 and d[1] == 0   # direction (1,0,1)/sqrt(2)
    # invalid and dropped pixels
    assert oracle.ray_setup(p, K, T, 32, 24, 0.0)[0] == 1
    assert oracle.ray_setup(p, K, T, 32, 24, float("nan"))[0] == 1
    assert oracle.ray_setup(p, K, T, 32, 24, 5.0)[0] == 2   # measured point beyond the grid


def test_ray_setup_round_trip():
    """the segment end re-projects onto its pixel (within the 2^-16 voxel quantisation)."""
    rng = np.random.default_rng(3)
    p = _params((64, 64, 64), 0.05)
    K = [525.0, 525.0, 319.5, 239.5]
    for _ in range(200):
        a = rng.normal(size=3)
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        if np.linalg.det(q) < 0:
            q[:, 0] = -q[:, 0]
        C = np.array([1.6, 1.6, 1.6]) + rng.uniform(-0.2, 0.2, 3)
        T = np.concatenate([q, C[:, None]], axis=1).reshape(-1)
        u, v = int(rng.integers(0, 640)), int(rng.integers(0, 480))
        z = float(rng.uniform(0.3, 1.0))
        s, G0, G1, Z, L = oracle.ray_setup(p, K, T, u, v, np.float32(z))
        assert s == 0
        X = G1 / ONE * 0.05  # end point (world), range L along the ray
        Xc = q.T @ (X - C)
        uu = K[0] * Xc[0] / Xc[2] + K[2]
        vv = K[1] * Xc[1] / Xc[2] + K[3]
        assert abs(uu - u) < 1e-3 and abs(vv - v) < 1e-3
        assert abs(np.linalg.norm(X - C) - L) < 1e-5
        del a
