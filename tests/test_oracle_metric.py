"""Pins of the oracle's §III.D evaluation metric (§V; SURVEY §8(f)
NEXT #2; readings R18-R21): visibility, occlusion probability, generating-surface
density and the per-pixel classification, checked against closed forms, an independent
quadrature, discretisation invariance and a brute-force ray marcher -- none of which calls
the oracle's own formula."""

import math

import numpy as np
import pytest

import oracle
import synth
from synth.scenes import Frame


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _random_ray(rng, n):
    x = rng.uniform(-8, 6, n)
    x[rng.random(n) < 0.3] = -40.0  # mostly-empty steps
    ell = rng.uniform(0.001, 0.09, n)
    return x, ell


def test_conservation_and_quadrature():
    """sum Omega_i + vis_inf = 1 (1e-9) and the quadrature of omega(s) over the ray
    equals 1 - vis_inf (1e-6), with alpha = -ln(1 - p) / res computed here from p = sigma(x)."""
    rng = np.random.default_rng(0)
    res = 0.05
    for _ in range(1000):
        n = int(rng.integers(1, 60))
        x, ell = _random_ray(rng, n)
        lvis, lom, _ = oracle.vis_profile(x, ell, res)
        vis = np.exp(lvis)
        Omega = vis[:-1] - vis[1:]
        assert abs(Omega.sum() + vis[-1] - 1.0) < 1e-9
        assert vis[0] == 1.0 and np.all(Omega >= -1e-15)
    for _ in range(50):  # quadrature at 1e-5 m (numpy, independent of the oracle recurrence)
        n = int(rng.integers(1, 20))
        x, ell = _random_ray(rng, n)
        lvis, _, _ = oracle.vis_profile(x, ell, res)
        alpha = -np.log1p(-_sigmoid(x)) / res
        h = 1e-5
        total, vis_s = 0.0, 1.0
        for a, L in zip(alpha, ell):
            m = max(1, int(round(L / h)))
            hh = L / m
            s = (np.arange(m) + 0.5) * hh
            total += np.sum(a * vis_s * np.exp(-a * s)) * hh  # midpoint rule of omega = alpha vis
            vis_s *= math.exp(-a * L)
        assert abs(total - (1.0 - math.exp(lvis[-1]))) < 1e-6
        assert abs(vis_s - math.exp(lvis[-1])) < 1e-12


def test_closed_forms():
    # one region alpha = 0.5 / m over 2 m (res = 1 m): vis at exit e^-1, Omega_0 = 1 - e^-1
    p = 1.0 - math.exp(-0.5)
    lvis, lom, best = oracle.vis_profile([math.log(p / (1 - p))], [2.0], 1.0)
    assert abs(math.exp(lvis[1]) - math.exp(-1.0)) < 1e-15
    assert best == 0 and abs(math.exp(lom[0]) - 0.5) < 1e-15  # omega at entry = alpha * vis_0
    # transparent map: vis = 1, omega = 0 everywhere, no generating surface
    lvis, lom, best = oracle.vis_profile(np.full(5, -800.0), np.full(5, 0.05), 0.05)
    assert np.all(lvis == 0.0) and np.all(lom == -np.inf) and best == -1
    # a full-side crossing multiplies visibility by (1 - p) exactly (reading R18)
    x = np.array([0.3, -1.2, 2.5])
    lvis, _, _ = oracle.vis_profile(x, np.full(3, 0.05), 0.05)
    assert np.allclose(np.exp(lvis), np.concatenate([[1.0], np.cumprod(1 - _sigmoid(x))]), rtol=1e-14)


def test_discretisation_invariance_and_monotonicity():
    """splitting every step into 4 equal sub-steps of the same alpha leaves vis_inf
    and s* unchanged; raising any p never increases a later visibility."""
    rng = np.random.default_rng(1)
    for _ in range(300):
        n = int(rng.integers(1, 30))
        x, ell = _random_ray(rng, n)
        lvis, lom, best = oracle.vis_profile(x, ell, 0.05)
        x4, ell4 = np.repeat(x, 4), np.repeat(ell / 4, 4)
        lvis4, _, best4 = oracle.vis_profile(x4, ell4, 0.05)
        assert abs(math.exp(lvis4[-1]) - math.exp(lvis[-1])) < 1e-12
        s = np.concatenate([[0.0], np.cumsum(ell)])
        s4 = np.concatenate([[0.0], np.cumsum(ell4)])
        if best >= 0:
            assert best4 == 4 * best and abs(s4[best4] - s[best]) < 1e-9
        k = int(rng.integers(0, n))
        x2 = x.copy()
        x2[k] += rng.uniform(0.1, 3.0)
        lvis2, _, _ = oracle.vis_profile(x2, ell, 0.05)
        assert np.all(lvis2[k + 1:] <= lvis[k + 1:] + 1e-15) and np.all(lvis2[:k + 1] == lvis[:k + 1])


def _box_map(dims, res, lo, hi, x_in=6.0, x_out=-8.0):
    nx, ny, nz = dims
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    c = (np.stack([x, y, z], -1) + 0.5) * res
    inside = np.all((c >= lo) & (c <= hi), -1)
    return np.where(inside, x_in, x_out).reshape(-1)


def _march(p, frame, u, v, xmap, h=2e-4):
    """Independent brute force: march the continuous ray in steps of h, alpha(s) of the voxel
    at s, vis(s) = exp(-int alpha), s* = argmax alpha(s) vis(s), s_inf = first s outside."""
    K, T = frame.K, frame.T_wc.reshape(3, 4)
    d = T[:, :3] @ np.array([(u - K[2]) / K[0], (v - K[3]) / K[1], 1.0])
    d /= np.linalg.norm(d)
    C, res, O = T[:, 3], p.geo[0], p.geo[1:4]
    dims = np.array(p.dims)
    lv, best, s_star, s = 0.0, -np.inf, -1.0, 0.0
    while True:
        c = np.floor((C + (s + 0.5 * h) * d - O) / res).astype(int)
        if np.any(c < 0) or np.any(c >= dims):
            break
        sp = math.log1p(math.exp(xmap[c[0] + dims[0] * (c[1] + dims[1] * c[2])]))
        lw = (math.log(sp / res) if sp > 0 else -np.inf) + lv
        if lw > best + 1e-12:
            best, s_star = lw, s
        lv -= (h / res) * sp
        s += h
    return s_star, s, math.exp(lv)


def test_eval_pixel_rules_and_brute_force():
    """The classification of reading R21 on a box map, and the oracle's DDA-based s*, s_inf and
    vis_inf against the brute-force marcher (within the marcher's step)."""
    w = synth.tiny()
    p = oracle.Params.from_workload(w)
    res = w.res
    xmap = _box_map(w.dims, res, (1.0, 0.2, 0.2), (1.2, 1.4, 1.4))  # slab 1.0..1.2 m along x
    fr = w.frames[0]  # camera at (0.8, 0.8, 0.8) looking along +x
    u, v = 32, 24
    depth = fr.depth.copy()
    rng = np.random.default_rng(2)
    for Zm, expect in [(0.2, 1), (0.2 + 0.05, 0), (0.9, 0)]:
        depth[v, u] = np.float32(Zm)
        f2 = Frame(depth, fr.K, fr.T_wc)
        cls, Z, s_star, s_inf, vis_inf = oracle.eval_pixel(p, f2, u, v, xmap, k_sigma=1.5)
        assert vis_inf < 0.5 and abs(s_star - 0.2) < 1e-6  # the slab face 0.2 m ahead (16-bit fixed point)
        sig = p.par[6] + p.par[7] * Z + p.par[8] * Z * Z
        assert cls == (abs(Z - s_star) <= 1.5 * sig) == expect
    # voxel-bounds mode (§III.D): accurate iff Z lies inside the argmax voxel [0.2, 0.25) m
    for Zm, expect in [(0.21, 1), (0.249, 1), (0.26, 0), (0.19, 0)]:
        depth[v, u] = np.float32(Zm)
        assert oracle.eval_pixel(p, Frame(depth, fr.K, fr.T_wc), u, v, xmap, mode=1)[0] == expect
    # empty map: accurate iff the measurement lies beyond the map boundary
    empty = np.full(p.V, -800.0)
    for Zm, expect in [(5.0, 1), (0.5, 0)]:
        depth[v, u] = np.float32(Zm)
        cls, Z, s_star, s_inf, vis_inf = oracle.eval_pixel(p, Frame(depth, fr.K, fr.T_wc), u, v, empty)
        assert vis_inf == 1.0 and s_star == -1.0 and abs(s_inf - 0.8) < 1e-6 and cls == expect
    # brute force on random pixels of a random map
    xr = rng.uniform(-9, 3, p.V)
    for _ in range(12):
        uu, vv = int(rng.integers(0, 64)), int(rng.integers(0, 48))
        depth[vv, uu] = np.float32(0.5)
        _, Z, s_star, s_inf, vis_inf = oracle.eval_pixel(p, Frame(depth, fr.K, fr.T_wc), uu, vv, xr)
        bs, binf, bvis = _march(p, fr, uu, vv, xr)
        assert abs(binf - s_inf) < 3e-4 and abs(bvis - vis_inf) < 2e-3
        assert abs(bs - s_star) < 3e-4


def test_eval_frame_counts():
    w = synth.tiny()
    p = oracle.Params.from_workload(w)
    fr = w.frames[0]
    xmap = np.full(p.V, -800.0)
    cls, nv, na = oracle.eval_frame(p, fr, xmap)
    assert nv == int(np.sum(fr.depth > 0)) and np.all(cls[fr.depth <= 0] == -1)
    assert na == int(np.sum(cls == 1))
    cls2, nv2, na2 = oracle.eval_frame(p, fr, xmap, rank=1, world=2)
    assert np.all(cls2[0::2] == -2) and np.array_equal(cls2[1::2], cls[1::2])
