"""Pins for the oracle's learnt per-patch noise model (NEXT #4 option, DESIGN reading R25).

P:209: the measurement is distributed around the bias-predicted mean with the learnt noise;
P:225: per pixel region a 2nd-degree polynomial in depth for the bias and for sigma.

* log nu of every incidence equals scipy's Gaussian log-density at the voxel depth
  d = Z + off_q / 2^15 (a library routine, independent of the oracle's C);
* on a tree graph BP with the per-patch nu equals joint enumeration (exact for trees);
* the traversal margin follows the pixel's own sigma: L - Z = margin_k * s(Z) of its patch;
* a patch model whose patches all carry the global coefficients builds the global graph.
"""

import math

import numpy as np
import pytest
from scipy.stats import norm

import oracle
import synth
from tests.exact import enum_joint_marginals


def _coef(rng, n):
    c = np.zeros((n, 6))
    c[:, 0] = rng.uniform(-0.01, 0.01, n)
    c[:, 1] = rng.uniform(-0.01, 0.01, n)
    c[:, 2] = rng.uniform(-2e-3, 2e-3, n)
    c[:, 3] = rng.uniform(0.0, 0.01, n)
    c[:, 4] = rng.uniform(0.0, 0.005, n)
    c[:, 5] = rng.uniform(5e-4, 3e-3, n)
    return c


class _P:
    def __init__(self, sigma_min):
        self.patch = synth.PatchNoise(20, np.zeros((1, 1, 6)), sigma_min)


def test_patch_log_nu_is_the_gaussian_log_density():
    rng = np.random.default_rng(5)
    n_rays = 50
    lens = rng.integers(0, 40, n_rays)
    row_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    off_q = rng.integers(-32767, 32768, int(row_ptr[-1])).astype(np.int16)
    Z = rng.uniform(0.3, 8.0, n_rays)
    coef = _coef(rng, n_rays)
    g = oracle.Graph(row_ptr, np.zeros(len(off_q), np.int32), off_q, Z, np.zeros(n_rays, np.int32),
                     np.arange(n_rays), 0, 0, coef)
    lnu = oracle.patch_log_nu(_P(1e-4), g)
    r = np.repeat(np.arange(n_rays), lens)
    d = Z[r] + off_q.astype(np.float64) / 32768.0
    k = coef[r]
    mean = d + (k[:, 0] + k[:, 1] * d + k[:, 2] * d * d)
    s = np.maximum(k[:, 3] + k[:, 4] * d + k[:, 5] * d * d, 1e-4)
    assert np.allclose(lnu, norm.logpdf(Z[r], loc=mean, scale=s), rtol=1e-12, atol=1e-9)
    # sigma floor: a zero-sigma patch evaluates with sigma_min
    coef0 = np.zeros((n_rays, 6))
    g.coef = coef0
    lnu0 = oracle.patch_log_nu(_P(2e-3), g)
    assert np.allclose(lnu0, norm.logpdf(Z[r], loc=d, scale=2e-3), rtol=1e-12, atol=1e-9)
    # no model -> None (the LUT path)
    assert oracle.patch_log_nu(oracle.Params((4, 4, 4), 0.05, (0, 0, 0), 0.5, np.zeros((2, 2), np.float32),
                                             0, 2, -1, 1, 0.1, 3, (0, 0, 0)), g) is None


def _tree_params(n_vox, rays, rng):
    """rays: list of voxel-id lists.  A patch model with one patch per ray; incidences at random
    offsets -> (p, g, per-ray nu lists)."""
    vid, offq, row_ptr = [], [], [0]
    for vox in rays:
        vid += list(vox)
        offq += list(rng.integers(-3000, 3000, len(vox)))
        row_ptr.append(len(vid))
    pm = synth.PatchNoise(1, np.zeros((1, len(rays), 6)), 1e-4)
    pm.coeffs[0, :, 3] = rng.uniform(0.02, 0.08, len(rays))   # wide sigma: nu in a useful range
    pm.coeffs[0, :, 0] = rng.uniform(-0.02, 0.02, len(rays))
    lut = np.zeros((2, 2), np.float32)
    p = oracle.Params((n_vox, 1, 1), 0.05, (0, 0, 0), 0.2, lut, 0.0, 2.0, -1.0, 1.0, 0.1, 3.0, (0, 0, 0), pm)
    Z = rng.uniform(0.8, 1.6, len(rays))
    coef = pm.coeffs[0].copy()
    g = oracle.Graph(np.array(row_ptr, np.int64), np.array(vid, np.int32), np.array(offq, np.int16), Z,
                     np.zeros(len(rays), np.int32), np.arange(len(rays)), 0, 0, coef)
    nus = []
    for r, vox in enumerate(rays):
        e = np.arange(row_ptr[r], row_ptr[r + 1])
        d = Z[r] + np.array(offq)[e] / 32768.0
        nus.append(list(norm.pdf(Z[r], loc=d + coef[r, 0], scale=coef[r, 3])))
    return p, g, nus


@pytest.mark.parametrize("seed", range(3))
def test_patch_tree_bp_matches_joint_enumeration(seed):
    rng = np.random.default_rng(seed)
    rays = [[0, 1, 2, 3], [4, 2, 5, 6], [7, 8, 5, 9]]   # a tree: rays share v2, v5
    p, g, nus = _tree_params(10, rays, rng)
    exact = enum_joint_marginals(10, list(zip(rays, nus)), 0.2)
    lam, T = oracle.bp(p, g, 8)
    assert np.allclose(oracle.marginals(p, T), exact, atol=1e-12, rtol=0)
    # kf-average variant with one ray per keyframe equals per-ray BP (S: one message per keyframe)
    g.frame = np.arange(len(rays), dtype=np.int32)
    _, _, Tk = oracle.kf_bp(p, g, 8, len(rays))
    assert np.allclose(oracle.marginals(p, Tk), exact, atol=1e-12, rtol=0)


def test_margin_follows_the_pixel_sigma():
    """B1 with the patch model: L = Z + max(margin_min, margin_k s(Z)) with the pixel's patch s."""
    lut = np.zeros((4, 4), np.float32)
    W, H = 64, 48
    pm = synth.PatchNoise(20, np.zeros((3, 4, 6)), 1e-4)
    pm.coeffs[..., 3] = np.arange(12).reshape(3, 4) * 0.01 + 0.005   # s0 per patch
    p = oracle.Params((32, 32, 32), 0.05, (0, 0, 0), 0.5, lut, 0, 2, -0.5, 0.5, 0.001, 3.0, (0, 0, 0.0012), pm)
    T = np.array([1, 0, 0, 0.8, 0, 1, 0, 0.8, 0, 0, 1, 0.3])
    K = [60.0, 60.0, 32.0, 24.0]
    for u, v in [(0, 0), (25, 3), (47, 21), (63, 47), (32, 24)]:
        s, G0, G1, Z, L = oracle.ray_setup(p, K, T, u, v, 0.6, W)
        assert s == 0
        assert math.isclose(L - Z, 3.0 * pm.coeffs[v // 20, u // 20, 3], rel_tol=0, abs_tol=1e-12)
        # without the frame width the global sigma applies (c2 Z^2, floored at margin_min)
        s, G0, G1, Z, L = oracle.ray_setup(p, K, T, u, v, 0.6)
        assert math.isclose(L - Z, max(0.001, 3.0 * 0.0012 * Z * Z), rel_tol=0, abs_tol=1e-12)


def test_global_coefficients_reproduce_the_global_graph():
    w = synth.tiny_patch(0)
    pm = w.patch
    flat = synth.PatchNoise(pm.patch_px, np.zeros_like(pm.coeffs), pm.sigma_min)
    flat.coeffs[..., 3:6] = w.sigma_c
    pg = oracle.Params.from_workload(w)
    pg.patch = None
    pf = oracle.Params.from_workload(w)
    pf.patch = flat
    g0 = oracle.build_graph(pg, w.frames)
    g1 = oracle.build_graph(pf, w.frames)
    assert g0.E > 0 and np.array_equal(g0.row_ptr, g1.row_ptr)
    assert np.array_equal(g0.vid, g1.vid) and np.array_equal(g0.off_q, g1.off_q)
    assert g0.coef is None and g1.coef.shape == (g1.n_rays, 6)
    # the real patch model changes the sensor model (the graph too where 3 s(Z) > margin_min)
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    lnu = oracle.patch_log_nu(p, g)
    assert np.all(np.isfinite(lnu)) and lnu.max() > 0
