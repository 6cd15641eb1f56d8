"""Pins for oracle B4-B7 (flooding BP, accumulation, marginals).

* single ray (a tree, P:67 / P:166): BP from zero messages equals the exact
  marginals of the joint Eq.1 after one iteration and stays there;
* tree-structured multi-ray graphs: BP equals joint enumeration after a few
  iterations (exact for trees);
* invariants: unseen voxel keeps its prior, marginals in [0,1],
  LUT-shift (nu-scale) invariance, determinism, and the
  frontal-plane sanity case.
Loopy graphs have no exact reference: parity there is oracle-vs-GPU only.
"""

import json
import math
import os

import numpy as np
import pytest

import oracle
from tests.exact import enum_joint_marginals, single_ray_marginals

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
N_COL = 64


def _lut_from_columns(lnu_cols):
    """2 identical rows; column j holds lnu_cols[j]; Z = 1.0 sits halfway between rows."""
    lut = np.full((2, N_COL), -50.0, np.float32)
    lut[:, :len(lnu_cols)] = np.asarray(lnu_cols, np.float32)
    return lut


def _offq(col):
    return int((col - 31.5) * 1024)  # exact bin centre of column col on a [-1, 1] m axis


def _graph_params(n_vox, rays, gamma):
    """rays: list of (voxel ids, nu values).  Each incidence gets its own LUT column."""
    cols = []
    vid, offq, row_ptr = [], [], [0]
    for vox, nu in rays:
        for v, n in zip(vox, nu):
            offq.append(_offq(len(cols)))
            cols.append(math.log(n))
            vid.append(v)
        row_ptr.append(len(vid))
    assert len(cols) <= N_COL
    lut = _lut_from_columns(cols)
    p = oracle.Params((n_vox, 1, 1), 0.05, (0, 0, 0), gamma, lut, 0.0, 2.0, -1.0, 1.0, 0.1, 3.0, (0, 0, 0))
    g = oracle.Graph(np.array(row_ptr, np.int64), np.array(vid, np.int32), np.array(offq, np.int16),
                     np.full(len(rays), 1.0), np.zeros(len(rays), np.int32), np.arange(len(rays)), 0, 0)
    return p, g


def test_lut_columns_are_exact():
    p, g = _graph_params(3, [([0, 1, 2], [0.3, 0.6, 2.0])], 0.5)
    for e in range(3):
        assert oracle.log_nu(p, 1.0, int(g.off_q[e])) == float(np.float32(math.log([0.3, 0.6, 2.0][e])))


def test_single_ray_golden_marginals():
    gold = json.load(open(os.path.join(GOLDEN, "single_ray_marginals.json")))
    for case in gold["cases"]:
        nu = case["nu"]
        p, g = _graph_params(len(nu), [(list(range(len(nu))), nu)], case["gamma"])
        nu32 = np.exp(p.lut[0, :len(nu)].astype(np.float64))  # what the LUT really holds
        lam, T = oracle.bp(p, g, 1)
        m = oracle.marginals(p, T)
        assert np.allclose(m, single_ray_marginals(nu32, case["gamma"]), rtol=0, atol=1e-12)
        assert np.allclose(m, case["p"], rtol=0, atol=case["tol"])


def test_single_ray_exact_after_one_iteration_and_fixed_point():
    rng = np.random.default_rng(11)
    for _ in range(40):
        N = int(rng.integers(1, 12))
        gamma = float(rng.uniform(0.02, 0.9))
        nu = np.exp(rng.uniform(-4, 3, N))
        p, g = _graph_params(N, [(list(rng.permutation(N)), nu)], gamma)
        nu32 = np.exp(p.lut[0, :N].astype(np.float64))
        lam1, T1 = oracle.bp(p, g, 1)
        lam2, T2 = oracle.bp(p, g, 2)
        exact = single_ray_marginals(nu32, gamma)
        order = g.vid
        assert np.allclose(oracle.marginals(p, T1)[order], exact, atol=1e-12, rtol=0)
        assert np.allclose(lam1, lam2, atol=1e-12, rtol=0)   # idempotent after iteration 1
        assert np.allclose(enum_joint_marginals(N, [(list(order), list(nu32))], gamma)[order], exact, atol=1e-12)


def _tree_cases():
    return [
        # two rays sharing exactly one voxel ("voxels connected by multiple rays")
        (7, [([0, 1, 2, 3], [0.2, 0.5, 3.0, 0.4]), ([4, 2, 5, 6], [0.1, 2.5, 0.3, 0.05])], 0.1),
        # three rays through one common voxel at different depths
        (9, [([0, 1, 2], [0.3, 1.5, 0.2]), ([3, 1, 4], [2.0, 0.4, 0.7]), ([5, 6, 7, 1, 8], [0.1, 0.2, 0.3, 4.0, 0.5])], 0.2),
        # chain: A-B share v2, B-C share v5
        (10, [([0, 1, 2], [0.5, 0.4, 3.0]), ([2, 3, 4, 5], [1.0, 0.2, 0.3, 2.0]), ([6, 7, 5, 8, 9], [0.1, 0.6, 1.2, 0.9, 0.1])], 0.3),
    ]


@pytest.mark.parametrize("case", range(3))
def test_tree_graphs_match_joint_enumeration(case):
    n_vox, rays, gamma = _tree_cases()[case]
    p, g = _graph_params(n_vox, rays, gamma)
    # use the float32-rounded nu the LUT actually stores
    e = 0
    rays32 = []
    for vox, nu in rays:
        nu32 = [math.exp(float(p.lut[0, e + i])) for i in range(len(nu))]
        rays32.append((vox, nu32))
        e += len(nu)
    exact = enum_joint_marginals(n_vox, rays32, gamma)
    lam, T = oracle.bp(p, g, 8)
    assert np.allclose(oracle.marginals(p, T), exact, atol=1e-12, rtol=0)


def test_unseen_voxels_keep_prior_and_marginals_in_range():
    p, g = _graph_params(10, [([0, 1, 2], [0.3, 2.0, 0.1]), ([5, 1, 6], [0.2, 0.1, 3.0])], 0.1)
    lam, T = oracle.bp(p, g, 5)
    m = oracle.marginals(p, T)
    for v in (3, 4, 7, 8, 9):
        assert abs(m[v] - 0.1) < 1e-15
    assert np.all((m >= 0) & (m <= 1))


def test_tiny_invariants_and_determinism():
    import synth
    w = synth.tiny()
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    lam_a, T_a = oracle.bp(p, g, w.n_iter)
    lam_b, T_b = oracle.bp(p, g, w.n_iter)
    assert np.array_equal(lam_a, lam_b) and np.array_equal(T_a, T_b)
    m = oracle.marginals(p, T_a)
    assert np.all((m >= 0) & (m <= 1))
    seen = np.zeros(p.V, bool)
    seen[g.vid] = True
    assert np.all(m[~seen] == 0.5)                       # gamma = 0.5
    assert np.all(np.abs(lam_a) <= 256)                  # clip (reading R9)
    # nu-scale invariance at the BP level: shift the whole table by a constant
    p2 = oracle.Params.from_workload(w)
    p2.lut = (p.lut + np.float32(7.0)).astype(np.float32)
    lam_c, T_c = oracle.bp(p2, g, w.n_iter)
    assert np.allclose(oracle.marginals(p2, T_c), m, atol=1e-6, rtol=0)


def test_frontal_plane_sanity():
    """plane at 2 m, sigma = 0.01, 0.05 m voxels, gamma = 0.1, 3 iterations:
    surface voxel > 0.9 and voxels >= 3 before it < 0.1 along the principal ray."""
    import synth
    from synth.scenes import Frame
    dims = (64, 32, 32)
    res = 0.05
    C = np.array([0.4, 0.8, 0.8])
    W, H, K = 16, 12, (20.0, 20.0, 8.0, 6.0)
    R = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])
    plane_x = 2.41
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    depth = np.full((H, W), plane_x - C[0], np.float32)  # z-depth to a frontal plane is constant
    T_wc = np.concatenate([R, C[:, None]], 1).reshape(-1)
    lut = synth.build_log_nu_lut(64, 256, 0.0, 4.0, -1.0, 1.0, (0.01, 0.0, 0.0), 0.0)
    p = oracle.Params(dims, res, (0, 0, 0), 0.1, lut, 0.0, 4.0, -1.0, 1.0, 0.1, 3.0, (0.01, 0.0, 0.0))
    g = oracle.build_graph(p, [Frame(depth, np.array(K), T_wc)])
    lam, T = oracle.bp(p, g, 3)
    m = oracle.marginals(p, T)
    r = int(np.nonzero(g.pixel == 6 * W + 8)[0][0])       # principal ray (u = cx, v = cy)
    vids = g.vid[g.row_ptr[r]:g.row_ptr[r + 1]]
    xs = vids % dims[0]
    surf = int(np.nonzero(xs == int(plane_x / res))[0][0])
    assert m[vids[surf]] > 0.9
    assert np.all(m[vids[:surf - 2]] < 0.1)
