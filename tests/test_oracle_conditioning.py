"""Conditioning of loopy BP on the paper-shaped workloads (reading R16).

Sum-product BP on loopy graphs has no convergence guarantee.  On the single-frame
room config, a relative perturbation eps of every message after iteration 1 of the fp64
oracle reappears in the marginals at iteration 8 multiplied by ~1e4 (linear response).  No
fp32 implementation -- whose messages carry ~1e-7 relative rounding -- can therefore track
the fp64 trajectory to 1e-4 on every voxel at the config's full iteration count; the GPU
parity bars are set accordingly (tests/test_gpu_parity.py).  This pins the oracle's own
behaviour, using only the oracle.
"""

import numpy as np
import pytest

import oracle
import synth


@pytest.mark.slow
def test_loopy_trajectory_amplifies_fp32_sized_noise():
    w = synth.single_frame()
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    lam_a, _ = oracle.bp(p, g, 1)
    rng = np.random.default_rng(0)
    eps = 1e-8
    lam_b = lam_a * (1.0 + eps * rng.standard_normal(g.E))
    lam_a, Ta = oracle.bp(p, g, 7, lam=lam_a)
    lam_b, Tb = oracle.bp(p, g, 7, lam=lam_b)
    dev = np.max(np.abs(oracle.marginals(p, Ta) - oracle.marginals(p, Tb)))
    # 1e-8 in the messages -> > 1e-5 in some marginal after 8 iterations (gain > 1e3)
    assert dev > 1e3 * eps
    # and the response is linear in eps (a property of the iteration, not of rounding)
    lam_c = oracle.bp(p, g, 1)[0]
    lam_c = lam_c * (1.0 + 2 * eps * rng.standard_normal(g.E))
    _, Tc = oracle.bp(p, g, 7, lam=lam_c)
    dev2 = np.max(np.abs(oracle.marginals(p, Ta) - oracle.marginals(p, Tc)))
    assert 0.3 < dev2 / (2 * dev) < 3.0


def test_tiny_trajectory_is_well_conditioned():
    """Tiny (one frame, 32^3) damps the same noise: full-trajectory parity is meaningful there."""
    w = synth.tiny()
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    lam_a, _ = oracle.bp(p, g, 1)
    lam_b = lam_a * (1.0 + 1e-7 * np.random.default_rng(0).standard_normal(g.E))
    _, Ta = oracle.bp(p, g, w.n_iter - 1, lam=lam_a)
    _, Tb = oracle.bp(p, g, w.n_iter - 1, lam=lam_b)
    assert np.max(np.abs(oracle.marginals(p, Ta) - oracle.marginals(p, Tb))) < 1e-5
