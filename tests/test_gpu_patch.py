"""GPU parity of the learnt per-patch sensor model (NEXT #4 option, DESIGN reading R25;
mrf_set_patch_noise) against the fp64 oracle (oracle.patch_log_nu + the same B1-B7).

Bars as for the global model (tests/test_gpu_parity.py): ray->voxel lists and offsets bit-exact
(the margins follow each pixel's patch sigma in fp64); messages within 1e-3 relative, marginals
within 1e-4 on the well-conditioned tiny config and after one step; the loopy frame1 trajectory
under the count rule of tests/traj.py.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2006_03512_b200 as pkg  # noqa: E402
from tests import traj  # noqa: E402
from tests.test_gpu_parity import _assert_graph_equal, _assert_msgs_close, _gpu_map, MARG_TOL  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tinyp():
    return synth.tiny_patch()


@pytest.fixture(scope="module")
def frame1p():
    return synth.frame1_patch()


@pytest.mark.parametrize("n_iter", [1, 3, 10])
def test_tiny_patch_graph_and_bp(tinyp, n_iter):
    p = oracle.Params.from_workload(tinyp)
    g = oracle.build_graph(p, tinyp.frames)
    lam_ref, T_ref = oracle.bp(p, g, n_iter)
    with _gpu_map(tinyp) as m:
        _assert_graph_equal(m.export_graph(), g)
        m.bp_iterate(n_iter)
        _assert_msgs_close(m.export_messages(), lam_ref)
        assert np.max(np.abs(m.marginals() - oracle.marginals(p, T_ref))) <= MARG_TOL


def test_patch_model_differs_from_global(tinyp):
    """The model is really in use: the global table's graph and messages differ from it."""
    w = synth.tiny_patch()
    w.patch = None
    with _gpu_map(tinyp) as m, _gpu_map(w) as m0:
        m.bp_iterate(1)
        m0.bp_iterate(1)
        g1, g0 = m.export_graph(), m0.export_graph()
        same_graph = g1["vid"].shape == g0["vid"].shape and np.array_equal(g1["vid"], g0["vid"])
        assert not same_graph or np.max(np.abs(m.export_messages() - m0.export_messages())) > 1e-2


def test_frame1_patch_graph_one_step_and_count_rule(frame1p):
    w = frame1p
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    ref = traj.reference_trajectory(p, g, (3, w.n_iter))
    noisy = traj.noisy_trajectories(p, g, (3, w.n_iter), seeds=(1, 2, 3, 4))
    lam_ref, T_ref = oracle.bp(p, g, 1)
    gpu = {}
    with _gpu_map(w) as m:
        _assert_graph_equal(m.export_graph(), g)
        m.bp_iterate(1)
        _assert_msgs_close(m.export_messages(), lam_ref)
        m.bp_iterate(2)
        gpu[3] = m.marginals()
        # one step (T3) from the GPU's own state at iteration 3
        lam0 = m.export_messages()
        m.import_messages(lam0)
        m.bp_iterate(1)
        lam = lam0.astype(np.float64)
        oracle.ray_pass(p, g, oracle.accumulate(p, g, lam), lam)
        _assert_msgs_close(m.export_messages(), lam)
        m.bp_iterate(w.n_iter - 4)
        gpu[w.n_iter] = m.marginals()
    for n in (3, w.n_iter):
        st = traj.dev_stats(gpu[n], ref[n])
        ns = [traj.dev_stats(nz[n], ref[n]) for nz in noisy]
        print(f"frame1_patch n={n}: gpu {st}, noisy oracle {ns}")
        assert st["p9999"] <= MARG_TOL, st
        assert st["over"] <= traj.count_bar([x["over"] for x in ns]), (st, ns)


@pytest.mark.parametrize("mode", ["kf", "sparse", "mf", "kfmf"])
def test_tiny_patch_modes(tinyp, mode):
    """The per-patch model in the keyframe-average, sparse-brick and matrix-free modes."""
    w = synth.tiny_frames()
    w.patch = synth.patch_noise_model(64, 48, 0, 20, w.sigma_c)
    p = oracle.Params.from_workload(w)
    bk = oracle.alloc_bricks(p, w.frames) if mode == "sparse" else None
    g = oracle.build_graph(p, w.frames, bricks=bk)
    m = pkg.MRFMap.from_workload(w)
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    if "kf" in mode:
        m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
    if "mf" in mode:
        m.set_matrix_free(2)
    if mode == "sparse":
        m.set_sparse_bricks(8)
    with m:
        for fr in w.frames:
            m.add_frame(fr.depth, fr.K, fr.T_wc)
        m.bp_iterate(5)
        marg = m.marginals()
        if mode == "sparse":
            assert np.array_equal(m.export_bricks() != 0, bk.mask != 0)
            _assert_graph_equal(m.export_graph(), g)
    if "kf" in mode:
        _, _, T_ref = oracle.kf_bp(p, g, 5, F=len(w.frames))
    else:
        _, T_ref = oracle.bp(p, g, 5)
    assert np.max(np.abs(marg - oracle.marginals(p, T_ref))) <= MARG_TOL
    if "mf" in mode:  # bit-identical to the stored graph (same walk, same closed form)
        m2 = pkg.MRFMap.from_workload(w)
        m2.set_stream(torch.cuda.current_stream().cuda_stream)
        if "kf" in mode:
            m2.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
        with m2:
            for fr in w.frames:
                m2.add_frame(fr.depth, fr.K, fr.T_wc)
            m2.bp_iterate(5)
            assert np.array_equal(m2.marginals(), marg)


def test_patch_evaluate_matches_oracle(tinyp):
    """mrf_evaluate with the per-patch sigma band: every pixel's class identical to the oracle's."""
    p = oracle.Params.from_workload(tinyp)
    fr = tinyp.frames[0]
    with _gpu_map(tinyp) as m:
        m.bp_iterate(10)
        xmap = p.L0 + m.export_beliefs().astype(np.float64) / 2.0 ** 23
        res = [m.evaluate(fr.depth, fr.K, fr.T_wc, k_sigma=k) for k in (1.5, 30.0)]
    for k, (cls, nv, na) in zip((1.5, 30.0), res):
        rcls, rnv, rna = oracle.eval_frame(p, fr, xmap, k_sigma=k)
        assert np.array_equal(cls, rcls) and (nv, na) == (rnv, rna)


def test_patch_noise_argument_checks(tinyp):
    w = tinyp
    pm = w.patch
    with _gpu_map(synth.tiny()) as m:
        with pytest.raises(pkg.MrfError, match="STATE"):
            m.set_patch_noise(pm.patch_px, pm.coeffs)            # after the first frame
    m = pkg.MRFMap.from_workload(synth.tiny())
    with m:
        with pytest.raises(pkg.MrfError, match="INVALID"):
            m.set_patch_noise(20, np.full((3, 4, 6), np.nan))
        with pytest.raises(pkg.MrfError, match="INVALID"):
            m.set_patch_noise(20, pm.coeffs, sigma_min=0.0)
        big = pm.coeffs.copy()
        big[..., 3] = 100.0                                      # 3 sigma over the grid diagonal
        with pytest.raises(pkg.MrfError, match="INVALID"):
            m.set_patch_noise(20, big)
        m.set_patch_noise(10, pm.coeffs)                         # 40 x 30 pixels < 64 x 48
        fr = w.frames[0]
        with pytest.raises(pkg.MrfError, match="INVALID"):
            m.add_frame(fr.depth, fr.K, fr.T_wc)
        m.set_patch_noise(0, None)                               # back to the table
        m.add_frame(fr.depth, fr.K, fr.T_wc)
        p = oracle.Params.from_workload(synth.tiny())
        g = oracle.build_graph(p, [fr])
        _assert_graph_equal(m.export_graph(), g)
