"""Pins of the oracle's sparse-brick variant ("new bricks
are allocated in a region around the reprojected 3D depth point cloud ... empty skip 3DDA ray
traversals"; reading R23): SPEC's allocate_for_depth_image examples and post-condition
(checked by an independent numpy enumeration), the empty-skip walk against the brute-force-pinned
dense walk, and skipped cells acting as certainly-empty voxels of the ray factor."""


import numpy as np

import oracle
import synth
from synth.scenes import Frame


def _points(p, fr):
    """Reprojected depth points (grid units) and 3 sigma radii (voxels), numpy, per valid pixel."""
    H, W = fr.depth.shape
    K, T = np.asarray(fr.K, float), np.asarray(fr.T_wc, float).reshape(3, 4)
    v, u = np.nonzero(np.isfinite(fr.depth) & (fr.depth > 0))
    z = fr.depth[v, u].astype(np.float64)
    xc, yc = (u - K[2]) / K[0], (v - K[3]) / K[1]
    D = T[:, :3] @ np.stack([xc, yc, np.ones_like(xc)])
    pts = ((T[:, 3:4] + z * D) - p.geo[1:4, None]) / p.geo[0]
    Z = z * np.sqrt(xc * xc + yc * yc + 1)
    sig = p.par[6] + p.par[7] * Z + p.par[8] * Z * Z
    r = p.par[5] * sig / p.geo[0]
    inside = np.all((pts >= 0) & (pts < p.dims[:, None]), axis=0)
    return pts[:, inside].T, r[inside]


def test_allocation_spec_examples():
    """SPEC: one valid pixel (SPEC's depth 1 m example at 0.5 m: the tiny grid is 1.6 m wide and
    the camera sits at x = 0.8 m) -> at least one brick, containing the reprojected point; an
    all-invalid image -> no brick."""
    w = synth.tiny()
    p = oracle.Params.from_workload(w)
    fr = w.frames[0]
    d = np.zeros_like(fr.depth)
    d[20, 30] = 0.5
    bk = oracle.alloc_bricks(p, [Frame(d, fr.K, fr.T_wc)])
    assert bk.added == [int(bk.mask.sum())] and bk.mask.sum() >= 1
    pts, _ = _points(p, Frame(d, fr.K, fr.T_wc))
    c = np.floor(pts[0]).astype(int) // bk.B
    assert bk.mask[c[2], c[1], c[0]] == 1
    bk0 = oracle.alloc_bricks(p, [Frame(np.zeros_like(fr.depth), fr.K, fr.T_wc)])
    assert bk0.added == [0] and bk0.mask.sum() == 0
    # allocating the same image again adds nothing (previously allocated bricks untouched)
    bk2 = oracle.alloc_bricks(p, [Frame(d, fr.K, fr.T_wc)], bricks=bk)
    assert bk2.added == [0]


def test_allocation_covers_every_voxel_within_r():
    """SPEC post-condition, by independent enumeration: every voxel whose cell lies within
    r_alloc = 3 sigma(Z) of a reprojected depth point belongs to an allocated brick."""
    for w in (synth.tiny(), synth.tiny_frames(n_frames=3)):
        p = oracle.Params.from_workload(w)
        bk = oracle.alloc_bricks(p, w.frames)
        for fr in w.frames:
            pts, r = _points(p, fr)
            for q, rr in zip(pts, r):
                lo = np.maximum(np.floor(q - rr - 1).astype(int), 0)
                hi = np.minimum(np.floor(q + rr + 1).astype(int), p.dims - 1)
                for cz in range(lo[2], hi[2] + 1):
                    for cy in range(lo[1], hi[1] + 1):
                        for cx in range(lo[0], hi[0] + 1):
                            c = np.array([cx, cy, cz])
                            dist = np.linalg.norm(np.maximum(0, np.maximum(c - q, q - (c + 1))))  # point-box
                            if dist <= rr:
                                assert bk.mask[cz // bk.B, cy // bk.B, cx // bk.B] == 1


def test_empty_skip_walk_is_the_dense_walk_filtered():
    """The sparse walk emits exactly the dense walk's cells (B2, pinned by the rational brute
    force) that lie in allocated bricks, with their own offsets and crossing parameters; a full
    mask gives the dense walk."""
    rng = np.random.default_rng(0)
    dims = np.array([40, 36, 24], np.int32)
    p = oracle.Params(dims, 0.05, (0, 0, 0), 0.5, np.zeros((4, 4), np.float32), 0, 2, -0.2, 0.2, 0.1, 3,
                      (0, 0, 0.0012))
    bk = oracle.Bricks(p, 8)
    bk.mask[...] = rng.integers(0, 2, bk.mask.shape)
    full = oracle.Bricks(p, 8)
    full.mask[...] = 1
    for _ in range(400):
        G0 = (rng.uniform(0, dims) * 65536).astype(np.int64)
        G1 = (rng.uniform(-2, dims + 2) * 65536).astype(np.int64)
        vid, off, tin, tout = oracle.dda(dims, G0, G1, 1.0, 1.3)
        x, y, z = vid % dims[0], (vid // dims[0]) % dims[1], vid // (dims[0] * dims[1])
        keep = bk.mask[z // 8, y // 8, x // 8] == 1
        sv, so, si, st = oracle.dda_sparse(dims, G0, G1, bk, 1.0, 1.3)
        assert np.array_equal(sv, vid[keep]) and np.array_equal(so, off[keep])
        assert np.array_equal(si, tin[keep]) and np.array_equal(st, tout[keep])
        fv, fo, _, _ = oracle.dda_sparse(dims, G0, G1, full, 1.0, 1.3)
        assert np.array_equal(fv, vid) and np.array_equal(fo, off)


def test_skipped_cells_are_certainly_empty():
    """A ray restricted to its allocated cells sends the messages that the full ray would send if
    its unallocated cells were certainly empty (cavity -> -inf: mu(o=0) = 1 in Eq.13/14)."""
    rng = np.random.default_rng(1)
    for _ in range(300):
        n = int(rng.integers(2, 30))
        c = rng.uniform(-6, 6, n)
        lnu = rng.uniform(-8, 2, n)
        keep = rng.random(n) < 0.6
        if keep.sum() < 1:
            continue
        lpos_s, lneg_s = oracle.ray_messages(c[keep], lnu[keep])
        c_full = np.where(keep, c, -np.inf)
        lpos_f, lneg_f = oracle.ray_messages(c_full, lnu)
        lam_s = np.clip(lpos_s - lneg_s, -256, 256)
        lam_f = np.clip(lpos_f - lneg_f, -256, 256)[keep]
        assert np.allclose(lam_s, lam_f, rtol=0, atol=1e-9)


def test_sparse_graph_and_bp():
    """Tiny scene: the sparse graph is the dense graph restricted to allocated cells, ray by ray;
    BP on it leaves unallocated voxels at the prior."""
    w = synth.tiny()
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    bk = oracle.alloc_bricks(p, w.frames)
    gs = oracle.build_graph(p, w.frames, bricks=bk)
    alloc = bk.cell_mask(p)
    assert np.array_equal(gs.pixel, g.pixel) or set(gs.pixel) <= set(g.pixel)
    kept = alloc[g.vid]
    assert gs.E == int(kept.sum()) < g.E
    assert np.array_equal(gs.vid, g.vid[kept])
    lam, T = oracle.bp(p, gs, 3)
    assert np.all(T[~alloc] == 0.0)
    m = oracle.marginals(p, T)
    assert np.all(np.abs(m[~alloc] - p.prior) < 1e-15)
