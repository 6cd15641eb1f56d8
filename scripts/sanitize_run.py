"""Workload for compute-sanitizer and for the bounds-checked build: the tiny scene from 4 keyframes through every
K5 / K6 path and mode of the library -- the class kernels, the long-ray tiled kernel (a
corridor), the TMA-staged K5 (MRF_K5=staged), the per-voxel K6 ablation (MRF_K6=voxel), the
compacted reduction (MRF_COMPACT=1), keyframe averages, sparse bricks, matrix-free walks, the
§III.D evaluation and the exports.  Results are not checked here (the parity tests do that);
the sanitizer's verdict is the point.  Run one mode per process: python scripts/sanitize_run.py MODE
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
import paper_2006_03512_b200 as pkg  # noqa: E402
from synth.scenes import Frame  # noqa: E402


def corridor():
    dims, res = (700, 8, 8), 0.01
    C = np.array([0.002, 0.04, 0.04])
    R = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])
    W, H, K = 6, 4, (2000.0, 2000.0, 2.5, 1.5)
    depth = np.full((H, W), 650.3 * res - C[0], np.float32)
    lut = synth.build_log_nu_lut(32, 128, 0.0, 12.0, -1.0, 1.0, (0.005, 0.0, 0.0), 0.0)
    return synth.Workload("corridor", dims, res, (0, 0, 0), 0.1, lut, 0.0, 12.0, -1.0, 1.0, 0.1, 3.0,
                          (0.005, 0.0, 0.0), 3, [Frame(depth, np.array(K), np.concatenate([R, C[:, None]], 1).reshape(-1))])


def run(mode):
    w = corridor() if mode == "long" else (synth.frames30(n_frames=3) if mode == "room" else synth.tiny_frames(n_frames=4))
    m = pkg.MRFMap.from_workload(w)
    with m:
        if mode in ("kfavg", "kfmf"):
            m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
        if mode == "sparse":
            m.set_sparse_bricks(8)
        if mode in ("mf", "kfmf"):
            m.set_matrix_free(2)
        for fr in w.frames[:-1] if len(w.frames) > 1 and mode != "sparse" else w.frames:
            m.add_frame(fr.depth, fr.K, fr.T_wc)
        m.bp_iterate(2)
        if len(w.frames) > 1 and mode != "sparse":  # warm start
            fr = w.frames[-1]
            m.add_frame(fr.depth, fr.K, fr.T_wc)
        m.bp_iterate(2)
        m.marginals()
        if mode != "kfmf":  # (keyframe averages + matrix-free walks keep no per-incidence messages)
            lam = m.export_messages()
            m.import_messages(lam)
        m.bp_iterate(1)
        if mode not in ("mf", "kfmf"):
            g = m.export_graph()
            m.export_rays(g["frame"][:50], g["pixel"][:50])
            m.export_transpose()
        fr = w.frames[0]
        m.evaluate(fr.depth, fr.K, fr.T_wc)
        m.graph_sizes()
    print(f"sanitize_run {mode}: done")


if __name__ == "__main__":
    run(sys.argv[1] if len(sys.argv) > 1 else "default")
