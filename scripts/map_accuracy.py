"""§III.D generating-surface accuracy (§V) of the maps the bench
builds, per frame, on the GPU (mrf_evaluate, K9): both classification modes of reading R21.

    python scripts/map_accuracy.py [--config frames30] [--frames 0,10,20]

Not a bench line.  See DESIGN.md §K9 for why the 5 cm configs score low under this metric
(walls on voxel faces, a 1.5-sigma band narrower than a voxel).
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="frames30")
    ap.add_argument("--frames", default="0")
    ap.add_argument("--iters", type=int, default=None)
    a = ap.parse_args()
    import torch
    import synth
    import paper_2006_03512_b200 as pkg
    from paper_2006_03512_b200.dist import EmulatedRanks
    w = synth.make_workload(a.config)
    emulate = 4 if a.config in ("frames100", "sweep300") else 1
    m = EmulatedRanks(w, emulate) if emulate > 1 else pkg.MRFMap.from_workload(w)
    for fr in w.frames:
        m.add_frame(torch.from_numpy(fr.depth).cuda(), fr.K, fr.T_wc)
    m.bp_iterate(w.n_iter if a.iters is None else a.iters)
    maps = m.maps if emulate > 1 else [m]
    for fi in (int(x) for x in a.frames.split(",")):
        fr = w.frames[fi]
        out = {"config": a.config, "frame": fi}
        for mode, name in ((pkg._lib.MRF_EVAL_SIGMA_BAND, "sigma_band_1.5"), (pkg._lib.MRF_EVAL_VOXEL_BOUNDS, "voxel_bounds")):
            res = [mm.evaluate(fr.depth, fr.K, fr.T_wc, mode=mode)[1:] for mm in maps]
            nv, na = sum(r[0] for r in res), sum(r[1] for r in res)
            out["valid_pixels"] = nv
            out[name] = na / max(nv, 1)
        print(json.dumps(out))
    m.close()


if __name__ == "__main__":
    main()
