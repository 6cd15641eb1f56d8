"""Distinct voxels per pixel block (DESIGN §5 K6b): how many different voxels the rays of a
block of neighbouring pixels traverse, from the oracle's graph of single frames of frames30.
Not a test; run by hand:  python tests/block_locality.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth.scenes as sc  # noqa: E402


def main():
    w = sc.frames30()
    p = oracle.Params.from_workload(w)
    W = w.frames[0].depth.shape[1]
    for fi in (3, 10, 17, 24, 29):
        g = oracle.build_graph(p, [w.frames[fi]])
        u, v = g.pixel % W, g.pixel // W
        ray_of = np.repeat(np.arange(g.n_rays), np.diff(g.row_ptr))
        out = []
        for bu, bv in [(32, 16), (16, 16), (32, 8), (16, 8)]:
            blk = (v // bv) * 1000 + (u // bu)
            key = np.unique(blk[ray_of].astype(np.int64) * (1 << 32) + g.vid)
            per = np.bincount(np.searchsorted(np.unique(blk), key >> 32))
            out.append(f"{bu}x{bv}: incidences/distinct {g.E / len(key):.0f}, distinct per block "
                       f"p50 {np.percentile(per, 50):.0f} p99 {np.percentile(per, 99):.0f} max {per.max()}")
        print(f"frame {fi} (E = {g.E}): " + " | ".join(out))


if __name__ == "__main__":
    main()
