"""Time the BP kernels (K5 ray messages, K6 voxel sums) under build/runtime variants on one
workload, and report how far each variant's marginals move from the first one's.

    python scripts/k_variants.py [--config frames30] [--iters 10] VAR=val,VAR=val ...

Each positional argument is one variant: comma-separated environment settings read by
mrf_create (MRF_K5_LSE=fast|acc, MRF_K6=tile|voxel|atomic, MRF_L2_FETCH=32|64|128).
A diagnostic for the kernel work, not a bench line.
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="*", default=[""])
    ap.add_argument("--config", default="frames30")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()

    import torch
    import synth
    import paper_2006_03512_b200 as pkg

    w = synth.make_workload(a.config)
    depth = [torch.from_numpy(fr.depth).cuda() for fr in w.frames]
    E_alg = None
    ref = None
    keys = ("MRF_K5", "MRF_K5_MATH", "MRF_K6", "MRF_L2_FETCH", "MRF_K6_ITEM", "MRF_K5_STREAMS", "MRF_K6_DYNAMIC", "MRF_K6_LPT", "MRF_K6_PAD", "MRF_K6_FRAMES", "MRF_RUN_FILL")
    for var in a.variants:
        for k in keys:
            os.environ.pop(k, None)
        env = dict(kv.split("=") for kv in var.split(",") if kv)
        os.environ.update(env)
        m = pkg.MRFMap.from_workload(w)
        m.set_stream(torch.cuda.current_stream().cuda_stream)
        for fr, d in zip(w.frames, depth):
            m.add_frame(d, fr.K, fr.T_wc)
        m.bp_iterate(1)  # prepare + warm-up
        torch.cuda.synchronize()
        E_alg = m.graph_sizes()["E"]
        best = None
        for _ in range(a.repeat):
            m.set_profiling(True)
            m.profile_read()
            m.bp_iterate(a.iters)
            torch.cuda.synchronize()
            prof = m.profile_read()
            m.set_profiling(False)
            t5 = prof["ray_messages"][1] / a.iters
            t6 = prof["voxel_sum"][1] / a.iters
            if best is None or t5 + t6 < best[0] + best[1]:
                best = (t5, t6)
        # parity between variants: fresh trajectory of `iters` iterations from zero messages
        m.reset()
        for fr, d in zip(w.frames, depth):
            m.add_frame(d, fr.K, fr.T_wc)
        m.bp_iterate(a.iters)
        out = torch.empty(w.n_voxels, dtype=torch.float32, device="cuda")
        m.marginals(out)
        marg = out.cpu().numpy()
        m.close()
        if ref is None:
            ref = marg
        t5, t6 = best
        V = w.n_voxels
        rec = {"variant": var or "default", "E": E_alg, "k5_ms": round(t5, 4), "k6_ms": round(t6, 4),
               "k5_GBs": round((14 * E_alg + 8 * V) / t5 / 1e6, 1) if t5 > 0 else None,
               "k6_GBs": round((8 * E_alg + 8 * V) / t6 / 1e6, 1) if t6 > 0 else None,
               "iter_ms": round(t5 + t6, 4),
               "bp_frac_22B": round((22 * E_alg + 16 * V) / (t5 + t6) / 1e6 / 6544.3, 4),
               "max_dmarg_vs_first": float(np.max(np.abs(marg.astype(np.float64) - ref)))}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
