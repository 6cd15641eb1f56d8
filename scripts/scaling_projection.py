"""Projected multi-GPU step time from per-rank measurements on ONE GPU (this run has one GPU).

    python scripts/scaling_projection.py [--config frames100] [--worlds 2 4 8] [--steps 3]

For each world size W the workload is split into W emulated ranks (dist.EmulatedRanks: the
pixel rows v % W == r, exactly the real path's sharding), one ctx per rank on this GPU, and each
rank's own kernel time per step (graph build + n BP iterations: CUDA events on its stream,
mrf_profile_read) is measured.  The projection for W GPUs is

    T_W = max_r (rank r's kernel time per step) + n * t_allreduce(8 * belief_slots bytes)

with t_allreduce = 2 (W - 1) / W * bytes / 725 GB/s, the measured 8-rank NCCL all-reduce bus
bandwidth on this pool (/opt/skills/guides/B200_PROFILING.md).  T_1 is the sum of the ranks'
kernel times of the W = 1 split.  This is a PROJECTION (no NCCL traffic, no per-GPU clocks or
HBM contention are measured), printed as one JSON line with "kind": "projection".
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BUSBW_GBS = 725.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="frames100")
    ap.add_argument("--worlds", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()

    import torch
    import synth
    from paper_2006_03512_b200.dist import EmulatedRanks

    w = synth.make_workload(a.config)
    depth = [torch.from_numpy(fr.depth).cuda() for fr in w.frames]
    n_iter = w.n_iter
    out = {"kind": "projection", "config": a.config, "bp_iterations": n_iter, "busbw_GBs": BUSBW_GBS,
           "worlds": {}}
    base = None
    for W in ([1] if a.config not in ("frames100", "sweep300") else []) + a.worlds:
        em = EmulatedRanks(w, W)

        def step():
            em.reset()
            for fr, d in zip(w.frames, depth):
                em.add_frame(d, fr.K, fr.T_wc)
            em.bp_iterate(n_iter)

        step()
        torch.cuda.synchronize()
        for m in em.maps:
            m.set_profiling(True)
            m.profile_read()
        for _ in range(a.steps):
            step()
        torch.cuda.synchronize()
        per_rank = []
        for m in em.maps:
            prof = m.profile_read()
            per_rank.append({k: v[1] / a.steps for k, v in prof.items()})
            m.set_profiling(False)
        tot = [sum(p.values()) for p in per_rank]
        slots = em.maps[0].belief_slots()
        t_ar = 2 * (W - 1) / W * 8 * slots / (BUSBW_GBS * 1e9) * 1e3 if W > 1 else 0.0
        T_W = max(tot) + n_iter * t_ar
        rec = {"rank_kernel_ms_per_step": [round(t, 3) for t in tot],
               "max_rank_ms": round(max(tot), 3), "sum_ranks_ms": round(sum(tot), 3),
               "imbalance_max_over_mean": round(max(tot) / (sum(tot) / W), 4),
               "allreduce_ms_per_iteration": round(t_ar, 4), "projected_ms_per_step": round(T_W, 3),
               "k5_ms": [round(p.get("ray_messages", 0.0), 3) for p in per_rank],
               "k6_ms": [round(p.get("voxel_sum", 0.0), 3) for p in per_rank]}
        if base is None:
            base = sum(tot)  # one GPU holding every rank: the sum of the ranks' kernel times
            out["one_gpu_kernel_ms_per_step"] = round(base, 3)
        rec["projected_speedup"] = round(base / T_W, 3)
        out["worlds"][W] = rec
        em.close()
        torch.cuda.empty_cache()
        print(json.dumps({W: rec}), file=sys.stderr, flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
