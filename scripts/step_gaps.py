"""Where the frames30 bench step spends the time that no kernel accounts for (a diagnostic):
device time of each phase of the step (CUDA events on the ctx stream) against the kernel
times the library records (mrf_profile_read) inside it.

    python scripts/step_gaps.py [--config frames30]
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
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import synth
    import paper_2006_03512_b200 as pkg
    w = synth.make_workload(a.config)
    st = torch.cuda.current_stream()
    depth = [torch.from_numpy(fr.depth).cuda() for fr in w.frames]
    m = pkg.MRFMap.from_workload(w)
    m.set_stream(st.cuda_stream)
    out = torch.empty(w.n_voxels, device="cuda")

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        return e

    for rep in range(a.reps + 1):
        m.set_profiling(True)
        m.profile_read()
        e0 = ev()
        m.reset()
        for fr, d in zip(w.frames, depth):
            m.add_frame(d, fr.K, fr.T_wc)
        e1 = ev()
        m.layout_sizes()  # the deferred fill + transpose build (prepare)
        e2 = ev()
        m.bp_iterate(w.n_iter)
        e3 = ev()
        m.marginals(out)
        e4 = ev()
        torch.cuda.synchronize()
        prof = m.profile_read()
        m.set_profiling(False)
        if rep == 0:
            continue
        k = {n: round(v[1], 3) for n, v in prof.items() if v[0]}
        print(json.dumps({"add_frames_ms": round(e0.elapsed_time(e1), 3), "prepare_ms": round(e1.elapsed_time(e2), 3),
                          "iterate_ms": round(e2.elapsed_time(e3), 3), "marginals_ms": round(e3.elapsed_time(e4), 3),
                          "step_ms": round(e0.elapsed_time(e4), 3), "kernels_ms": k,
                          "kernel_sum_ms": round(sum(k.values()), 3)}), flush=True)
    m.close()


if __name__ == "__main__":
    main()
