"""Parity report (GPU vs oracle) per iteration count -- a diagnostic, run by hand:

    python -m tests.parity_report [tiny|frame1|frames30:k] [n_iter ...]
"""

import sys

import numpy as np

import oracle
import synth
import paper_2006_03512_b200 as pkg


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    iters = [int(x) for x in sys.argv[2:]] or [1, 3, 10]
    if name.startswith("frames30:"):
        w = synth.frames30(n_frames=int(name.split(":")[1]))
    else:
        w = synth.make_workload(name)
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    deg = np.bincount(g.vid, minlength=p.V)
    print(f"{name}: E={g.E} rays={g.n_rays} max deg={deg.max()}")
    for n in iters:
        lam_ref, T_ref = oracle.bp(p, g, n)
        m = pkg.MRFMap.from_workload(w)
        for fr in w.frames:
            m.add_frame(fr.depth, fr.K, fr.T_wc)
        m.bp_iterate(n)
        lam = m.export_messages().astype(np.float64)
        marg = m.marginals().astype(np.float64)
        T = m.export_beliefs().astype(np.float64) / 2 ** 23
        m.close()
        rel = np.abs(lam - lam_ref) / np.maximum(1, np.abs(lam_ref))
        mref = oracle.marginals(p, T_ref)
        dm = np.abs(marg - mref)
        v = int(dm.argmax())
        e = int(rel.argmax())
        print(f" n={n:3d} msg rel max {rel.max():.2e} p99 {np.quantile(rel, 0.99):.2e} | marg max {dm.max():.2e} "
              f"at v={v} deg={deg[v]} T_gpu={T[v]:.4f} T_ref={T_ref[v]:.4f} p={mref[v]:.4f} | "
              f"worst msg e={e} lam={lam[e]:.5f} ref={lam_ref[e]:.5f} | dT max {np.abs(T - T_ref).max():.2e}")


if __name__ == "__main__":
    main()
