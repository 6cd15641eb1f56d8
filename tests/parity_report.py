"""Parity report (GPU vs oracle) per iteration count -- a diagnostic, run by hand:

    python -m tests.parity_report [tiny|frame1|frames30:k] [n_iter ...]
"""

import sys

import numpy as np

import oracle
import synth
import paper_2006_03512_b200 as pkg


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "onestep":
        return onestep(sys.argv[2] if len(sys.argv) > 2 else "frames30:2", int(sys.argv[3]) if len(sys.argv) > 3 else 2)
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


def onestep(name="frames30:2", k=2):
    """One step from the GPU state after k iterations: signed error statistics."""
    w = synth.frames30(n_frames=int(name.split(":")[1])) if name.startswith("frames30:") else synth.make_workload(name)
    p = oracle.Params.from_workload(w)
    g = oracle.build_graph(p, w.frames)
    deg = np.bincount(g.vid, minlength=p.V)
    m = pkg.MRFMap.from_workload(w)
    for fr in w.frames:
        m.add_frame(fr.depth, fr.K, fr.T_wc)
    m.bp_iterate(k)
    lam0 = m.export_messages()
    m.import_messages(lam0)
    lam0 = m.export_messages()
    m.bp_iterate(1)
    lam1 = m.export_messages().astype(np.float64)
    Tg = m.export_beliefs().astype(np.float64) / 2 ** 23
    marg = m.marginals().astype(np.float64)
    m.close()
    lam = lam0.astype(np.float64)
    oracle.ray_pass(p, g, oracle.accumulate(p, g, lam), lam)
    T = oracle.accumulate(p, g, lam)
    d = lam1 - lam
    q = np.abs(d) / np.maximum(1, np.abs(lam))
    print(f"{name} k={k}: E={g.E} msg rel max {q.max():.2e}  mean signed err {d.mean():.3e}  mean|err| {np.abs(d).mean():.3e}")
    for lo, hi in [(0, 1e-6), (1e-6, 1e-3), (1e-3, 0.1), (0.1, 1), (1, 10), (10, 300)]:
        sel = (np.abs(lam) >= lo) & (np.abs(lam) < hi)
        if sel.any():
            print(f"   |lam| in [{lo:g},{hi:g}): n={sel.sum():9d} mean err {d[sel].mean():+.3e} rms {np.sqrt((d[sel]**2).mean()):.3e}")
    dT = Tg - T
    mref = oracle.marginals(p, T)
    dm = np.abs(marg - mref)
    v = int(dm.argmax())
    print(f"   marg max {dm.max():.2e} at v={v} deg={deg[v]} dT={dT[v]:.3e} p={mref[v]:.4f}; "
          f"dT/deg for deg>1000: mean {np.mean(dT[deg > 1000] / deg[deg > 1000]):.2e}")


if __name__ == "__main__":
    main()
