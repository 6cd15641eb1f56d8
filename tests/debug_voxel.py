"""Diagnostic (test infrastructure: compares with the oracle): messages into the worst one-step
marginal voxel (run by hand on a GPU box: python -m tests.debug_voxel)."""
import numpy as np

import oracle
import synth
import paper_2006_03512_b200 as pkg

w = synth.frames30(n_frames=2)
p = oracle.Params.from_workload(w)
g = oracle.build_graph(p, w.frames)
m = pkg.MRFMap.from_workload(w)
for fr in w.frames:
    m.add_frame(fr.depth, fr.K, fr.T_wc)
m.bp_iterate(2)
lam0 = m.export_messages()
m.import_messages(lam0)
lam0 = m.export_messages()
m.bp_iterate(1)
lam1 = m.export_messages().astype(np.float64)
marg = m.marginals().astype(np.float64)
lam = lam0.astype(np.float64)
T0 = oracle.accumulate(p, g, lam)
oracle.ray_pass(p, g, T0, lam)
T = oracle.accumulate(p, g, lam)
mref = oracle.marginals(p, T)
dm = np.abs(marg - mref)
order = np.argsort(-dm)[:5]
ray_of = np.repeat(np.arange(g.n_rays), np.diff(g.row_ptr))
pos_of = np.arange(g.E) - g.row_ptr[ray_of]
for v in order:
    es = np.nonzero(g.vid == v)[0]
    d = lam1[es] - lam[es]
    print(f"v={v} dm={dm[v]:.2e} deg={len(es)} T={T[v]:.4f} sum err {d.sum():.3e} mean {d.mean():.2e}")
    big = es[np.argsort(-np.abs(d))[:6]]
    for e in big:
        r = ray_of[e]
        n = g.row_ptr[r + 1] - g.row_ptr[r]
        c = p.L0 + T0[v] - lam0[e]
        print(f"   e={e} ray={r} pos={pos_of[e]}/{n} lam_ref={lam[e]:+.6f} gpu={lam1[e]:+.6f} err={lam1[e]-lam[e]:+.2e} cav={c:+.3f}")
    # error distribution by position relative to ray end
    rel = (g.row_ptr[ray_of[es] + 1] - es)
    print("   err by (n - pos) bucket:", {int(k): float(np.mean(d[rel == k])) for k in np.unique(rel)[:8]})
m.close()
