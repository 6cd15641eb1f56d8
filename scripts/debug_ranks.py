"""Diagnostic: world=1 vs emulated ranks (run by hand on a GPU box)."""
import numpy as np
import torch

import synth
import paper_2006_03512_b200 as pkg


def gmap(w, **kw):
    m = pkg.MRFMap.from_workload(w, **kw)
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    for fr in w.frames:
        m.add_frame(fr.depth, fr.K, fr.T_wc)
    return m


w = synth.frames30(n_frames=2)
for iters in (0, 1, 2):
    m1 = gmap(w)
    m1.bp_iterate(iters)
    T1 = m1.export_beliefs()
    g1 = m1.export_graph()
    lam1 = m1.export_messages()
    maps = [gmap(w, rank=r, world=2, comm=pkg.MRF_COMM_EXTERNAL) for r in range(2)]
    parts = [torch.zeros(maps[0].belief_slots(), dtype=torch.int64, device="cuda") for _ in range(2)]
    for _ in range(iters):
        for m, p in zip(maps, parts):
            m.bp_partial(p, iterate=True)
        tot = parts[0] + parts[1]
        for m in maps:
            m.bp_finish(tot)
    torch.cuda.synchronize()
    Ts = [m.export_beliefs() for m in maps]
    print(f"iters={iters}: T equal r0 {np.array_equal(Ts[0], T1)} r1 {np.array_equal(Ts[1], T1)} "
          f"ndiff {(Ts[0] != T1).sum()} maxdiff {np.abs(Ts[0] - T1).max()}")
    # per-rank messages vs the same rays in world=1
    key1 = {(int(f), int(p)): i for i, (f, p) in enumerate(zip(g1["frame"], g1["pixel"]))}
    for r, m in enumerate(maps):
        g = m.export_graph()
        lam = m.export_messages()
        bad = 0
        for i in range(len(g["frame"])):
            j = key1[(int(g["frame"][i]), int(g["pixel"][i]))]
            a = lam[g["row_ptr"][i]:g["row_ptr"][i + 1]]
            b = lam1[g1["row_ptr"][j]:g1["row_ptr"][j + 1]]
            if not np.array_equal(a, b):
                bad += 1
        print(f"   rank {r}: rays {len(g['frame'])} with differing messages: {bad}")
    for m in maps + [m1]:
        m.close()
