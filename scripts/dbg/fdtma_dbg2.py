"""Debug: FULL_FD TMA vs LDG fused at 512x512xNZ: first differing step, where."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2107_14774_b200 as P
import synth

for nz in (32, 32, 64):
    w = synth.CONFIGS["weak"].scaled(nz=nz, corrections=synth.CORR_FULL_FD)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 2024)

    def mk(tma):
        os.environ["LBM_FD_FUSED"] = "1"
        os.environ["LBM_FD_TMA"] = "1" if tma else "0"
        g = P.Lattice(**w.params(), graphs=1)
        g.init_fields(rho, u)
        return g

    a, b, b2 = mk(False), mk(True), mk(True)
    for step in range(1, 6):
        for g in (a, b, b2):
            g.step(1)
        fa, fb, fb2 = a.get_populations(), b.get_populations(), b2.get_populations()
        d = np.abs(fb - fa)
        bad = np.argwhere(d.max(axis=0) > 0)
        print(nz, step, "tma==tma", np.array_equal(fb, fb2), "max", d.max(), "nbad", len(bad),
              "z", sorted(set(bad[:, 0].tolist()))[:12], "y", sorted(set(bad[:, 1].tolist()))[:12],
              "x", sorted(set(bad[:, 2].tolist()))[:12], flush=True)
        if len(bad):
            q = np.argwhere(d[:, bad[0][0], bad[0][1], bad[0][2]] > 0).ravel()
            print("   first bad node", bad[0], "q", q.tolist(), flush=True)
    for g in (a, b, b2):
        g.close()
