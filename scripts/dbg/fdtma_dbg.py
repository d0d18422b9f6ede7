"""Debug: locate differences of the FULL_FD TMA kernel against the LDG fused kernel."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2107_14774_b200 as P
import synth

w = synth.CONFIGS["tgv"].scaled(nx=160, ny=36, nz=12, corrections=synth.CORR_FULL_FD)
rho, u = synth.random_fields(w.nx, w.ny, w.nz, 31)


def mk(tma, **kw):
    os.environ["LBM_FD_FUSED"] = "1"
    os.environ["LBM_FD_TMA"] = "1" if tma else "0"
    g = P.Lattice(**w.params(), **kw)
    g.init_fields(rho, u)
    return g


for steps in (1, 2, 23):
    a = mk(False, graphs=1)
    a.step(steps)
    fa = a.get_populations()
    a.close()
    for name, kw in [("g1", dict(graphs=1)), ("g1b", dict(graphs=1)), ("g2", dict(graphs=2)), ("g0", {}),
                     ("nccl", dict(halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id()))]:
        g = mk(True, **kw)
        g.step(steps)
        fg = g.get_populations()
        g.close()
        d = np.abs(fg - fa)
        idx = np.unravel_index(np.argmax(d), d.shape)
        bad = np.argwhere(d.max(axis=0) > 1e-14)
        xs = sorted(set(bad[:, 2].tolist()))[:20]
        ys = sorted(set(bad[:, 1].tolist()))[:20]
        zs = sorted(set(bad[:, 0].tolist()))[:20]
        print(steps, name, "max", d.max(), "at", idx, "nbad", len(bad), "x", xs, "y", ys, "z", zs, flush=True)
