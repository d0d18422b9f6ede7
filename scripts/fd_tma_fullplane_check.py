"""FULL_FD at the bench's plane (512 x 512, 32 planes, periodic, config-5
physics), 200 steps from random fields: the TMA-staged fused kernel against the
LDG fused kernel (same per-node arithmetic: expected bitwise) and the two-pass
path (equal to rounding), fp64 and fp32 storage, and a second TMA run
(deterministic).  Writes
results/fd_tma_fullplane.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2107_14774_b200 as P  # noqa: E402
import synth  # noqa: E402

STEPS = 200
out = {"lattice": "512x512x32 periodic, config-5 physics, FULL_FD", "steps": STEPS, "cases": []}
for prec in (0, 1):
    w = synth.CONFIGS["weak"].scaled(nz=32, corrections=synth.CORR_FULL_FD, precision=prec)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 2024)
    res = {}
    for name, env in (("tma", {"LBM_FD_TMA": "1"}), ("tma_again", {"LBM_FD_TMA": "1"}),
                      ("ldg_fused", {"LBM_FD_TMA": "0", "LBM_FD_FUSED": "1"}),
                      ("two_pass", {"LBM_FD_TMA": "0", "LBM_FD_FUSED": "0"})):
        for k in ("LBM_FD_TMA", "LBM_FD_FUSED"):
            os.environ.pop(k, None)
        os.environ.update(env)
        g = P.Lattice(**w.params())
        kname = g.kernel_name()
        g.init_fields(rho, u)
        g.step(STEPS)
        res[name] = (g.get_populations(), kname)
        g.close()
    ft = res["tma"][0]
    case = {"precision": "fp64" if prec == 0 else "fp32 storage", "kernels": {k: v[1] for k, v in res.items()}}
    for other in ("tma_again", "ldg_fused", "two_pass"):
        fo = res[other][0]
        case[f"tma_vs_{other}"] = {"bitwise_equal": bool(np.array_equal(ft, fo)),
                                   "max_abs_diff": float(np.abs(ft - fo).max()),
                                   "max_rel_diff": float((np.abs(ft - fo) / np.abs(fo)).max())}
    case["finite"] = bool(np.all(np.isfinite(ft)))
    out["cases"].append(case)
    print(json.dumps(case), flush=True)
os.makedirs(os.path.join(ROOT, "results"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "results", "fd_tma_fullplane.json"), "w"), indent=1)
