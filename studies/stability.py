#!/usr/bin/env python
"""Numerical-stability study of PAPER.md §7 (Figs. 8-10) on the GPU.

Lid-driven cubic cavity (physical box; halfway bounce-back on five faces, Eq. 69
lid on +y), cs2 = 0.08, all rates but omega_nu equal to 1 unless varied.  For
each (model, aspect ratios, omega_nu, omega_xi) the largest lid speed U that
stays stable for `steps` steps (no NaN, rho <= 0 or |u| > 1; lbm_cuboid_check)
is found by bisection.  All bisection points of one iteration run concurrently,
one small lattice per CUDA stream, advanced with the library's CUDA graphs.

  python -m studies.stability --study fig8  --steps 100000 --out results/stability_fig8.json
  python -m studies.stability --study fig9  ...
  python -m studies.stability --study fig10 ...   (max Re at U = 0.2)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CS2 = 0.08
BB, MW = 1, 2
CAVITY_BC = (BB, BB, BB, MW, BB, BB)


def case_params(model, nx, ny, nz, r, s, omega_nu, omega_xi, U):
    return dict(nx=nx, ny=ny, nz=nz, r=r, s=s, cs2=CS2, omega_nu=omega_nu, omega_xi=omega_xi,
                omega_1=1.0, omega_high=1.0, bc=CAVITY_BC, wall_u=U, corrections=0, model=model)


def run_batch(cases, steps, check_every=5000):
    """Advance every case concurrently; returns a list of booleans (stable?)."""
    import torch

    import paper_2107_14774_b200 as P

    lats = []
    for c in cases:
        st = torch.cuda.Stream()
        lat = P.Lattice(stream=st, graphs=2, **c)
        nz, ny, nx = lat.local_shape
        rho = torch.ones((nz, ny, nx), dtype=torch.float64, device="cuda")
        u = torch.zeros((3, nz, ny, nx), dtype=torch.float64, device="cuda")
        lat.init_fields(rho, u)
        lats.append(lat)
    torch.cuda.synchronize()
    alive = [True] * len(cases)
    done = 0
    while done < steps:
        n = min(check_every, steps - done)
        for i, lat in enumerate(lats):
            if alive[i]:
                lat.step(n)
        for i, lat in enumerate(lats):
            if alive[i] and lat.check(raise_on_unstable=False)["bad_nodes"] > 0:
                alive[i] = False
        done += n
        if not any(alive):
            break
    for lat in lats:
        lat.close()
    return alive


def bisect(points, steps, u_lo=0.0, u_hi=0.6, iters=7):
    """points: list of dicts with model, grid, r, s, omega_nu, omega_xi.  Returns
    the largest stable U per point (bisection in [u_lo, u_hi])."""
    lo = [u_lo] * len(points)
    hi = [u_hi] * len(points)
    for _ in range(iters):
        mids = [(a + b) / 2 for a, b in zip(lo, hi)]
        cases = [case_params(p["model"], *p["grid"], p["r"], p["s"], p["omega_nu"], p["omega_xi"], m)
                 for p, m in zip(points, mids)]
        ok = run_batch(cases, steps)
        for i, good in enumerate(ok):
            if good:
                lo[i] = mids[i]
            else:
                hi[i] = mids[i]
    return lo, hi


def max_reynolds(points, steps, U=0.2, iters=7):
    """Fig. 10: at fixed U find the smallest stable omega-based viscosity,
    i.e. the largest stable omega_nu in (1, 2), reported as Re = U L / nu with L
    the cavity side in x units."""
    lo = [1.0] * len(points)
    hi = [1.999] * len(points)
    for _ in range(iters):
        mids = [(a + b) / 2 for a, b in zip(lo, hi)]
        cases = [case_params(p["model"], *p["grid"], p["r"], p["s"], m, p["omega_xi"], U)
                 for p, m in zip(points, mids)]
        ok = run_batch(cases, steps)
        for i, good in enumerate(ok):
            if good:
                lo[i] = mids[i]
            else:
                hi[i] = mids[i]
    out = []
    for p, w in zip(points, lo):
        nu = CS2 * (1.0 / w - 0.5)
        out.append({"omega_nu_max": w, "nu_min": nu, "Re_max": U * p["grid"][0] / nu})
    return out


def study_points(name):
    pts = []
    if name == "fig8":  # CM vs RM, (r,s) = (0.75,1) on 30x40x30 and (0.5,1) on 30x60x30
        for (grid, r, s) in (((30, 40, 30), 0.75, 1.0), ((30, 60, 30), 0.5, 1.0)):
            for model in (0, 1):
                for w in (1.0, 1.2, 1.4, 1.6, 1.7, 1.8, 1.9, 1.95):
                    pts.append(dict(model=model, grid=grid, r=r, s=s, omega_nu=w, omega_xi=1.0))
    elif name == "fig9":  # omega_xi = 0.5, 1.0, 1.4 for CM on 30x60x30
        for wx in (0.5, 1.0, 1.4):
            for w in (1.0, 1.2, 1.4, 1.6, 1.7, 1.8, 1.9, 1.95):
                pts.append(dict(model=0, grid=(30, 60, 30), r=0.5, s=1.0, omega_nu=w, omega_xi=wx))
    elif name == "fig10":
        for grid in ((40, 80, 40), (50, 100, 50), (90, 180, 90)):
            for model in (0, 1):
                pts.append(dict(model=model, grid=grid, r=0.5, s=1.0, omega_xi=1.0))
    return pts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--study", choices=["fig8", "fig9", "fig10"], default="fig8")
    ap.add_argument("--steps", type=int, default=100000)
    ap.add_argument("--iters", type=int, default=7)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    pts = study_points(a.study)
    t0 = time.time()
    if a.study == "fig10":
        res = max_reynolds(pts, a.steps, iters=a.iters)
        rows = [dict(p, **r) for p, r in zip(pts, res)]
    else:
        lo, hi = bisect(pts, a.steps, iters=a.iters)
        rows = [dict(p, U_stable=l, U_unstable=h) for p, l, h in zip(pts, lo, hi)]
    out = {"study": a.study, "steps": a.steps, "cs2": CS2, "seconds": time.time() - t0, "rows": rows}
    txt = json.dumps(out, indent=1)
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as fh:
            fh.write(txt)
    print(txt)


if __name__ == "__main__":
    main()
