#!/usr/bin/env python
"""Pulsatile square-duct flow of PAPER.md L804-853 on the GPU, against the
Womersley series (studies/analytic.py, erratum E14 form).

2a = 40, F_m = 1e-5, T = 10,000, Wo in {3.09, 6.25}; grids 40x80x40 (r,s) =
(0.5,1), 40x80x80 (0.5,0.5), 40x160x80 (0.25,0.5); cs2 = min(1,r^2,s^2)/3;
nu = a^2 omega / Wo^2.  The force is updated every step through
lbm_cuboid_set_force (F_x = F_m cos(omega t_n) for the collision producing t_n).
Enough periods for the start-up transient to decay below 1e-3 (3 at Wo = 3.09,
9 at Wo = 6.25); L2 error of u_x over the cross-section at four phases of the
last period.

  python -m studies.womersley --out results/womersley.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from studies.analytic import womersley  # noqa: E402

GRIDS = [((40, 80, 40), 0.5, 1.0), ((40, 80, 80), 0.5, 0.5), ((40, 160, 80), 0.25, 0.5)]


def transient_periods(a, nu, T, tol=1e-3):
    """Periods to wait until the slowest homogeneous duct mode, decaying at
    nu ((pi/2a)^2 + (pi/2a)^2) per step, is below tol; plus the measured one."""
    rate = 2.0 * nu * (np.pi / (2.0 * a)) ** 2
    return int(np.ceil(np.log(1.0 / tol) / rate / T)) + 1


def run_case(grid, r, s, Wo, T=10000, periods=None, twoa=40.0, Fm=1e-5, model=0):
    import paper_2107_14774_b200 as P
    import synth

    nx, ny, nz = grid
    a = twoa / 2
    om = 2 * np.pi / T
    nu = a * a * om / Wo ** 2
    cs2 = synth.auto_cs2(r, s)
    if periods is None:
        periods = max(3, transient_periods(a, nu, T))
    lat = P.Lattice(nx, ny, nz, r, s, cs2=cs2, omega_nu=synth.omega_from_nu(nu, cs2),
                    bc=(0, 0, 1, 1, 1, 1), model=model)
    lat.init_fields(np.ones((nz, ny, nx)), np.zeros((3, nz, ny, nx)))
    y = (np.arange(ny) + 0.5) * r - a
    z = (np.arange(nz) + 0.5) * s - a
    Z, Y = np.meshgrid(z, y, indexing="ij")
    nsteps = periods * T
    errs, phases = [], []
    t0 = time.time()
    for n in range(1, nsteps + 1):
        lat.set_force((Fm * np.cos(om * n), 0.0, 0.0))
        lat.step(1)
        if n > nsteps - T and (nsteps - n) % (T // 4) == 0:
            u = lat.get_macroscopic()[1][0].mean(axis=2)  # x-average (uniform along the duct)
            ua = womersley(Y, Z, n, a, Fm, om, nu)
            errs.append(float(np.sqrt(((u - ua) ** 2).sum() / (ua ** 2).sum())))
            phases.append(float((n % T) / T))
            umax = float(np.abs(ua).max())
    lat.sync()
    el = time.time() - t0
    lat.close()
    return {"grid": list(grid), "r": r, "s": s, "Wo": Wo, "nu": nu, "cs2": cs2, "model": model,
            "steps": nsteps, "seconds": el, "phases": phases, "l2_rel_err": errs, "u_amplitude": umax}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--periods", type=int, default=None, help="default: enough for the start-up transient")
    a = ap.parse_args()
    rows = [run_case(g, r, s, Wo, periods=a.periods) for (g, r, s) in GRIDS for Wo in (3.09, 6.25)]
    txt = json.dumps({"study": "womersley", "rows": rows}, indent=1)
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        open(a.out, "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main()
