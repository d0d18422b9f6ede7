"""Long runs of the config-1 Taylor-Green vortex (32x32x16, r = 1, s = 2,
nu = 0.01) to observe the weak linear instability found by the von Neumann
analysis (tests/linear_stability.py): omega_xi = 1 (the
paper's setting) vs omega_xi = omega_nu.  Prints max |u| and the energy of the
z-Nyquist content (u_z alternating sign plane to plane) over time."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2107_14774_b200 as P  # noqa: E402
import synth  # noqa: E402


def nyquist_z(u):
    """amplitude of the z-Nyquist component of all velocity components"""
    sign = (-1.0) ** np.arange(u.shape[1])[None, :, None, None]
    return float(np.abs((u * sign).mean(axis=1)).max())


def main():
    w0 = synth.CONFIGS["tgv"]
    out = []
    for label, oxi in (("omega_xi=1", 1.0), ("omega_xi=omega_nu", w0.omega_nu)):
        w = w0.scaled(omega_xi=oxi)
        lat = P.Lattice(device=0, **w.params())
        rho, u = synth.initial_fields(w)
        lat.init_fields(rho, u)
        t = 0
        for target in (200, 1000, 2000, 5000, 10000, 20000, 40000):
            lat.step(target - t)
            t = target
            d = lat.check(raise_on_unstable=False)
            _, uu = lat.get_macroscopic()
            rec = {"case": label, "steps": t, "max_speed": d["max_speed"], "kinetic_energy": d["kinetic_energy"],
                   "nyquist_z": nyquist_z(uu), "bad_nodes": d["bad_nodes"]}
            print(json.dumps(rec), flush=True)
            out.append(rec)
            if d["bad_nodes"]:
                break
        lat.close()


if __name__ == "__main__":
    main()
