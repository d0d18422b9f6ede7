"""Linear (von Neumann) stability of the 3DCCM-LBM at the BASELINE configs,
computed on the CPU oracle (builder action (i)).  Test
infrastructure (it drives the oracle): the pins are in
test_oracle_linear_stability.py; `python -m tests.linear_stability` writes
results/linear_stability.json.

The update is linearised about a uniform equilibrium f^eq(rho = 1, U): J is the
Jacobian of the oracle's collision (central differences, 27 x 27), and a Fourier
mode exp(i kappa . x) of the pull-streamed update f(x, t+1) = f~(x - e, t) is
amplified by G(kappa) = diag(exp(-i kappa . e_a)) J, with e_a the integer index
displacements and kappa in index space (the physical wavenumber along y is
kappa_y / r, along z kappa_z / s).  The scheme is linearly stable when every
eigenvalue of G has modulus <= 1 for every kappa.

  python -m tests.linear_stability [--n 25] [--out results/linear_stability.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (the study runs on the oracle)
import synth  # noqa: E402

E_INDEX = O.velocities(1.0, 1.0).round()  # index displacements, paper order


def collision_jacobian(o: "O.Oracle", r: float, s: float, U=(0.0, 0.0, 0.0), h: float = 1e-7) -> np.ndarray:
    """d f~ / d f of the oracle's collision at f^eq(1, U) (central differences)."""
    f0 = o.feq(1.0, np.asarray(U, dtype=np.float64))
    J = np.zeros((27, 27))
    for b in range(27):
        e = np.zeros(27)
        e[b] = h
        J[:, b] = (o.collide(f0 + e) - o.collide(f0 - e)) / (2 * h)
    return J


def eigenvalues(J: np.ndarray, kappa: np.ndarray) -> np.ndarray:
    """Eigenvalues of G(kappa) = diag(exp(-i kappa . e)) J for kappa of shape (n, 3)."""
    ph = np.exp(-1j * (np.atleast_2d(kappa) @ E_INDEX.T))
    return np.linalg.eigvals(ph[:, :, None] * J[None, :, :])


def max_growth(J: np.ndarray, n: int = 25):
    """max |lambda| over the n^3 grid kappa_d = -pi + 2 pi k/n (n odd: contains the
    Nyquist wavenumber -pi, never kappa = 0, whose conserved modes have |lambda| = 1)
    and the wavenumber where it occurs."""
    if n % 2 == 0:
        raise ValueError("n must be odd")
    ks = np.linspace(-np.pi, np.pi, n, endpoint=False)
    K = np.stack(np.meshgrid(ks, ks, ks, indexing="ij"), -1).reshape(-1, 3)
    a = np.abs(eigenvalues(J, K)).max(axis=1)
    i = int(a.argmax())
    return float(a[i]), K[i]


def lattice(r, s, nu, omega_xi=1.0, corrections=synth.CORR_FULL_LOCAL, model=0, cs2=None):
    cs2 = synth.auto_cs2(r, s) if cs2 is None else cs2
    return O.Oracle(2, 2, 2, r, s, cs2, synth.omega_from_nu(nu, cs2), omega_xi=omega_xi,
                    corrections=corrections, model=model), cs2


CASES = {
    # BASELINE configs (readings R2, R3, R15): omega_xi = 1, FULL_LOCAL
    "config1_5_tgv": dict(r=1.0, s=2.0, nu=0.01),
    "config2_duct": dict(r=1.0, s=2.0, nu=0.05),
    "config3_cavity_re100": dict(r=1.0, s=2.0, nu=0.128),
    "config3_cavity_re1000": dict(r=1.0, s=2.0, nu=0.0128),
    "config4_shear_layer": dict(r=0.5, s=1.0, nu=0.01),
    # P13 variations of configs 1/5
    "config1_5_omega_xi_eq_omega_nu": dict(r=1.0, s=2.0, nu=0.01, omega_xi="omega_nu"),
    "config1_5_corrections_off": dict(r=1.0, s=2.0, nu=0.01, corrections=synth.CORR_OFF),
}


def run_case(name, n=25, U=(0.0, 0.0, 0.0)):
    kw = dict(CASES[name])
    if kw.get("omega_xi") == "omega_nu":
        cs2 = synth.auto_cs2(kw["r"], kw["s"])
        kw["omega_xi"] = synth.omega_from_nu(kw["nu"], cs2)
    o, cs2 = lattice(**kw)
    J = collision_jacobian(o, kw["r"], kw["s"], U)
    m, k = max_growth(J, n)
    return {"case": name, **{k2: v for k2, v in kw.items()}, "cs2": cs2, "U": list(U), "grid": n,
            "max_abs_lambda": m, "at_kappa": [float(x) for x in k]}


def max_stable_speed(r, s, cs2, omega_nu, model, omega_xi=1.0, n=15, du=0.025, u_max=0.6):
    """Largest uniform speed U along x (steps of du) for which the linearised
    update is stable on an n^3 grid (None if unstable at rest): the linear
    counterpart of the paper's section-7 robustness study."""
    o = O.Oracle(2, 2, 2, r, s, cs2, omega_nu, omega_xi=omega_xi, corrections=synth.CORR_FULL_LOCAL, model=model)
    best = None
    for U in np.arange(0.0, u_max + 1e-12, du):
        m, _ = max_growth(collision_jacobian(o, r, s, (float(U), 0.0, 0.0)), n)
        if m > 1.0 + 1e-9:
            break
        best = float(U)
    return best


def main_mean_flow(out):
    rows = []
    for model in (0, 1):
        for wn in (1.0, 1.4, 1.6, 1.8, 1.9):
            u = max_stable_speed(0.5, 1.0, 0.08, wn, model)
            rows.append({"model": "3DCRM" if model else "3DCCM", "r": 0.5, "s": 1.0, "cs2": 0.08, "omega_nu": wn,
                         "omega_xi": 1.0, "max_linearly_stable_U": u})
            print(json.dumps(rows[-1]), flush=True)
    with open(out, "w") as fh:
        json.dump(rows, fh, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=25)
    ap.add_argument("--out", default=os.path.join(ROOT, "results", "linear_stability.json"))
    ap.add_argument("--mean-flow", action="store_true",
                    help="max linearly stable uniform speed, CM vs RM (section-7 setting)")
    args = ap.parse_args()
    if args.mean_flow:
        main_mean_flow(os.path.join(ROOT, "results", "linear_stability_mean_flow.json"))
        return
    res = [run_case(c, args.n) for c in CASES]
    res += [run_case(c, args.n, U=(0.05, 0.0, 0.0)) for c in ("config3_cavity_re1000", "config4_shear_layer")]
    for r in res:
        print(json.dumps(r))
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
