#!/usr/bin/env python
"""The five BASELINE.json configurations at FULL size on the GPU, each checked
against what its description names (SURVEY §4 layer 4):

  config 1  TGV 32x32x16 (r=1, s=2), 200 steps: velocity-amplitude and kinetic-
            energy decay vs exp(-3 nu k^2 t) / exp(-6 nu k^2 t) (reading R9)
  config 2  duct 8x128x64 (r=1, s=2), F = 1e-6, nu = 0.05, to steady state
            (reading R14): L2 error vs the Eq. 70 series (E15)
  config 3  cavity 256x256x128 (s=2), U = 0.05, Re 100 and 1000, 20k steps:
            centreline profiles vs a cubic 256^3 run of the same flow (the
            paper's cuboid-vs-cubic check)
  config 4  shear layer 512x256x512 (r=0.5, s=1), 1000 steps: mass and tangential
            momentum conserved, kinetic energy history, no blow-up
  config 5  TGV 512^3 per GPU (r=1, s=2), 500 steps: KE decay and conservation

  python -m studies.configs_physics --out results/configs_physics.json
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

import synth  # noqa: E402
from studies.analytic import duct_poiseuille  # noqa: E402


def _lat(w, **kw):
    import paper_2107_14774_b200 as P

    d = w.params()
    d.update(kw)
    return P.Lattice(**d)


def tgv_base_amplitude(u, w, nz_global=None):
    nz = w.nz if nz_global is None else nz_global
    X = 2 * np.pi * np.arange(w.nx) / w.nx
    Y = 2 * np.pi * np.arange(w.ny) / w.ny
    Z = 2 * np.pi * np.arange(nz) / nz
    basis = np.sin(X)[None, None, :] * np.cos(Y)[None, :, None] * np.cos(Z)[:, None, None]
    return float((u[0] * basis).sum() / (basis * basis).sum())


def config1():
    w = synth.CONFIGS["tgv"]
    lat = _lat(w)
    rho, u = synth.initial_fields(w)
    lat.init_fields(rho, u)
    a0 = tgv_base_amplitude(u, w)
    ke0 = lat.check()["kinetic_energy"]
    lat.step(w.steps)
    _, u1 = lat.get_macroscopic()
    d = lat.check()
    k = 2 * np.pi / 32
    t = w.steps
    return {"config": w.name, "steps": t, "amplitude_ratio": tgv_base_amplitude(u1, w) / a0,
            "amplitude_theory": float(np.exp(-3 * w.nu * k * k * t)), "ke_ratio": d["kinetic_energy"] / ke0,
            "ke_theory": float(np.exp(-6 * w.nu * k * k * t)), "mass_rel_change": None}


def config2(max_steps=600000, chunk=1000):
    w = synth.CONFIGS["duct"]
    lat = _lat(w)
    rho, u = synth.initial_fields(w)
    lat.init_fields(rho, u)
    prev = None
    steps = 0
    t0 = time.time()
    while steps < max_steps:
        lat.step(chunk)
        steps += chunk
        u = lat.get_macroscopic()[1][0]
        if prev is not None and np.abs(u - prev).max() / np.abs(u).max() < 1e-9:
            break
        prev = u
    el = time.time() - t0
    L = 128.0
    y = (np.arange(w.ny) + 0.5) * w.r - L / 2
    z = (np.arange(w.nz) + 0.5) * w.s - L / 2
    Z, Y = np.meshgrid(z, y, indexing="ij")
    ua = duct_poiseuille(Y, Z, L, w.force[0], 1.0, w.nu)
    ux = u.mean(axis=2)
    return {"config": w.name, "steps_to_steady": steps, "seconds": el,
            "l2_rel_err_vs_eq70": float(np.sqrt(((ux - ua) ** 2).sum() / (ua ** 2).sum())),
            "centre_u": float(ux[w.nz // 2 - 1:w.nz // 2 + 1, w.ny // 2 - 1:w.ny // 2 + 1].mean()),
            "centre_u_eq70": float(duct_poiseuille(0.0, 0.0, L, w.force[0], 1.0, w.nu))}


def _centrelines(u, w, U):
    def mid(a, axis):
        n = a.shape[axis]
        return 0.5 * (np.take(a, n // 2 - 1, axis=axis) + np.take(a, n // 2, axis=axis))

    uy = mid(mid(u[0], 0), 1) / U        # u_x(y) at x = L/2, z = W/2
    vx = mid(mid(u[1], 0), 0) / U        # u_y(x) at y = H/2, z = W/2
    return uy, vx


def config3(steps=20000):
    out = []
    for key in ("cavity100", "cavity1000"):
        w = synth.CONFIGS[key]
        res = {"config": w.name, "steps": steps}
        prof = {}
        for label, ww in (("cuboid", w), ("cuboid_fp32_storage", w.scaled(precision=synth.PREC_FP32)),
                          ("cubic", w.scaled(nz=256, s=1.0))):
            lat = _lat(ww)
            rho, u = synth.rest_fields(ww.nx, ww.ny, ww.nz)
            lat.init_fields(rho, u)
            m0 = lat.check()["mass"]
            t0 = time.time()
            lat.step(steps)
            _, u = lat.get_macroscopic()
            d = lat.check()
            prof[label] = _centrelines(u, ww, ww.wall_u)
            res[f"{label}_seconds"] = time.time() - t0
            res[f"{label}_mass_rel_change"] = abs(d["mass"] - m0) / m0
            lat.close()
        res["max_abs_du_over_U"] = float(np.abs(prof["cuboid"][0] - prof["cubic"][0]).max())
        res["max_abs_dv_over_U"] = float(np.abs(prof["cuboid"][1] - prof["cubic"][1]).max())
        # BASELINE config 3 asks for the fp32-storage variant too: same grid, fp32 populations
        res["fp32_vs_fp64_max_abs_du_over_U"] = float(np.abs(prof["cuboid_fp32_storage"][0] - prof["cuboid"][0]).max())
        res["fp32_vs_fp64_max_abs_dv_over_U"] = float(np.abs(prof["cuboid_fp32_storage"][1] - prof["cuboid"][1]).max())
        res["u_min_over_U_cuboid"] = float(prof["cuboid"][0].min())
        res["u_min_over_U_cubic"] = float(prof["cubic"][0].min())
        out.append(res)
    return out


def config4():
    w = synth.CONFIGS["shear"]
    lat = _lat(w)
    rho, u = synth.initial_fields(w)
    lat.init_fields(rho, u)
    d0 = lat.check()
    hist = [d0["kinetic_energy"]]
    for _ in range(10):
        lat.step(w.steps // 10)
        hist.append(lat.check()["kinetic_energy"])
    d1 = lat.check()
    return {"config": w.name, "steps": w.steps, "mass_rel_change": abs(d1["mass"] - d0["mass"]) / d0["mass"],
            "momentum_x_change_over_mass": abs(d1["momentum"][0] - d0["momentum"][0]) / d0["mass"],
            "momentum_z_change_over_mass": abs(d1["momentum"][2] - d0["momentum"][2]) / d0["mass"],
            "ke_history": hist, "bad_nodes": d1["bad_nodes"], "max_speed": d1["max_speed"]}


def config5():
    import torch

    w = synth.CONFIGS["weak"]
    lat = _lat(w)
    rho, u = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0, xp=torch, device="cuda")
    lat.init_fields(rho, u)
    del rho, u
    d0 = lat.check()
    lat.step(w.steps)
    d1 = lat.check()
    # wave numbers: x and y one period over 512 nodes; z one period over 512 nodes of spacing s = 2
    k2 = (2 * np.pi / 512) ** 2 * 2 + (2 * np.pi / (512 * w.s)) ** 2
    return {"config": w.name, "steps": w.steps, "ke_ratio": d1["kinetic_energy"] / d0["kinetic_energy"],
            "ke_theory_linear": float(np.exp(-2 * w.nu * k2 * w.steps)),
            "mass_rel_change": abs(d1["mass"] - d0["mass"]) / d0["mass"],
            "momentum_over_mass": [abs(x) / d0["mass"] for x in d1["momentum"]], "bad_nodes": d1["bad_nodes"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default="1,2,3,4,5")
    a = ap.parse_args()
    fns = {"1": config1, "2": config2, "3": config3, "4": config4, "5": config5}
    res = {}
    for k in a.only.split(","):
        t0 = time.time()
        res[f"config{k}"] = fns[k]()
        print(f"config{k}: {time.time() - t0:.1f} s", flush=True)
    txt = json.dumps(res, indent=1, default=float)
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        open(a.out, "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main()
