#!/usr/bin/env python
"""Cuboid-vs-cubic cost study of PAPER.md §6 on the GPU.

Lid-driven shallow cavity L/H = 4, W/H = 2, Re = U L / nu = 100, N_y = 64:
  cubic 256x64x128 (r = s = 1, cs2 = 1/3) and the cuboid grids
  (i) 104x64x40 (0.406, 1.3), (ii) 96x64x64 (0.375, 0.75), (iii) 96x64x48 (0.375, 1.0)
with cs2 = 0.04.  The lid speed is U = 0.05 lattice units on every grid,
so one step covers a physical time proportional to dx and the cuboid runs need
N_x/256 of the cubic run's steps for the same physical time.  Reported: nodes,
memory, GPU time per step and to solution, and the centreline profiles
u(y) at x = L/2, z = W/2 and v(x) at y = H/2, z = W/2 (Fig. 6) compared with the
cubic run.  The paper quotes only the memory ratios (7.88, 5.33, 7.11) and
"about similar reductions" in turnaround time, on unstated hardware.

  python -m studies.shallow_cavity --out results/shallow_cavity.json
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

CASES = [("cubic", (256, 64, 128), 1.0, 1.0, 1.0 / 3.0),
         ("cuboid-i", (104, 64, 40), 0.406, 1.3, 0.04),
         ("cuboid-ii", (96, 64, 64), 0.375, 0.75, 0.04),
         ("cuboid-iii", (96, 64, 48), 0.375, 1.0, 0.04)]
U = 0.05
RE = 100.0


def centre_avg(a, axis):
    n = a.shape[axis]
    if n % 2:
        return np.take(a, n // 2, axis=axis)
    return 0.5 * (np.take(a, n // 2 - 1, axis=axis) + np.take(a, n // 2, axis=axis))


def run_case(name, grid, r, s, cs2, cubic_steps, chunks=8):
    import torch

    import paper_2107_14774_b200 as P
    import synth

    nx, ny, nz = grid
    nu = U * nx / RE  # L = nx in x units
    steps = int(round(cubic_steps * nx / 256))
    lat = P.Lattice(nx, ny, nz, r, s, cs2=cs2, omega_nu=synth.omega_from_nu(nu, cs2),
                    bc=(1, 1, 1, 2, 1, 1), wall_u=U)
    lat.init_fields(np.ones((nz, ny, nx)), np.zeros((3, nz, ny, nx)))
    stream = lat.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hist = []
    prev = None
    done = 0
    e0.record(stream)
    for c in range(chunks):
        n = steps // chunks if c < chunks - 1 else steps - done
        lat.step(n)
        done += n
        if c >= chunks - 2:
            rho, u = lat.get_macroscopic()
            if prev is not None:
                hist.append(float(np.abs(u - prev).max() / U))
            prev = u
    e1.record(stream)
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1)
    # short timing run for the per-step cost (graphs on, no host reads)
    lat.sync()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    lat.step(512)
    t1.record(stream)
    torch.cuda.synchronize()
    ms_step = t0.elapsed_time(t1) / 512
    rho, u = lat.get_macroscopic()
    d = lat.check()
    lat.close()
    # u_x along y at x = L/2, z = W/2 ; u_y along x at y = H/2, z = W/2
    uy_prof = centre_avg(centre_avg(u[0], 0), 1) / U      # over y
    vx_prof = centre_avg(centre_avg(u[1], 0), 0) / U      # over x
    yc = (np.arange(ny) + 0.5) / ny
    xc = (np.arange(nx) + 0.5) / nx
    return {"name": name, "grid": list(grid), "r": r, "s": s, "cs2": cs2, "nu": nu, "nodes": nx * ny * nz,
            "bytes_fp64_two_buffers": 2 * 27 * 8 * nx * ny * (nz + 2), "steps": steps,
            "gpu_ms_total": gpu_ms, "ms_per_step": ms_step, "mlups": nx * ny * nz / ms_step / 1e3,
            "last_chunk_change_over_U": hist[-1] if hist else None, "max_speed_over_U": d["max_speed"] / U,
            "y": yc.tolist(), "u_of_y": uy_prof.tolist(), "x": xc.tolist(), "v_of_x": vx_prof.tolist()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cubic-steps", type=int, default=120000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = [run_case(n, g, r, s, c, a.cubic_steps) for (n, g, r, s, c) in CASES]
    ref = rows[0]
    for row in rows[1:]:
        du = np.interp(row["y"], ref["y"], ref["u_of_y"]) - np.array(row["u_of_y"])
        dv = np.interp(row["x"], ref["x"], ref["v_of_x"]) - np.array(row["v_of_x"])
        row["max_abs_du_vs_cubic"] = float(np.abs(du).max())
        row["max_abs_dv_vs_cubic"] = float(np.abs(dv).max())
        row["memory_ratio_cubic_over_this"] = ref["bytes_fp64_two_buffers"] / row["bytes_fp64_two_buffers"]
        row["node_ratio_cubic_over_this"] = ref["nodes"] / row["nodes"]
        row["time_per_step_ratio"] = ref["ms_per_step"] / row["ms_per_step"]
        row["time_to_solution_ratio"] = ref["gpu_ms_total"] / row["gpu_ms_total"]
    txt = json.dumps({"study": "shallow_cavity", "U": U, "Re": RE, "rows": rows}, indent=1)
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        open(a.out, "w").write(txt)
    summary = [{k: v for k, v in r.items() if k not in ("y", "x", "u_of_y", "v_of_x")} for r in rows]
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
