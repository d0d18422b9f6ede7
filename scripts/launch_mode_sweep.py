"""MLUPS of the three single-GPU launch modes of step(n) across lattice sizes
(include/lbm_cuboid.h `graphs`: 1 one launch per step, 2 CUDA graphs of 32
steps, 3 persistent cooperative kernel).  TGV physics of config 1 (r=1, s=2,
nu=0.01), fp64 and fp32 storage; CUDA events on the library's compute stream
around step(n) after a warm-up.  Writes one JSON line per (grid, precision, mode).

  python scripts/launch_mode_sweep.py [--out gpurun_out/launch_modes.jsonl]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2107_14774_b200 as P  # noqa: E402
import synth  # noqa: E402

GRIDS = [(32, 32, 16), (30, 60, 30), (8, 128, 64), (64, 64, 32), (104, 64, 40), (96, 64, 64),
         (128, 128, 64), (256, 64, 128), (256, 256, 64), (256, 256, 128)]


def run(nx, ny, nz, prec, mode, budget_nodes=4e9):
    w = synth.CONFIGS["tgv"].scaled(nx=nx, ny=ny, nz=nz, precision=prec)
    lat = P.Lattice(device=0, graphs=mode, **w.params())
    rho, u = synth.initial_fields(w)
    lat.init_fields(rho, u)
    steps = int(max(64, min(20000, budget_nodes / w.nodes)))
    steps -= steps % 64
    lat.step(64)
    lat.sync()
    s = lat.stream
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    lat.step(steps)
    b.record(s)
    lat.sync()
    ms = a.elapsed_time(b)
    bad = lat.check(raise_on_unstable=False)["bad_nodes"]
    lat.close()
    return {"grid": [nx, ny, nz], "nodes": w.nodes, "precision": "fp64" if prec == 0 else "fp32",
            "mode": {1: "launch/step", 2: "graphs", 3: "persistent"}[mode], "steps": steps,
            "us_per_step": 1e3 * ms / steps, "mlups": w.nodes * steps / (ms * 1e-3) / 1e6, "bad_nodes": bad}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "launch_modes.jsonl"))
    args = ap.parse_args()
    with open(args.out, "w") as fh:
        for prec in (0, 1):
            for g in GRIDS:
                for mode in (1, 2, 3):
                    r = run(*g, prec, mode)
                    print(json.dumps(r), flush=True)
                    fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
