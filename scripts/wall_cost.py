"""Cost of the wall rules on the config-3 grid (256x256x128, r=1, s=2, fp64):
MLUPS with walls on different faces (CUDA events, 200 back-to-back steps).

  python scripts/wall_cost.py [--precision fp64|fp32]
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

PER, BB, MW, FS = 0, 1, 2, 3
CASES = {
    "periodic": (PER, PER, PER, PER, PER, PER),
    "cavity (all walls + lid)": (BB, BB, BB, MW, BB, BB),
    "walls y,z + lid": (PER, PER, BB, MW, BB, BB),
    "walls x only": (BB, BB, PER, PER, PER, PER),
    "walls y,z no lid": (PER, PER, BB, BB, BB, BB),
    "free-slip y": (PER, PER, FS, FS, PER, PER),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--streaming", choices=["ab", "aa"], default="ab")
    ap.add_argument("--case", default=None, help="run only the cases whose name starts with this")
    args = ap.parse_args()
    prec = 0 if args.precision == "fp64" else 1
    base = synth.CONFIGS["cavity100"].scaled(precision=prec)
    for name, bc in CASES.items():
        if args.case and not name.startswith(args.case):
            continue
        w = base.scaled(bc=bc)
        lat = P.Lattice(device=0, graphs=1, streaming=1 if args.streaming == "aa" else 0, **w.params())
        rho, u = synth.rest_fields(w.nx, w.ny, w.nz)
        lat.init_fields(rho, u)
        lat.step(20)
        lat.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(lat.stream)
        lat.step(args.steps)
        b.record(lat.stream)
        lat.sync()
        ms = a.elapsed_time(b) / args.steps
        print(json.dumps({"case": name, "precision": args.precision, "streaming": args.streaming, "ms_per_step": ms,
                          "mlups": w.nodes / ms / 1e3}), flush=True)
        lat.close()


if __name__ == "__main__":
    main()
