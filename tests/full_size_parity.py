"""One-off full-size parity run ("100 steps at full size where
the oracle finishes in <= 30 min"): BASELINE config 3 (cavity, 256x256x128,
r = 1, s = 2, six walls with the Eq. 69 lid) from seeded rough fields, 100
steps on the CPU oracle (single thread, ~20 min) and on the GPU through the C
ABI, every one of the 226 M populations compared.  Test infrastructure (drives
the oracle); run under gpurun:

  python -m tests.full_size_parity [--workload cavity1000] [--steps 100] [--out results/full_size_parity.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2107_14774_b200 as P  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cavity1000")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--precision", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "results", "full_size_parity.json"))
    args = ap.parse_args()
    w = synth.CONFIGS[args.workload].scaled(precision=args.precision)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 2024)
    g = P.Lattice(**w.params())
    g.init_fields(rho, u)
    t0 = time.time()
    g.step(args.steps)
    g.sync()
    t_gpu = time.time() - t0
    fg = g.get_populations()
    g.close()
    o = O.Oracle(**w.params())
    o.init_fields(rho, u)
    t0 = time.time()
    o.step(args.steps)
    t_cpu = time.time() - t0
    fo = o.get_populations()
    d = np.abs(fg - fo)
    res = {"workload": w.name, "grid": [w.nx, w.ny, w.nz], "steps": args.steps, "precision": args.precision,
           "populations_compared": int(fo.size), "max_abs_diff": float(d.max()),
           "max_rel_diff": float((d / np.abs(fo)).max()), "max_abs_f": float(np.abs(fo).max()),
           "oracle_seconds": t_cpu, "gpu_seconds": t_gpu}
    print(json.dumps(res), flush=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
    bar = 1e-12 if args.precision == 0 else 1e-5
    metric = res["max_abs_diff"] if args.precision == 0 else res["max_rel_diff"]
    sys.exit(0 if metric <= bar else 1)


if __name__ == "__main__":
    main()
