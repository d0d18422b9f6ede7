"""One-off full-size parity run ("100 steps at full size where
the oracle finishes in <= 30 min"): BASELINE config 3 (cavity, 256x256x128,
r = 1, s = 2, six walls with the Eq. 69 lid) from seeded rough fields, 100
steps on the CPU oracle (single thread, ~20 min) and on the GPU through the C
ABI, every one of the 226 M populations compared.  Test infrastructure (drives
the oracle); run under gpurun:

  python -m tests.full_size_parity [--workload cavity1000] [--steps 100] [--precisions 0,1] [--out results/full_size_parity.json]
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
    ap.add_argument("--precisions", default="0", help="comma list: 0 fp64, 1 fp32 storage (one oracle run)")
    ap.add_argument("--out", default=os.path.join(ROOT, "results", "full_size_parity.json"),
                    help="fp64 result file; fp32 goes to the same name with _fp32")
    args = ap.parse_args()
    w0 = synth.CONFIGS[args.workload]
    rho, u = synth.random_fields(w0.nx, w0.ny, w0.nz, 2024)
    gpu = {}
    for prec in [int(p) for p in args.precisions.split(",")]:
        w = w0.scaled(precision=prec)
        g = P.Lattice(**w.params())
        g.init_fields(rho, u)
        t0 = time.time()
        g.step(args.steps)
        g.sync()
        gpu[prec] = (g.get_populations(), time.time() - t0)
        g.close()
    o = O.Oracle(**w0.params())
    o.init_fields(rho, u)
    t0 = time.time()
    o.step(args.steps)
    t_cpu = time.time() - t0
    fo = o.get_populations()
    ok = True
    for prec, (fg, t_gpu) in gpu.items():
        d = np.abs(fg - fo)
        res = {"workload": w0.name, "grid": [w0.nx, w0.ny, w0.nz], "steps": args.steps, "precision": prec,
               "populations_compared": int(fo.size), "max_abs_diff": float(d.max()),
               "max_rel_diff": float((d / np.abs(fo)).max()), "max_abs_f": float(np.abs(fo).max()),
               "oracle_seconds": t_cpu, "gpu_seconds": t_gpu}
        print(json.dumps(res), flush=True)
        out = args.out if prec == 0 else args.out.replace(".json", "_fp32.json")
        with open(out, "w") as fh:
            json.dump(res, fh, indent=1)
        bar = 1e-12 if prec == 0 else 1e-5
        ok = ok and (res["max_abs_diff"] if prec == 0 else res["max_rel_diff"]) <= bar
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
