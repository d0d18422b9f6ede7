"""MLUPS of every collide-stream kernel variant on one lattice (default the
bench's 512^3 config-5 TGV, periodic), CUDA events over back-to-back steps:
model (CM / RM) x rates (paper omega_1 = omega_high = 1 / generic) x
corrections (FULL_LOCAL / FULL_FD) x storage (fp64 / fp32) x streaming (AB / AA).

  python scripts/kernel_matrix.py [--nz 512] [--steps 20]
"""
import argparse
import itertools
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2107_14774_b200 as P  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nz", type=int, default=512)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    base = synth.CONFIGS["weak"].scaled(nz=args.nz)
    for model, rates, corr, prec, aa in itertools.product((0, 1), ("paper", "generic"), (0, 3), (0, 1), (0, 1)):
        if corr == 3 and aa:
            continue
        w = base.scaled(model=model, corrections=corr, precision=prec,
                        omega_1=1.0 if rates == "paper" else 1.2, omega_high=1.0 if rates == "paper" else 1.1)
        lat = P.Lattice(device=0, graphs=1, streaming=aa, **w.params())
        rho, u = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0, xp=torch, device="cuda")
        lat.init_fields(rho, u)
        del rho, u
        lat.step(4)
        lat.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(lat.stream)
        lat.step(args.steps)
        b.record(lat.stream)
        lat.sync()
        ms = a.elapsed_time(b) / args.steps
        bpn = lat.info()["bytes_per_node_update"]
        print(json.dumps({"model": "RM" if model else "CM", "rates": rates,
                          "corrections": "FULL_FD" if corr == 3 else "FULL_LOCAL",
                          "storage": "fp32" if prec else "fp64", "streaming": "AA" if aa else "AB",
                          "ms_per_step": round(ms, 4), "mlups": round(w.nodes / ms / 1e3),
                          "hbm_frac": round(bpn * w.nodes / (ms * 1e-3) / 6543.4e9, 3)}), flush=True)
        lat.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
