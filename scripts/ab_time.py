"""A/B timing of two builds of the library on the bench workload (512^3 TGV):
python scripts/ab_time.py <package root> <fp64|fp32> <steps>"""
import os
import sys

root = os.path.abspath(sys.argv[1])
sys.path.insert(0, root)
import torch  # noqa: E402

import paper_2107_14774_b200 as P  # noqa: E402
import synth  # noqa: E402

prec, steps = sys.argv[2], int(sys.argv[3])
w = synth.CONFIGS["weak"].scaled(precision=0 if prec == "fp64" else 1)
g = P.Lattice(**w.params())
rho, u = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0, xp=torch, device=torch.device("cuda", 0))
g.init_fields(rho, u)
torch.cuda.synchronize()
with torch.cuda.stream(g.stream):
    g.step(5)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(g.stream)
g.step(steps)
b.record(g.stream)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / steps
print(f"{os.path.basename(root) or 'repo'} {prec} {steps} steps: {ms:.3f} ms/step {w.nodes / ms / 1e3:.0f} MLUPS", flush=True)
