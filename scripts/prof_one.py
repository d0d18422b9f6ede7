"""One small run for ncu captures: 512 x 512 x 64 periodic TGV slab (config-5
physics), 3 steps.  python scripts/prof_one.py [fp64|fp32] [corrections]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_14774_b200 as P  # noqa: E402
import synth  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
corr = sys.argv[2] if len(sys.argv) > 2 else "full_local"
c = {"full_local": 0, "full_fd": 3, "full_fd_lag": 4}[corr]
w = synth.CONFIGS["weak"].scaled(nz=64, precision=0 if prec == "fp64" else 1, corrections=c)
g = P.Lattice(**w.params(), graphs=1)
rho, u = synth.initial_fields(w)
g.init_fields(rho, u)
g.step(3)
g.sync()
print("ok", prec, corr)
