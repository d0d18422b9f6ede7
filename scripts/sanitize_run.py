#!/usr/bin/env python
"""Exercise every kernel of liblbm_cuboid.so on small grids (for compute-sanitizer
or the -DLBM_DEBUG_BOUNDS build): init (host and device), collide-stream
(paper-rate, generic, raw; fp64 and fp32), FULL_FD fused and two-pass, all wall
kinds, ghost-plane NCCL self-exchange, fused P2P halo (self and two in-process
slabs), graphs, the persistent kernel, AA, macro, pack/unpack, check; round 2:
FULL_FD_LAG (all paths), the TMA-staged FULL_FD kernel, the opt-in TMA and
x-pair kernels, the event trace."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_14774_b200 as P  # noqa: E402
import synth  # noqa: E402

cases = [
    synth.CONFIGS["tgv"].scaled(nx=19, ny=13, nz=6),
    synth.CONFIGS["cavity100"].scaled(nx=11, ny=9, nz=5),
    synth.CONFIGS["shear"].scaled(nx=8, ny=12, nz=6),
    synth.CONFIGS["duct"].scaled(nx=3, ny=10, nz=7),
    synth.Workload("generic", 9, 7, 5, r=0.75, s=1.3, nu=0.02, omega_1=1.2, omega_high=0.9, init="random"),
    synth.CONFIGS["tgv"].scaled(nx=7, ny=6, nz=5, corrections=synth.CORR_FULL_FD),
    synth.CONFIGS["cavity100"].scaled(nx=6, ny=7, nz=4, corrections=synth.CORR_FULL_FD),
    synth.CONFIGS["tgv"].scaled(nx=7, ny=6, nz=6, corrections=synth.CORR_FULL_FD_LAG),
    synth.CONFIGS["cavity100"].scaled(nx=6, ny=7, nz=4, corrections=synth.CORR_FULL_FD_LAG),
]
FD_MODES = (synth.CORR_FULL_FD, synth.CORR_FULL_FD_LAG)
for w in cases:
    for prec in (0, 1):
        for model in (0, 1):
            ww = w.scaled(precision=prec, model=model)
            for kw in ({}, {"halo": 1, "nccl_uid": P.nccl_unique_id()}, {"graphs": 2}, {"streaming": 1},
                       {"streaming": 1, "graphs": 2}, {"halo": 2}, {"graphs": 3}, {"fd_two_pass": 1}):
                if kw.get("halo") and ww.bc[4] != 0:
                    continue
                if "streaming" in kw and ww.corrections in FD_MODES:
                    continue
                if "fd_two_pass" in kw:
                    if ww.corrections != synth.CORR_FULL_FD:
                        continue
                    kw = {}
                    os.environ["LBM_FD_FUSED"] = "0"
                g = P.Lattice(**ww.params(), **kw)
                rho, u = synth.random_fields(ww.nx, ww.ny, ww.nz, 5)
                g.init_fields(rho, u)
                g.step(35)
                f = g.get_populations()
                g.set_populations(f)
                g.init_fields(torch.from_numpy(rho).cuda(), torch.from_numpy(u).cuda())
                g.step(3)
                g.get_macroscopic()
                g.get_macroscopic(device=True)
                g.get_populations_planes(1, 2)
                g.check()
                g.timing(True)
                g.step(2)
                g.timing_read()
                g.timing(False)
                g.sync()
                g.close()
                os.environ.pop("LBM_FD_FUSED", None)
            # two P2P slabs in this process, stepped one at a time (remote ghost stores)
            if ww.nz % 2 == 0 and ww.corrections != synth.CORR_FULL_FD:  # FULL_FD_LAG included
                hs = [P.Lattice(**ww.params(), rank=r, world=2, halo=2) for r in range(2)]
                blobs = [h.p2p_export() for h in hs]
                for h in hs:
                    h.p2p_connect(*P.lbm.p2p_neighbour_blobs(P.lbm.halo_plan(h.p), blobs))
                rho, u = synth.random_fields(ww.nx, ww.ny, ww.nz, 6)
                n = ww.nz // 2
                for r, h in enumerate(hs):
                    h.init_fields(np.ascontiguousarray(rho[r * n:(r + 1) * n]),
                                  np.ascontiguousarray(u[:, r * n:(r + 1) * n]))
                    h.sync()
                for _ in range(5):
                    for h in hs:
                        h.step(1)
                        h.sync()
                for h in hs:
                    h.close()
# opt-in kernels: TMA-staged (rows of >= 128 nodes) and x-pair (fp32, nx even), with walls
# and periodic faces, plus the event trace
for env, ws in (("LBM_TMA", [synth.CONFIGS["tgv"].scaled(nx=136, ny=5, nz=4),
                             synth.CONFIGS["cavity100"].scaled(nx=128, ny=5, nz=4)]),
                ("LBM_XPAIR", [synth.CONFIGS["tgv"].scaled(nx=70, ny=5, nz=4, precision=1),
                               synth.CONFIGS["cavity100"].scaled(nx=66, ny=5, nz=4, precision=1)])):
    os.environ[env] = "1"
    for w in ws:
        for prec in ((0, 1) if env == "LBM_TMA" else (1,)):
            g = P.Lattice(**w.scaled(precision=prec).params())
            rho, u = synth.random_fields(w.nx, w.ny, w.nz, 7)
            g.init_fields(rho, u)
            g.trace(True)
            g.step(6)
            g.trace_read()
            g.trace(False)
            g.sync()
            g.close()
    os.environ.pop(env)
# the TMA-staged FULL_FD kernel: staged, x-seam and LDG-body tiles, x/y walls with
# periodic z, the NCCL ghost path and a 2-plane slab
os.environ["LBM_FD_TMA"] = "1"
for w, kw in ((synth.CONFIGS["tgv"].scaled(nx=96, ny=20, nz=6, corrections=3), {}),
              (synth.CONFIGS["tgv"].scaled(nx=96, ny=20, nz=6, corrections=3), {"halo": P.HALO_NCCL}),
              (synth.CONFIGS["tgv"].scaled(nx=64, ny=16, nz=2, corrections=3), {"halo": P.HALO_NCCL}),
              (synth.CONFIGS["cavity100"].scaled(nx=100, ny=18, nz=5, corrections=3, bc=(1, 1, 1, 2, 0, 0)), {})):
    for prec in (0, 1):
        if "halo" in kw:
            kw = dict(kw, nccl_uid=P.nccl_unique_id())
        g = P.Lattice(**w.scaled(precision=prec).params(), **kw)
        assert "fd_tma" in g.kernel_name(), g.kernel_name()
        rho, u = synth.random_fields(w.nx, w.ny, w.nz, 7)
        g.init_fields(rho, u)
        g.step(6)
        g.sync()
        g.close()
os.environ.pop("LBM_FD_TMA")
torch.cuda.synchronize()
print("sanitize_run: all kernels exercised")
