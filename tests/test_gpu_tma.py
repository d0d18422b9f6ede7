"""The TMA-staged collide-stream kernel (csrc/cm_tma.cuh: 27 cp.async.bulk.tensor
boxes per 128-node row tile, mbarrier ring, one producer warp) against the
one-node-per-thread kernel (LBM_TMA=0) on the same inputs, after 21 steps.

Geometries cover every branch of the TMA kernel: periodic x (the 16-byte wrap
boxes at both row ends), rows that are not a multiple of the tile (ragged
last tile), several tiles per row, wall warps (the out-of-line gather path),
free-slip, the moving lid, periodic y/z wrap of the box coordinates, the
NCCL ghost-plane path (strided boundary planes, ghost-plane boxes), generic
rates, the raw-moment model, fp64 and fp32 storage.  The two kernels inline
the same per-node arithmetic; where ptxas fuses a multiply-add differently
the results differ by rounding only: max|df| <= 1e-14 (fp64), relative
<= 1e-6 (fp32).  (Oracle parity of the TMA kernel: test_gpu_fastpath.py.)
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2107_14774_b200 as P

    P.load()
    return P


CASES = {
    "tgv_2tiles": (synth.CONFIGS["tgv"].scaled(nx=256, ny=9, nz=6), {}),
    "tgv_ragged": (synth.CONFIGS["tgv"].scaled(nx=200, ny=7, nz=5), {}),
    "tgv_one_tile": (synth.CONFIGS["tgv"].scaled(nx=128, ny=5, nz=4), {}),
    "cavity_lid": (synth.CONFIGS["cavity100"].scaled(nx=136, ny=10, nz=6), {}),
    "shear_slip_raw": (synth.CONFIGS["shear"].scaled(nx=132, ny=12, nz=6), {"model": 1}),
    "duct_generic_force": (synth.CONFIGS["duct"].scaled(nx=140, ny=10, nz=8),
                           {"omega_1": 1.2, "omega_high": 0.9, "force": (1e-5, -2e-6, 3e-6)}),
}


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("case", list(CASES))
def test_tma_kernel_matches_node_kernel(P, case, prec, monkeypatch):
    w, kw = CASES[case]
    w = w.scaled(precision=prec)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 93)
    monkeypatch.setenv("LBM_TMA", "0")
    a = P.Lattice(**dict(w.params(), **kw), graphs=1)
    monkeypatch.setenv("LBM_TMA", "1")
    hs = [P.Lattice(**dict(w.params(), **kw), graphs=1), P.Lattice(**dict(w.params(), **kw), graphs=2)]
    if w.bc[4] == synth.BC_PERIODIC:
        hs.append(P.Lattice(**dict(w.params(), **kw), halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id()))
    monkeypatch.delenv("LBM_TMA")
    for g in [a] + hs:
        g.init_fields(rho, u)
        g.step(21)
    fa = a.get_populations()
    a.close()
    for g in hs:
        fg = g.get_populations()
        g.close()
        assert np.all(np.isfinite(fg))
        if prec == 0:
            assert np.abs(fg - fa).max() <= 1e-14
        else:
            assert (np.abs(fg - fa) / np.abs(fa)).max() <= 1e-6


def test_tma_kernel_bench_geometry_sampled_oracle(P):
    """512 x 512 x 8 periodic TGV (the bench's rows): one step through the TMA
    kernel equals the oracle's update of sampled nodes, including every tile
    edge x = 0, 127, 128, 255, 256, 383, 384, 511."""
    import oracle as O

    w = synth.CONFIGS["weak"].scaled(nz=8)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 5)
    g = P.Lattice(**w.params(), graphs=1)
    g.init_fields(rho, u)
    g.step(1)
    f1 = g.get_populations()
    g.close()
    xs = [0, 1, 127, 128, 255, 256, 383, 384, 510, 511]
    # patch oracle: a periodic 3x3x3 neighbourhood is enough for one step of a pull scheme
    for x in xs:
        for (y, z) in [(0, 0), (255, 3), (511, 7)]:
            sub = O.Oracle(**w.scaled(nx=3, ny=3, nz=3).params())
            ix = [(x - 1) % w.nx, x, (x + 1) % w.nx]
            iy = [(y - 1) % w.ny, y, (y + 1) % w.ny]
            iz = [(z - 1) % w.nz, z, (z + 1) % w.nz]
            r = rho[np.ix_(iz, iy, ix)]
            uu = u[:, iz][:, :, iy][:, :, :, ix]
            sub.init_fields(np.ascontiguousarray(r), np.ascontiguousarray(uu))
            sub.step(1)
            ref = sub.get_populations()[:, 1, 1, 1]
            assert np.abs(f1[:, z, y, x] - ref).max() <= 1e-14, (x, y, z)
