"""FULL_FD_LAG (reading R16b: the lambda / e_rho corrections with the gradient of
the stored state's density, one time level behind) on the B200 against the CPU
oracle (corrections = 4), element by element after 100 steps: fp64 max|df| <=
1e-12, fp32 storage max|df|/|f| <= 1e-5 (R12); the ghost-plane paths (NCCL send
to self, fused P2P with the slab as its own neighbour, P2P slabs stepped one at a
time) against the single-launch lattice; checkpoint/resume bit for bit."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

LAG = synth.CORR_FULL_FD_LAG


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2107_14774_b200 as P

    P.load()
    return P


CASES = {
    "tgv_config1": (synth.CONFIGS["tgv"], {}),
    "tgv_wide": (synth.CONFIGS["tgv"].scaled(nx=160, ny=36, nz=12), {}),
    "cavity_lid": (synth.CONFIGS["cavity1000"].scaled(nx=21, ny=19, nz=11), {}),
    "shear_slip_raw": (synth.CONFIGS["shear"].scaled(nx=16, ny=29, nz=12), {"model": 1}),
    "duct_generic": (synth.CONFIGS["duct"].scaled(nx=5, ny=37, nz=19), {"omega_1": 1.2, "omega_high": 0.9}),
}


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("case", list(CASES))
def test_fd_lag_matches_oracle_100_steps(P, case, prec):
    import oracle as O

    w, kw = CASES[case]
    w = w.scaled(corrections=LAG, precision=prec, **kw)
    o = O.Oracle(**w.params())
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 19)
    o.init_fields(rho, u)
    f0 = o.get_populations() * (1.0 + 1e-3 * synth.noise((27, w.nz, w.ny, w.nx), 1900))
    o.set_populations(f0)
    g = P.Lattice(**w.params())
    g.set_populations(f0)
    o.step(100)
    g.step(100)
    fo, fg = o.get_populations(), g.get_populations()
    g.close()
    assert np.all(np.isfinite(fg))
    if prec == 0:
        assert np.abs(fg - fo).max() <= 1e-12
    else:
        assert (np.abs(fg - fo) / np.abs(fo)).max() <= 1e-5


@pytest.mark.parametrize("prec", [0, 1])
def test_fd_lag_ghost_paths_match_wrap(P, prec):
    w = synth.CONFIGS["weak"].scaled(nx=40, ny=24, nz=12, corrections=LAG, precision=prec)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 23)
    a = P.Lattice(**w.params())
    b = P.Lattice(**w.params(), halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id())
    c = P.Lattice(**w.params(), halo=P.HALO_P2P)
    for g in (a, b, c):
        g.init_fields(rho, u)
        g.step(30)
    fa = a.get_populations()
    tol = 1e-14 if prec == 0 else 1e-6
    for g in (b, c):
        fg = g.get_populations()
        d = np.abs(fg - fa).max() if prec == 0 else (np.abs(fg - fa) / np.abs(fa)).max()
        assert d <= tol
        g.close()
    a.close()


@pytest.mark.parametrize("world", [2, 3])
def test_fd_lag_p2p_slabs_match_single_lattice(P, world):
    """Slabs of one process wired with the fused P2P halo, stepped one at a time
    (the density ghost planes travel with the populations in the same publish)."""
    w = synth.CONFIGS["cavity100"].scaled(nx=17, ny=13, nz=6 * world, corrections=LAG)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 29)
    ref = P.Lattice(**w.params())
    ref.init_fields(rho, u)
    ref.step(20)
    fr = ref.get_populations()
    ref.close()
    hs = [P.Lattice(**w.params(), rank=r, world=world, halo=P.HALO_P2P) for r in range(world)]
    blobs = [h.p2p_export() for h in hs]
    for h in hs:
        h.p2p_connect(*P.lbm.p2p_neighbour_blobs(P.lbm.halo_plan(h.p), blobs))
    n = w.nz // world
    for r, h in enumerate(hs):
        h.init_fields(np.ascontiguousarray(rho[r * n:(r + 1) * n]), np.ascontiguousarray(u[:, r * n:(r + 1) * n]))
        h.sync()
    for _ in range(20):
        for h in hs:
            h.step(1)
            h.sync()
    f = np.concatenate([h.get_populations() for h in hs], axis=1)
    for h in hs:
        h.close()
    assert np.abs(f - fr).max() <= 1e-14


def test_fd_lag_checkpoint_resume_exact(P):
    w = synth.CONFIGS["cavity100"].scaled(nx=21, ny=19, nz=11, corrections=LAG)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 31)
    a = P.Lattice(**w.params())
    a.init_fields(rho, u)
    a.step(24)
    ref = a.get_populations()
    a.close()
    b = P.Lattice(**w.params())
    b.init_fields(rho, u)
    b.step(11)
    ck = b.get_populations()
    b.close()
    c = P.Lattice(**w.params())
    c.set_populations(ck)
    c.step(13)
    assert np.array_equal(c.get_populations(), ref)
    c.close()
