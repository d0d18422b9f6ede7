"""The TMA-staged fused FULL_FD kernel (csrc/cm_tma.cuh, k_collide_stream_fd_tma,
LBM_FD_TMA=1: 27 cp.async.bulk.tensor boxes per plane of a 32 x 4 tile and its
ring, mbarrier ring, producer warp; same-time density of P:L494, L1171-1186,
reading R16) on the B200:

* against the CPU oracle (corrections = FULL_FD) element by element after 100
  steps on lattices wide enough that most tiles are staged (nx >= 128: tiles
  with 32 <= x0 <= nx - 34 and 4 <= y0 <= ny - 6): fp64 max|df| <= 1e-12, fp32
  storage max|df|/|f| <= 1e-5 (R12);
* against the LDG fused kernel (LBM_FD_FUSED=1) on the same inputs: the two
  inline the same per-node arithmetic on the same source values (max|df| <=
  1e-14 fp64, relative <= 1e-6 fp32; equal unless ptxas contracts a
  multiply-add differently), through the NCCL ghost-plane path and the fused
  P2P halo too (interior launch staged, the density of the planes next to the
  ghost faces from the density field);
* geometries: periodic (seam tiles on the LDG body), free-slip y walls, x and y
  bounce-back walls with the moving lid and periodic z, generic rates and body
  force, the raw-moment model; z walls select the LDG kernel (kernel_name).
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

FD = synth.CORR_FULL_FD
P_, BB, MW, FS = synth.BC_PERIODIC, synth.BC_BOUNCE_BACK, synth.BC_MOVING_WALL, synth.BC_FREE_SLIP


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2107_14774_b200 as P

    P.load()
    return P


CASES = {
    "tgv_wide": (synth.CONFIGS["tgv"].scaled(nx=160, ny=36, nz=12), {}),
    "tgv_ragged": (synth.CONFIGS["tgv"].scaled(nx=196, ny=30, nz=7), {}),
    "shear_slip_raw": (synth.CONFIGS["shear"].scaled(nx=128, ny=26, nz=10), {"model": 1}),
    "walls_xy_lid_zper": (synth.CONFIGS["cavity100"].scaled(nx=136, ny=22, nz=9, bc=(BB, BB, BB, MW, P_, P_)), {}),
    "generic_force": (synth.CONFIGS["tgv"].scaled(nx=128, ny=20, nz=8),
                      {"omega_1": 1.2, "omega_high": 0.9, "force": (1e-5, -2e-6, 3e-6)}),
    # one- and two-plane slabs: with ghost planes the boundary launch is contiguous
    # and collides planes whose density comes from the exchanged field
    "tgv_nz2": (synth.CONFIGS["tgv"].scaled(nx=96, ny=20, nz=2), {}),
    "tgv_nz1": (synth.CONFIGS["tgv"].scaled(nx=64, ny=16, nz=1), {}),
}


def _lattice(P, monkeypatch, w, kw, tma, **extra):
    monkeypatch.setenv("LBM_FD_FUSED", "1")
    monkeypatch.setenv("LBM_FD_TMA", "1" if tma else "0")
    g = P.Lattice(**dict(w.params(), **kw), **extra)
    monkeypatch.delenv("LBM_FD_TMA")
    monkeypatch.delenv("LBM_FD_FUSED")
    return g


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("case", list(CASES))
def test_fd_tma_matches_oracle_100_steps(P, case, prec, monkeypatch):
    import oracle as O

    w, kw = CASES[case]
    w = w.scaled(corrections=FD, precision=prec, **kw)
    o = O.Oracle(**w.params())
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 23)
    o.init_fields(rho, u)
    f0 = o.get_populations() * (1.0 + 1e-3 * synth.noise((27, w.nz, w.ny, w.nx), 2300))
    o.set_populations(f0)
    g = _lattice(P, monkeypatch, w, {}, True)
    assert "fd_tma" in g.kernel_name()
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
@pytest.mark.parametrize("case", list(CASES))
def test_fd_tma_matches_ldg_fused(P, case, prec, monkeypatch):
    w, kw = CASES[case]
    w = w.scaled(corrections=FD, precision=prec, **kw)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 31)
    a = _lattice(P, monkeypatch, w, {}, False)
    assert "fd_tma" not in a.kernel_name()
    hs = [_lattice(P, monkeypatch, w, {}, True, graphs=1), _lattice(P, monkeypatch, w, {}, True, graphs=2)]
    if w.bc[4] == synth.BC_PERIODIC:
        hs.append(_lattice(P, monkeypatch, w, {}, True, halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id()))
        hs.append(_lattice(P, monkeypatch, w, {}, True, halo=P.HALO_P2P))  # the slab is its own neighbour
    for g in hs:
        assert "fd_tma" in g.kernel_name()
    for g in [a] + hs:
        g.init_fields(rho, u)
        g.step(23)
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


def test_fd_tma_not_selected_with_z_walls(P, monkeypatch):
    w = synth.CONFIGS["cavity100"].scaled(nx=128, ny=16, nz=8, corrections=FD)
    g = _lattice(P, monkeypatch, w, {}, True)
    name = g.kernel_name()
    g.close()
    assert "fd_tma" not in name and "k_collide_stream_fd" in name


def test_fd_tma_default_selection(P):
    """Default (no LBM_FD_TMA): the TMA kernel where >= 3/4 of the tiles are
    staged (the bench's 512 x 512 planes), the two-pass path otherwise."""
    for (nx, ny, on) in [(512, 512, True), (160, 36, True), (64, 16, False), (40, 24, False), (196, 30, False)]:
        w = synth.CONFIGS["tgv"].scaled(nx=nx, ny=ny, nz=4, corrections=FD)
        g = P.Lattice(**w.params())
        name = g.kernel_name()
        g.close()
        assert ("fd_tma" in name) == on, (nx, ny, name)


def test_fd_tma_bench_geometry_sampled_oracle(P, monkeypatch):
    """512 x 512 x 8 periodic TGV with FULL_FD (the bench's plane): one step
    through the TMA kernel equals the oracle's update at sampled nodes on staged
    tiles, seam tiles and tile edges.  One FULL_FD step of a node depends on the
    populations within two nodes (its neighbours' pulled densities), so a
    periodic 5 x 5 x 5 oracle lattice around it, initialised from the same
    fields, reproduces it."""
    import oracle as O

    w = synth.CONFIGS["weak"].scaled(nz=8, corrections=FD)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 7)
    g = _lattice(P, monkeypatch, w, {}, True)
    assert "fd_tma" in g.kernel_name()
    g.init_fields(rho, u)
    g.step(1)
    f1 = g.get_populations()
    g.close()
    xs = [0, 1, 31, 32, 33, 63, 64, 255, 256, 478, 479, 480, 510, 511]
    for x in xs:
        for (y, z) in [(0, 0), (3, 1), (4, 7), (255, 3), (508, 4), (511, 7)]:
            sub = O.Oracle(**w.scaled(nx=5, ny=5, nz=5).params())
            ix = [(x + d) % w.nx for d in range(-2, 3)]
            iy = [(y + d) % w.ny for d in range(-2, 3)]
            iz = [(z + d) % w.nz for d in range(-2, 3)]
            r = rho[np.ix_(iz, iy, ix)]
            uu = u[:, iz][:, :, iy][:, :, :, ix]
            sub.init_fields(np.ascontiguousarray(r), np.ascontiguousarray(uu))
            sub.step(1)
            ref = sub.get_populations()[:, 2, 2, 2]
            assert np.abs(f1[:, z, y, x] - ref).max() <= 1e-13, (x, y, z)


@pytest.mark.parametrize("prec", [0, 1])
def test_fd_tma_full_plane_bitwise_and_deterministic(P, prec, monkeypatch):
    """The bench's 512 x 512 planes, 64 planes (two 32-plane chunks per tile: 34
    pipelined planes per CTA), 12 steps: two runs of the TMA kernel are bitwise
    equal to each other and to the LDG fused kernel.  (Without the proxy fence
    before a stage is released, a warp's outstanding shared-memory loads could
    read the refilled stage: one warp row in 10^5 went wrong, differently in
    every run.)"""
    w = synth.CONFIGS["weak"].scaled(nz=64, corrections=FD, precision=prec)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 2024)
    hs = [_lattice(P, monkeypatch, w, {}, t, graphs=1) for t in (False, True, True)]
    for g in hs:
        g.init_fields(rho, u)
        g.step(12)
    fa, fb, fc = (g.get_populations() for g in hs)
    for g in hs:
        g.close()
    assert np.array_equal(fb, fc)
    assert np.array_equal(fa, fb)
