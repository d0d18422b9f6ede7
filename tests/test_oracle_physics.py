"""Physics pins of the oracle (no GPU): analytic solutions the paper cites.

  * shear-wave decay nu k^2 with nu from Eq. 53
  * isotropy of the recovered viscous stress on cuboid grids (the purpose of
    the corrections, Eqs. 38-40 / App D): a 2D Taylor-Green vortex
    rotated into each coordinate plane decays at 2 nu k^2, while the scheme with
    the corrections OFF does not
  * the 3D Taylor-Green vortex of BASELINE config 1 (exp(-3 nu k^2 t))
  * the square-duct Poiseuille series, Eq. 70 (erratum E15)
  * conservation over many steps with walls (P2)
"""
import numpy as np
import pytest

import oracle as O
import synth

FULL, LOW, OFF = 0, 1, 2


def _decay_rate(o, proj, n_skip, n_meas):
    o.step(n_skip)
    a1 = proj(o)
    o.step(n_meas)
    a2 = proj(o)
    return -np.log(a2 / a1) / n_meas


def _tgv2d_rate(plane, r, s, nphys, nu, corr, amp=1e-4):
    return _tgv2d_rate_model(plane, r, s, nphys, nu, corr, amp, model=0)


def _tgv2d_rate_model(plane, r, s, nphys, nu, corr, amp=1e-4, model=0):
    """Exact z-invariant 2D TGV in `plane` with equal physical wavelength nphys
    along both axes; amplitude decays as exp(-2 nu k^2 t)."""
    cs2 = synth.auto_cs2(r, s)
    sp = {"x": 1.0, "y": r, "z": s}
    n = {d: (int(round(nphys / sp[d])) if d in plane else 1) for d in "xyz"}
    o = O.Oracle(n["x"], n["y"], n["z"], r, s, cs2, synth.omega_from_nu(nu, cs2), corrections=corr,
                 model=model)
    k = 2 * np.pi / nphys
    Z, Y, X = np.meshgrid(np.arange(n["z"]) * s, np.arange(n["y"]) * r, np.arange(n["x"]) * 1.0,
                          indexing="ij")
    c = {"x": X, "y": Y, "z": Z}
    a, b = plane
    ia, ib = "xyz".index(a), "xyz".index(b)
    u = np.zeros((3,) + X.shape)
    u[ia] = amp * np.sin(k * c[a]) * np.cos(k * c[b])
    u[ib] = -amp * np.cos(k * c[a]) * np.sin(k * c[b])
    o.init_fields(np.ones(X.shape), u)
    basis = np.sin(k * c[a]) * np.cos(k * c[b])
    rate = _decay_rate(o, lambda o: (o.macroscopic()[1][ia] * basis).sum(), 50, 200)
    return rate / (2 * nu * k * k)


@pytest.mark.parametrize("axis", ["y", "z"])
@pytest.mark.parametrize("r,s", [(1.0, 2.0), (0.5, 1.0)])
def test_shear_wave_viscosity(r, s, axis):
    """u_x = A sin(k y) (or sin(k z)) decays at nu k^2; this mode involves only
    k_110 / k_101, so it pins Eq. 53 and the y/z streaming scale (r, s)."""
    nu = 0.05
    cs2 = synth.auto_cs2(r, s)
    L = 64.0
    h = r if axis == "y" else s
    n = int(round(L / h))
    ny, nz = (n, 1) if axis == "y" else (1, n)
    o = O.Oracle(1, ny, nz, r, s, cs2, synth.omega_from_nu(nu, cs2))
    k = 2 * np.pi / L
    coord = (np.arange(n) * h).reshape((1, n, 1) if axis == "y" else (n, 1, 1))
    u = np.zeros((3, nz, ny, 1))
    u[0] = 1e-4 * np.sin(k * coord)
    o.init_fields(np.ones((nz, ny, 1)), u)
    basis = np.sin(k * coord)
    rate = _decay_rate(o, lambda o: (o.macroscopic()[1][0] * basis).sum(), 20, 300)
    assert rate / (nu * k * k) == pytest.approx(1.0, abs=0.01)


@pytest.mark.parametrize("r,s,plane", [(1.0, 2.0, "xz"), (1.0, 2.0, "yz"), (0.5, 1.0, "xy"),
                                       (0.5, 1.0, "xz"), (0.5, 1.0, "yz")])
def test_viscous_isotropy_with_corrections(r, s, plane):
    """P9: with the corrections (FULL_LOCAL) the normal viscous stresses are
    isotropic: every plane decays at 2 nu k^2 (within 1.5% at wavelength 32
    x-units); with the corrections OFF the off-axis rate is >2x wrong."""
    full = _tgv2d_rate(plane, r, s, 32, 0.02, FULL)
    assert full == pytest.approx(1.0, abs=0.015)
    off = _tgv2d_rate(plane, r, s, 32, 0.02, OFF)
    assert off > 2.0


def test_isotropy_error_converges_second_order():
    """Discretisation error of the corrected scheme shrinks ~4x per doubling."""
    e32 = abs(_tgv2d_rate("xz", 0.5, 1.0, 32, 0.02, FULL) - 1.0)
    e64 = abs(_tgv2d_rate("xz", 0.5, 1.0, 64, 0.02, FULL) - 1.0)
    assert e64 < e32 / 2.5


def test_tgv3d_config1_decay():
    """BASELINE config 1 geometry (32x32x16, r=1, s=2, nu=0.01) in the linear
    regime: base-mode amplitude decays at 3 nu k^2, k = 2 pi/32 (reading R9);
    32 nodes/wavelength give a 2.6% second-order discretisation error."""
    w = synth.CONFIGS["tgv"]
    o = O.Oracle(**w.params())
    rho, u = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, 1e-4)
    o.init_fields(rho, u)
    X = 2 * np.pi * np.arange(w.nx) / w.nx
    Y = 2 * np.pi * np.arange(w.ny) / w.ny
    Zc = 2 * np.pi * np.arange(w.nz) / w.nz
    Zg, Yg, Xg = np.meshgrid(Zc, Y, X, indexing="ij")
    basis = np.sin(Xg) * np.cos(Yg) * np.cos(Zg)
    k = 2 * np.pi / 32
    rate = _decay_rate(o, lambda o: (o.macroscopic()[1][0] * basis).sum(), 60, 40)
    assert rate / (3 * w.nu * k * k) == pytest.approx(1.0, abs=0.035)


def _tgv3d_rate(n, nu=0.01, amp=1e-4, skip=60, meas=40):
    """Config-1 geometry scaled to n x n x n/2 nodes (r = 1, s = 2, so the
    physical box stays cubic, reading R9): measured base-mode decay rate over
    the analytic 3 nu k^2, k = 2 pi/n."""
    w = synth.CONFIGS["tgv"]
    cs2 = w.cs2_value
    o = O.Oracle(n, n, n // 2, w.r, w.s, cs2, synth.omega_from_nu(nu, cs2))
    rho, u = synth.tgv_fields(n, n, n // 2, cs2, amp)
    o.init_fields(rho, u)
    X = 2 * np.pi * np.arange(n) / n
    Zc = 2 * np.pi * np.arange(n // 2) / (n // 2)
    Zg, Yg, Xg = np.meshgrid(Zc, X, X, indexing="ij")
    basis = np.sin(Xg) * np.cos(Yg) * np.cos(Zg)
    k = 2 * np.pi / n
    return _decay_rate(o, lambda o: (o.macroscopic()[1][0] * basis).sum(), skip, meas) / (3 * nu * k * k)


def test_tgv3d_decay_converges_to_the_analytic_rate():
    """P12, tightened: the 3D TGV decay rate on the config-1 lattice family
    (r = 1, s = 2) converges at second order to exp(-3 nu k^2 t): the error
    shrinks >= 3.5x from 32 to 64 nodes per wavelength, and the Richardson
    extrapolation (4 e64 - e32)/3 of the two rates matches 3 nu k^2 within
    0.5 %.  (Measured: 1.0258 at 32, 1.0063 at 64, extrapolated 0.9997.)"""
    r32 = _tgv3d_rate(32)
    r64 = _tgv3d_rate(64)
    assert abs(r64 - 1.0) < abs(r32 - 1.0) / 3.5
    assert (4 * r64 - r32) / 3 == pytest.approx(1.0, abs=0.005)


def _eq70(y, z, L, F, rho, nu, nmax=199):
    """Eq. 70 with the exponent read as (-1)^((n-1)/2) (erratum E15)."""
    acc = 0.0
    for n in range(1, nmax + 1, 2):
        acc = acc + (-1) ** ((n - 1) // 2) * (1 - np.cosh(n * np.pi * z / L) / np.cosh(n * np.pi / 2)) \
            * np.cos(n * np.pi * y / L) / n ** 3
    return 4 * L * L * F / (np.pi ** 3 * rho * nu) * acc


@pytest.mark.parametrize("r,s,ny,nz,cs2", [(1.0, 2.0, 16, 8, 1 / 3), (0.5, 1.0, 32, 16, 1 / 12)])
def test_duct_poiseuille_eq70(r, s, ny, nz, cs2):
    """P6: body-force-driven square duct with halfway bounce-back walls matches
    Eq. 70 (L = 16) at steady state within 3% (L2)."""
    L, nu, F = 16.0, 0.1, 1e-5
    o = O.Oracle(1, ny, nz, r, s, cs2, synth.omega_from_nu(nu, cs2), force=(F, 0, 0),
                 bc=(0, 0, 1, 1, 1, 1))
    o.init_fields(np.ones((nz, ny, 1)), np.zeros((3, nz, ny, 1)))
    o.step(3000)
    u = o.macroscopic()[1][0][:, :, 0]
    y = (np.arange(ny) + 0.5) * r - L / 2
    z = (np.arange(nz) + 0.5) * s - L / 2
    Z, Y = np.meshgrid(z, y, indexing="ij")
    ua = _eq70(Y, Z, L, F, 1.0, nu)
    assert np.sqrt(((u - ua) ** 2).sum() / (ua ** 2).sum()) < 0.03
    # centre value coefficient 0.0736714 F L^2/(rho nu) (series at y=z=0)
    assert _eq70(0.0, 0.0, L, F, 1.0, nu) == pytest.approx(0.0736714 * F * L * L / nu, rel=1e-5)


def test_walls_conserve_mass_and_lid_drives_flow():
    """Closed cavity (all halfway bounce-back, +y moving): total mass is constant
    to round-off; the lid drags the fluid next to it along +x."""
    w = synth.CONFIGS["cavity100"].scaled(nx=12, ny=12, nz=6)
    o = O.Oracle(**w.params())
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, seed=9, rho_amp=1e-3, u_amp=1e-3)
    o.init_fields(rho, u)
    m0 = o.f.sum()
    o.step(200)
    assert abs(o.f.sum() - m0) / m0 < 1e-13
    _, uu = o.macroscopic()
    assert uu[0, :, -1, 1:-1].mean() > 0.2 * w.wall_u


def test_free_slip_conserves_mass_and_tangential_momentum():
    """Free-slip y walls (reading R7), periodic x and z: total mass and total x/z
    momentum are conserved exactly (up to round-off)."""
    w = synth.CONFIGS["shear"].scaled(nx=8, ny=16, nz=8)
    o = O.Oracle(**w.params())
    rho, u = synth.shear_layer_fields(w.nx, w.ny, w.nz, w.u0, thickness=3.0, seed=1)
    o.init_fields(rho, u)
    e = O.velocities(w.r, w.s)
    m0 = o.f.sum()
    p0 = np.einsum("qzyx,qd->d", o.f, e)
    o.step(100)
    assert abs(o.f.sum() - m0) / m0 < 1e-13
    p1 = np.einsum("qzyx,qd->d", o.f, e)
    assert abs(p1[0] - p0[0]) < 1e-12 * m0 and abs(p1[2] - p0[2]) < 1e-12 * m0


@pytest.mark.parametrize("r,s,axis", [(1.0, 2.0, "y"), (0.5, 1.0, "y"), (1.0, 2.0, "z")])
def test_free_slip_cosine_shear_mode_decay(r, s, axis):
    """Analytic pin of the free-slip rule (reading R7): between two stress-free
    walls the shear mode u_x = A cos(n pi (j + 1/2)/N) satisfies du_x/dn = 0 and
    u_n = 0 at the halfway wall positions j = -1/2 and N - 1/2, so it decays at
    nu k^2 with k = n pi / (N h), h the node spacing across the walls.  A wrong
    mirror (e.g. plain bounce-back, or a slip rule that loses tangential
    momentum) gives a no-slip-like rate for the n = 1 mode (k -> ~2x, rate ~4x)."""
    nu = 0.05
    cs2 = synth.auto_cs2(r, s)
    h = r if axis == "y" else s
    N = int(round(64.0 / h))
    FS, PER = synth.BC_FREE_SLIP, synth.BC_PERIODIC
    bc = (PER, PER, FS, FS, PER, PER) if axis == "y" else (PER, PER, PER, PER, FS, FS)
    ny, nz = (N, 1) if axis == "y" else (1, N)
    o = O.Oracle(1, ny, nz, r, s, cs2, synth.omega_from_nu(nu, cs2), bc=bc)
    for n_mode in (1, 2):
        k = n_mode * np.pi / (N * h)
        j = np.arange(N)
        prof = np.cos(n_mode * np.pi * (j + 0.5) / N)
        basis = prof.reshape((1, N, 1) if axis == "y" else (N, 1, 1))
        u = np.zeros((3, nz, ny, 1))
        u[0] = 1e-4 * basis
        o.init_fields(np.ones((nz, ny, 1)), u)
        rate = _decay_rate(o, lambda o: (o.macroscopic()[1][0] * basis).sum(), 20, 300)
        assert rate / (nu * k * k) == pytest.approx(1.0, abs=0.015), (n_mode, rate / (nu * k * k))


@pytest.mark.parametrize("r,s", [(1.0, 2.0), (0.5, 1.0), (1.0, 1.0)])
def test_moving_wall_couette_profile(r, s):
    """Analytic pin of the moving-wall rule (Eq. 69, readings R4/R5):
    plane Couette flow between a bounce-back wall at j = -1/2 and the +y lid at
    j = N - 1/2 moving with U reaches the linear profile u_x = U (j + 1/2)/N.
    Only du_x/dy is non-zero, so the corrections are inactive and the steady
    profile is exact up to compressibility (observed <= 6e-5 U)."""
    nu, N, U = 0.1, 16, 0.05
    cs2 = synth.auto_cs2(r, s)
    o = O.Oracle(1, N, 1, r, s, cs2, synth.omega_from_nu(nu, cs2), bc=(0, 0, 1, 2, 0, 0), wall_u=U)
    o.init_fields(np.ones((1, N, 1)), np.zeros((3, 1, N, 1)))
    H = N * r
    o.step(int(12 * H * H / nu))  # slowest mode decays as exp(-nu (pi/H)^2 t): < 1e-40
    _, u = o.macroscopic()
    exact = U * (np.arange(N) + 0.5) / N
    assert np.abs(u[0, 0, :, 0] - exact).max() <= 2e-4 * U
    assert np.abs(u[1]).max() < 1e-12 and np.abs(u[2]).max() < 1e-12


def test_periodic_momentum_grows_by_force():
    """Fully periodic: total momentum grows by exactly N F per step (P2)."""
    w = synth.CONFIGS["tgv"].scaled(nx=6, ny=5, nz=4, force=(1e-5, -2e-5, 3e-6))
    o = O.Oracle(**w.params())
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, seed=3)
    o.init_fields(rho, u)
    e = O.velocities(w.r, w.s)
    p0 = np.einsum("qzyx,qd->d", o.f, e)
    o.step(10)
    p1 = np.einsum("qzyx,qd->d", o.f, e)
    assert np.allclose(p1 - p0, 10 * w.nodes * np.array(w.force), rtol=1e-9, atol=1e-14)


def test_pulsatile_duct_womersley():
    """Time-periodic forcing F_x = F_m cos(omega t) in a square duct (PAPER.md
    L804-853) against the Womersley series (erratum E14 form, studies/analytic.py):
    Wo = 3.09, 2a = 16 on a (r, s) = (0.5, 1) lattice, second period, four phases,
    L2 error < 2%."""
    from studies.analytic import womersley

    r, s, ny, nz, twoa, T, Wo = 0.5, 1.0, 32, 16, 16.0, 1600, 3.09
    a = twoa / 2
    om = 2 * np.pi / T
    nu = a * a * om / Wo ** 2
    Fm = 1e-5
    cs2 = synth.auto_cs2(r, s)
    o = O.Oracle(1, ny, nz, r, s, cs2, synth.omega_from_nu(nu, cs2), bc=(0, 0, 1, 1, 1, 1))
    o.init_fields(np.ones((nz, ny, 1)), np.zeros((3, nz, ny, 1)))
    y = (np.arange(ny) + 0.5) * r - a
    z = (np.arange(nz) + 0.5) * s - a
    Z, Y = np.meshgrid(z, y, indexing="ij")
    errs = []
    for n in range(1, 2 * T + 1):
        o.set_force((Fm * np.cos(om * n), 0.0, 0.0))
        o.step(1)
        if n > T and (2 * T - n) % (T // 4) == 0:
            u = o.macroscopic()[1][0][:, :, 0]
            ua = womersley(Y, Z, n, a, Fm, om, nu)
            errs.append(np.sqrt(((u - ua) ** 2).sum() / (ua ** 2).sum()))
    assert len(errs) == 4 and max(errs) < 0.02, errs
