"""Pins of the FULL_FD corrections (density-gradient terms lambda and e_rho of
PAPER.md L1171-1186 with the isotropic gradient of P:L494, reading R16)."""
import numpy as np
import pytest

import oracle as O
import synth

FULL, LOW, OFF, FD = 0, 1, 2, 3


@pytest.mark.parametrize("r,s", [(1.0, 2.0), (0.5, 1.0), (0.75, 1.3)])
def test_isotropic_gradient_exact_on_linear_fields(r, s):
    """The lattice-weighted stencil (1/cs2) sum_a w_a e_a rho(x + e_a) is exact for
    linear density fields at interior nodes (sum_a w_a e_a e_a = cs2 I)."""
    cs2 = synth.auto_cs2(r, s)
    nx, ny, nz = 5, 6, 7
    o = O.Oracle(nx, ny, nz, r, s, cs2, 1.5, bc=(1, 1, 1, 1, 1, 1), corrections=FD)
    g0 = np.array([0.013, -0.007, 0.021])
    Z, Y, X = np.meshgrid(np.arange(nz) * s, np.arange(ny) * r, np.arange(nx) * 1.0, indexing="ij")
    rho = 1.0 + g0[0] * X + g0[1] * Y + g0[2] * Z
    for (x, y, z) in [(2, 3, 3), (1, 1, 1), (3, 4, 5)]:
        assert np.allclose(o.density_gradient(rho, x, y, z), g0, rtol=1e-12, atol=1e-15)
    # a wall-adjacent node sees zero normal gradient contributions from across the wall
    gw = o.density_gradient(np.ones((nz, ny, nx)), 0, 0, 0)
    assert np.allclose(gw, 0.0, atol=1e-15)


def test_gradient_second_order_on_periodic_sine():
    r, s = 1.0, 2.0
    cs2 = synth.auto_cs2(r, s)
    errs = []
    for n in (16, 32):
        o = O.Oracle(n, 2, 2, r, s, cs2, 1.5, corrections=FD)
        k = 2 * np.pi / n
        rho = np.broadcast_to(1.0 + 0.01 * np.sin(k * np.arange(n)), (2, 2, n)).copy()
        x = n // 8  # same phase k x = pi/4 on both grids
        g = o.density_gradient(rho, x, 0, 0)
        errs.append(abs(g[0] - 0.01 * k * np.cos(k * x)) / (0.01 * k))
    assert errs[1] < errs[0] / 3.5


@pytest.mark.parametrize("model", [0, 1])
def test_fd_equals_full_local_without_density_gradient(model):
    rng = np.random.default_rng(3)
    r, s, cs2 = 1.0, 2.0, 1 / 3
    a = O.Oracle(2, 2, 2, r, s, cs2, 1.6, omega_xi=1.2, corrections=FULL, model=model)
    b = O.Oracle(2, 2, 2, r, s, cs2, 1.6, omega_xi=1.2, corrections=FD, model=model)
    e = O.velocities(r, s)
    for _ in range(3):
        f = b.feq(1.02, np.array([0.03, -0.02, 0.04])) * (1 + 0.02 * rng.uniform(-1, 1, 27))
        assert np.array_equal(a.collide(f), b.collide(f, np.zeros(3)))
        fd = b.collide(f, np.array([1e-3, -2e-3, 5e-4]))
        assert np.abs(fd - a.collide(f)).max() > 1e-8
        # mass and momentum are untouched by the corrections
        assert abs(fd.sum() - f.sum()) < 1e-14 and np.allclose(fd @ e, f @ e, atol=2e-15)


def _sound_rate(corr, Ub, axis, r, s, nphys=64, nu=0.02, amp=1e-5, model=0, steps=400):
    """Attenuation of a right-going sound wave along `axis` riding on a uniform
    background flow Ub along the same axis, over theory k^2 (2 nu/3 + xi/2)
    (linearised NS with bulk viscosity, Eqs. 51/53)."""
    cs2 = synth.auto_cs2(r, s)
    h = {"x": 1.0, "y": r, "z": s}[axis]
    n = int(round(nphys / h))
    shape = {"x": (1, 1, n), "y": (1, n, 1), "z": (n, 1, 1)}[axis]
    nz, ny, nx = shape
    o = O.Oracle(nx, ny, nz, r, s, cs2, synth.omega_from_nu(nu, cs2), corrections=corr, model=model)
    c = (np.arange(n) * h).reshape(shape)
    k = 2 * np.pi / nphys
    d = "xyz".index(axis)
    rho = 1 + amp * np.cos(k * c)
    u = np.zeros((3,) + shape)
    u[d] = Ub + np.sqrt(cs2) * amp * np.cos(k * c)
    o.init_fields(rho, u)
    basis = np.exp(-1j * k * c)
    ts, amps = [], []
    for t in range(steps):
        o.step(1)
        if t >= 50 and t % 10 == 0:
            ts.append(t)
            amps.append(np.log(abs(((o.macroscopic()[0] - 1) * basis).sum())))
    rate = -np.polyfit(ts, amps, 1)[0]
    xi = (2 * cs2 / 3) * (1 / 1.0 - 0.5)
    return rate / (k * k * (2 * nu / 3 + xi / 2))


@pytest.mark.parametrize("model", [0, 1])
def test_density_gradient_corrections_restore_acoustic_attenuation(model):
    """Along the stretched axis (3 cs2 - s^2 = -3 at (r,s) = (1,2)) with a
    background flow U_b = 0.1, the u d(rho) truncation errors (Eqs. 22, 38-40)
    change the sound attenuation by > 8% unless the lambda / e_rho terms are
    included (FULL_FD: within 1%)."""
    assert _sound_rate(FD, 0.1, "z", 1.0, 2.0, model=model) == pytest.approx(1.0, abs=0.01)
    assert abs(_sound_rate(FULL, 0.1, "z", 1.0, 2.0, model=model) - 1.0) > 0.08
    # no background flow: every mode agrees with theory
    assert _sound_rate(FD, 0.0, "z", 1.0, 2.0, model=model) == pytest.approx(1.0, abs=0.01)


def test_density_gradient_corrections_on_x_axis_of_05_1_lattice():
    """(r,s) = (0.5,1), cs2 = 1/12: the x axis carries 3 cs2 - 1 = -0.75."""
    assert _sound_rate(FD, 0.08, "x", 0.5, 1.0) == pytest.approx(1.0, abs=0.04)
    assert abs(_sound_rate(FULL, 0.08, "x", 0.5, 1.0) - 1.0) > 0.15


FD_LAG = 4


@pytest.mark.parametrize("model", [0, 1])
def test_lagged_density_corrections_restore_acoustic_attenuation(model):
    """Reading R16b (FULL_FD_LAG: the gradient of the stored state's density, one
    time level behind): the same moving-frame sound attenuation as the same-time
    density of R16 -- within 1 % of the Navier-Stokes rate along the stretched
    axis with U_b = 0.1 (FULL_LOCAL: > 8 % off) and at rest."""
    assert _sound_rate(FD_LAG, 0.1, "z", 1.0, 2.0, model=model) == pytest.approx(1.0, abs=0.01)
    assert _sound_rate(FD_LAG, 0.0, "z", 1.0, 2.0, model=model) == pytest.approx(1.0, abs=0.01)


def test_lagged_density_on_x_axis_of_05_1_lattice():
    assert _sound_rate(FD_LAG, 0.08, "x", 0.5, 1.0) == pytest.approx(1.0, abs=0.04)


def test_lagged_density_is_the_stored_states_density():
    """The time level of R16b: a stored state whose every node holds density 1
    (f^eq(1, u) with u varying from node to node: sum_q f^eq = 1 per node) has a
    zero stored-density gradient, so one FULL_FD_LAG step equals one FULL_LOCAL
    step (the lambda / e_rho terms vanish with the gradient), while the
    same-time density of the PULLED populations varies and FULL_FD differs."""
    r, s = 1.0, 2.0
    cs2 = synth.auto_cs2(r, s)
    n = (6, 5, 4)
    rng = np.random.default_rng(8)
    u = rng.uniform(-0.05, 0.05, (3, n[2], n[1], n[0]))
    outs = {}
    for corr in (FULL, FD, FD_LAG):
        o = O.Oracle(*n, r, s, cs2, 1.6, omega_xi=1.2, corrections=corr)
        o.init_fields(np.ones((n[2], n[1], n[0])), u)
        o.step(1)
        outs[corr] = o.get_populations()
    assert np.abs(outs[FD_LAG] - outs[FULL]).max() < 1e-15
    assert np.abs(outs[FD] - outs[FULL]).max() > 1e-9


def test_lagged_density_conserves_mass_and_momentum():
    """Periodic lattice with a body force: mass constant, momentum + N F per step."""
    r, s = 0.75, 1.3
    cs2 = synth.auto_cs2(r, s)
    F = np.array([2e-5, -1e-5, 3e-5])
    o = O.Oracle(6, 5, 4, r, s, cs2, 1.5, omega_xi=1.1, force=F, corrections=FD_LAG)
    rho, u = synth.random_fields(6, 5, 4, 12)
    o.init_fields(rho, u)
    e = O.velocities(r, s)
    f0 = o.get_populations().reshape(27, -1)
    o.step(5)
    f1 = o.get_populations().reshape(27, -1)
    assert abs(f1.sum() - f0.sum()) < 1e-12
    assert np.allclose(e.T @ f1.sum(axis=1) - e.T @ f0.sum(axis=1), 5 * 120 * F, rtol=0, atol=1e-12)
