"""Pins of the oracle's body-force bookkeeping (Eq. 12 half force, reading R8)
and of the FULL_FD density gradient next to walls (reading R16), no GPU.

The expected values come from the mathematics, not from the oracle:
  * Eq. 12: rho u = sum_a f_a e_a + F/2 of the PRE-collision
    populations; the collision conserves k_000 and sends the first central
    moments to +F/2, so the stored post-collision state carries
    sum f~ e = rho u + F/2 and the velocity a caller reads back from f~ must be
    Eq. 12's u of the populations that were collided;
  * reading R8: the initial state is f^eq(rho0, u0 + F/(2 rho0)) in the closed
    per-axis product form (tests/_util.feq_product);
  * reading R16: the isotropic stencil (1/cs2) sum_a w_a e_a rho(x + e_a) with
    mirror-image neighbours across walls is exact on fields linear along the
    wall, and for a field linear along the wall normal it returns half the
    slope (only the e_n = +1 side differs from the node's own density:
    (1/cs2) c^2 phi(+1) g = g/2 with phi(+1) = cs2/(2 c^2)).
"""
import numpy as np
import pytest

import oracle as O
from tests import _util as U

FULL, LOW, OFF, FD = 0, 1, 2, 3
RS = [(1.0, 2.0), (0.5, 1.0), (0.75, 1.3)]


def _cs2(r, s):
    return min(1.0, r * r, s * s) / 3.0


def _e(r, s):
    """Eqs. 1a-1c, re-typed here: e_a = (EX, r EY, s EZ)."""
    return np.stack([np.array(U.EX, float), r * np.array(U.EY, float), s * np.array(U.EZ, float)], axis=1)


def _eq12_u(f, r, s, F):
    """Eq. 12: u = (sum_a f_a e_a + F/2) / sum_a f_a."""
    return (f @ _e(r, s) + 0.5 * np.asarray(F)) / f.sum()


@pytest.mark.parametrize("r,s", RS)
def test_init_stores_half_shifted_equilibrium(r, s):
    """R8: init writes f^eq(rho, u + F/(2 rho)); its first moment is rho u + F/2."""
    cs2 = _cs2(r, s)
    F = np.array([3e-4, -2e-4, 1e-4])
    rng = np.random.default_rng(21)
    shape = (2, 3, 4)
    rho = rng.uniform(0.97, 1.03, shape)
    u = rng.uniform(-0.03, 0.03, (3,) + shape)
    o = O.Oracle(4, 3, 2, r, s, cs2, 1.4, force=F)
    o.init_fields(rho, u)
    f = o.get_populations()
    for (z, y, x) in [(0, 0, 0), (1, 2, 3), (0, 1, 2)]:
        fx = f[:, z, y, x]
        expect = U.feq_product(r, s, cs2, rho[z, y, x], u[:, z, y, x] + F / (2 * rho[z, y, x]))
        assert np.allclose(fx, expect, rtol=1e-14, atol=1e-17)
        assert np.allclose(fx @ _e(r, s), rho[z, y, x] * u[:, z, y, x] + F / 2, rtol=0, atol=2e-16)


@pytest.mark.parametrize("r,s", RS)
def test_macroscopic_after_init_returns_the_fields(r, s):
    """get_macroscopic(init(rho, u)) == (rho, u) with F != 0 (R8 + P:L1207-1210)."""
    cs2 = _cs2(r, s)
    F = np.array([-4e-4, 2e-4, 3e-4])
    rng = np.random.default_rng(22)
    shape = (3, 2, 5)
    rho = rng.uniform(0.95, 1.05, shape)
    u = rng.uniform(-0.04, 0.04, (3,) + shape)
    o = O.Oracle(5, 2, 3, r, s, cs2, 1.2, force=F)
    o.init_fields(rho, u)
    rho2, u2 = o.macroscopic()
    assert np.abs(rho2 - rho).max() <= 1e-15
    assert np.abs(u2 - u).max() <= 1e-15


@pytest.mark.parametrize("model", [0, 1])
@pytest.mark.parametrize("corr", [FULL, OFF])
@pytest.mark.parametrize("r,s", RS)
def test_velocity_read_back_after_collision_is_eq12(r, s, corr, model):
    """For random non-equilibrium f and omega_1 in {0.7, 1, 1.6}: the velocity
    the oracle reports for the collided state f~ equals Eq. 12's u of f, and its
    density equals sum f.  A sign or factor slip in the F/2 of either Eq. 12,
    the first-order relaxation or the read-back shows up as a u error ~F/rho."""
    cs2 = _cs2(r, s)
    F = np.array([2e-3, -1.5e-3, 1e-3])  # large, so an F/2 slip is ~1e-3, far above round-off
    rng = np.random.default_rng(23)
    for w1 in (0.7, 1.0, 1.6):
        o = O.Oracle(1, 1, 1, r, s, cs2, omega_nu=1.7, omega_xi=1.1, omega_1=w1, omega_high=1.3,
                     force=F, corrections=corr, model=model)
        for _ in range(3):
            rho0 = rng.uniform(0.95, 1.05)
            u0 = rng.uniform(-0.05, 0.05, 3)
            f = U.feq_product(r, s, cs2, rho0, u0) * (1.0 + 0.02 * rng.uniform(-1, 1, 27))
            ft = o.collide(f)
            o.set_populations(ft.reshape(27, 1, 1, 1))
            rho, u = o.macroscopic()
            assert abs(rho.ravel()[0] - f.sum()) <= 1e-15
            assert np.abs(u.reshape(3) - _eq12_u(f, r, s, F)).max() <= 2e-16


@pytest.mark.parametrize("r,s", RS)
def test_uniform_periodic_state_accelerates_by_F_over_rho(r, s):
    """A uniform periodic state is streamed onto itself, so one step is one
    collision: u advances by exactly F/rho per step (Newton's law for the
    body force), rho is unchanged."""
    cs2 = _cs2(r, s)
    F = np.array([1e-4, -2e-4, 5e-5])
    rho0, u0 = 1.02, np.array([0.01, 0.02, -0.015])
    o = O.Oracle(2, 3, 2, r, s, cs2, 1.5, force=F)
    o.init_fields(np.full((2, 3, 2), rho0), np.broadcast_to(u0.reshape(3, 1, 1, 1), (3, 2, 3, 2)).copy())
    o.step(5)
    rho, u = o.macroscopic()
    assert np.abs(rho - rho0).max() <= 2e-15
    expect = u0 + 5 * F / rho0
    assert np.abs(u.reshape(3, -1) - expect[:, None]).max() <= 2e-15


def _grid(nx, ny, nz, r, s):
    return np.meshgrid(np.arange(nz) * s, np.arange(ny) * r, np.arange(nx) * 1.0, indexing="ij")


@pytest.mark.parametrize("r,s", RS)
def test_wall_gradient_exact_along_the_wall(r, s):
    """R16 at walls: for a density linear in the wall-parallel coordinates the
    gradient at every wall-adjacent node (faces, edges, corners) is exact."""
    cs2 = _cs2(r, s)
    nx, ny, nz = 4, 5, 6
    o = O.Oracle(nx, ny, nz, r, s, cs2, 1.5, bc=(1, 1, 1, 2, 3, 3), corrections=FD)
    Z, Y, X = _grid(nx, ny, nz, r, s)
    gvec = np.array([0.011, -0.006, 0.017])
    coords = (X, Y, Z)
    for (x, y, z) in [(0, 2, 3), (nx - 1, 2, 3), (2, 0, 3), (2, ny - 1, 3), (2, 2, 0), (2, 2, nz - 1),
                      (0, 0, 3), (nx - 1, ny - 1, 0), (0, ny - 1, nz - 1), (nx - 1, 0, 0)]:
        walled = [x in (0, nx - 1), y in (0, ny - 1), z in (0, nz - 1)]
        g = np.where(walled, 0.0, gvec)  # linear only along the axes without an adjacent wall
        rho = 1.0 + sum(g[d] * coords[d] for d in range(3))
        assert np.allclose(o.density_gradient(rho, x, y, z), g, rtol=1e-12, atol=1e-16), (x, y, z)


@pytest.mark.parametrize("r,s", RS)
def test_wall_gradient_normal_component_is_half_the_slope(r, s):
    """R16 at walls: a field linear along the wall normal gives g/2 there (the
    mirror-image neighbour equals the node's own density); the wall-parallel
    components of that field are 0.  On both faces of every axis."""
    cs2 = _cs2(r, s)
    nx, ny, nz = 4, 5, 6
    o = O.Oracle(nx, ny, nz, r, s, cs2, 1.5, bc=(1, 1, 1, 1, 1, 1), corrections=FD)
    Z, Y, X = _grid(nx, ny, nz, r, s)
    coords = (X, Y, Z)
    n = (nx, ny, nz)
    for d in range(3):
        slope = 0.013 * (d + 1)
        rho = 1.0 + slope * coords[d]
        for at in (0, n[d] - 1):
            xyz = [1, 2, 3]  # interior along the other two axes
            xyz[d] = at
            g = o.density_gradient(rho, *xyz)
            expect = np.zeros(3)
            expect[d] = slope / 2
            assert np.allclose(g, expect, rtol=1e-12, atol=1e-16), (d, at, g)
