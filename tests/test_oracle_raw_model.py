"""Pins of the oracle's 3DCRM (raw-moment) variant, PAPER.md L642-648 (Eq.
LBErawmomentcuboidlattice), L744 remark (ii) and L1011: relax raw moments to the
Eq. 10 equilibria with the Eq. 11 sources, the same B grouping, rates and
corrections as the central-moment scheme."""
import numpy as np
import pytest

import oracle as O
from tests import _util as U

RS = [(1.0, 1.0), (1.0, 2.0), (0.5, 1.0), (0.75, 1.0)]


def _cs2(r, s):
    return min(1.0, r * r, s * s) / 3.0


def _near_eq(r, s, cs2, rng, amp=1e-2):
    rho = rng.uniform(0.95, 1.05)
    u = rng.uniform(-0.05, 0.05, 3)
    return U.feq_product(r, s, cs2, rho, u) * (1.0 + amp * rng.uniform(-1, 1, 27))


def test_eq11_is_binomial_of_eq11c_to_second_order():
    """Eq. 11 (raw source moments) follows from Eq. 11c (central: sigma_100 = F) by
    the binomial transform; it keeps the moments up to second order."""
    rng = np.random.default_rng(1)
    for _ in range(5):
        u = rng.uniform(-0.1, 0.1, 3)
        F = rng.normal(size=3) * 1e-3
        sigma = np.zeros(27)
        sigma[1:4] = F
        full = O.frame(sigma, u)
        phi = O.raw_source(u, F)
        order = np.array([sum(map(int, m)) for m in U.MOMENTS])
        assert np.allclose(phi[order <= 2], full[order <= 2], rtol=1e-14, atol=1e-18)
        assert np.all(phi[order >= 3] == 0.0)


@pytest.mark.parametrize("corr", [0, 1, 2])
@pytest.mark.parametrize("r,s", RS)
def test_raw_conservation(r, s, corr):
    rng = np.random.default_rng(2)
    cs2 = _cs2(r, s)
    F = np.array([1e-4, -3e-5, 2e-5])
    e = O.velocities(r, s)
    for w1 in (1.0, 0.7):
        o = O.Oracle(2, 2, 2, r, s, cs2, omega_nu=1.7, omega_xi=1.1, omega_1=w1, omega_high=1.3,
                     force=F, corrections=corr, model=1)
        f = _near_eq(r, s, cs2, rng)
        ft = o.collide(f)
        assert abs(ft.sum() - f.sum()) < 1e-14
        assert np.allclose(ft @ e, f @ e + F, rtol=0, atol=2e-15)


@pytest.mark.parametrize("omega", [0.8, 1.0, 1.6])
@pytest.mark.parametrize("r,s", RS)
def test_raw_srt_limit(r, s, omega):
    """All rates equal, corrections off: f~ = (1-w) f + w f^eq + (1-w/2) P^-1 S^-1 Phi,
    with P^-1 from the printed App G and S from Eq. 59 (independent of the
    oracle's numeric inverse)."""
    rng = np.random.default_rng(3)
    cs2 = _cs2(r, s)
    F = np.array([2e-4, -1e-4, 3e-4])
    o = O.Oracle(2, 2, 2, r, s, cs2, omega_nu=omega, omega_xi=omega, omega_1=omega, omega_high=omega,
                 force=F, corrections=2, model=1)
    Qi = U.appendix_G() / U.eq59_S(r, s)[None, :]
    e = O.velocities(r, s)
    for _ in range(3):
        f = _near_eq(r, s, cs2, rng, 0.05)
        rho = f.sum()
        u = (f @ e + F / 2) / rho
        expect = (1 - omega) * f + omega * U.feq_product(r, s, cs2, rho, u) + \
            (1 - omega / 2) * Qi @ O.raw_source(u, F)
        assert np.allclose(o.collide(f), expect, rtol=1e-12, atol=1e-15)


def test_raw_and_central_differ_off_equilibrium_only():
    r, s, cs2 = 0.5, 1.0, 1 / 12
    rng = np.random.default_rng(4)
    cm = O.Oracle(2, 2, 2, r, s, cs2, 1.6, model=0)
    rm = O.Oracle(2, 2, 2, r, s, cs2, 1.6, model=1)
    feq = U.feq_product(r, s, cs2, 1.01, np.array([0.04, -0.03, 0.02]))
    assert np.allclose(cm.collide(feq), rm.collide(feq), atol=1e-15)
    f = _near_eq(r, s, cs2, rng, 0.05)
    assert np.abs(cm.collide(f) - rm.collide(f)).max() > 1e-6


@pytest.mark.parametrize("r,s,plane", [(1.0, 2.0, "xz"), (0.5, 1.0, "xy")])
def test_raw_model_viscous_isotropy(r, s, plane):
    """The corrections carried by the extended equilibria make the raw-moment
    scheme isotropic as well (the second-order non-equilibrium raw and
    central moments coincide)."""
    from tests.test_oracle_physics import _tgv2d_rate_model

    assert _tgv2d_rate_model(plane, r, s, 32, 0.02, 0, model=1) == pytest.approx(1.0, abs=0.015)
    assert _tgv2d_rate_model(plane, r, s, 32, 0.02, 2, model=1) > 2.0
