"""Pins of the oracle's collision (App D) and wall rules (Eq. 69), no GPU."""
import numpy as np
import pytest

import oracle as O
from tests import _util as U

FULL, LOW, OFF = 0, 1, 2
RS = [(1.0, 1.0), (1.0, 2.0), (0.5, 1.0), (0.406, 1.3), (0.75, 1.0)]


def _cs2(r, s):
    return min(1.0, r * r, s * s) / 3.0


def _near_eq(r, s, cs2, rng, amp=1e-2):
    rho = rng.uniform(0.95, 1.05)
    u = rng.uniform(-0.05, 0.05, 3)
    f = U.feq_product(r, s, cs2, rho, u)
    return f * (1.0 + amp * rng.uniform(-1, 1, 27))


@pytest.mark.parametrize("corr", [FULL, LOW, OFF])
@pytest.mark.parametrize("r,s", RS)
def test_conservation_per_collision(r, s, corr):
    """P2: k~_000 = k_000 and k~_100 = k_100 + omega_1(0 - k_100) + (1 - omega_1/2) F with
    k_100 = -F/2 (Eq. 12 half force) give sum f~ = sum f and sum f~ e = sum f e + F,
    for any omega_1."""
    rng = np.random.default_rng(11)
    cs2 = _cs2(r, s)
    F = np.array([1e-4, -3e-5, 2e-5])
    e = O.velocities(r, s)
    for w1 in (1.0, 0.7, 1.6):
        o = O.Oracle(2, 2, 2, r, s, cs2, omega_nu=1.7, omega_xi=1.1, omega_1=w1, omega_high=1.3,
                     force=F, corrections=corr)
        f = _near_eq(r, s, cs2, rng)
        ft = o.collide(f)
        assert abs(ft.sum() - f.sum()) < 1e-14
        assert np.allclose(ft @ e, f @ e + F, rtol=0, atol=2e-15)


@pytest.mark.parametrize("omega", [0.8, 1.0, 1.5, 1.9])
@pytest.mark.parametrize("r,s", RS)
def test_srt_limit_closed_form(r, s, omega):
    """P4: with all rates equal (B^-1 Lambda B = omega I) and the corrections off,
    Eq. LBEcentralmomentcuboidlattice is linear in f:
      f~ = (1 - omega) f + omega f^eq(rho, u) + (1 - omega/2) S(u, F),
    with f^eq the product form of Eq. 10 and S the velocity-space source whose
    central moments are Eq. 11c.  Pins P, S, F, the relax/B/B^-1 bookkeeping and
    Q^-1 together against a closed form."""
    rng = np.random.default_rng(5)
    cs2 = _cs2(r, s)
    F = np.array([2e-4, -1e-4, 3e-4])
    o = O.Oracle(2, 2, 2, r, s, cs2, omega_nu=omega, omega_xi=omega, omega_1=omega,
                 omega_high=omega, force=F, corrections=OFF)
    e = O.velocities(r, s)
    for _ in range(4):
        f = _near_eq(r, s, cs2, rng, amp=0.05)
        rho = f.sum()
        u = (f @ e + F / 2) / rho
        expect = (1 - omega) * f + omega * U.feq_product(r, s, cs2, rho, u) + \
            (1 - omega / 2) * U.source_product(r, s, u, F)
        assert np.allclose(o.collide(f), expect, rtol=1e-12, atol=1e-15)


def test_corrections_vanish_on_cubic_lattice():
    """at r = s = 1, cs2 = 1/3 all grid-anisotropy terms vanish, so the
    low-Mach corrected scheme equals the uncorrected one."""
    rng = np.random.default_rng(2)
    kw = dict(omega_nu=1.6, omega_xi=1.2, force=(1e-4, 0, 0))
    a = O.Oracle(2, 2, 2, 1.0, 1.0, 1 / 3, corrections=LOW, **kw)
    b = O.Oracle(2, 2, 2, 1.0, 1.0, 1 / 3, corrections=OFF, **kw)
    c = O.Oracle(2, 2, 2, 1.0, 1.0, 1 / 3, corrections=FULL, **kw)
    for _ in range(5):
        f = _near_eq(1.0, 1.0, 1 / 3, rng, 0.05)
        assert np.allclose(a.collide(f), b.collide(f), rtol=0, atol=1e-16)
        # FULL keeps only the Galilean-invariance term -3 rho u^2 (1/omega - 1/2): O(u^2 * noneq)
        d = np.abs(c.collide(f) - b.collide(f)).max()
        assert 0 < d < 1e-3


def test_correction_order_cubic_vs_cuboid():
    """on the cubic lattice (r = s = 1, cs2 = 1/3) FULL_LOCAL differs
    from the uncorrected scheme only by the Galilean-invariance term
    -3 rho u^2 (1/omega - 1/2) times the strain, O(u^2 * noneq): with u and the
    non-equilibrium both scaled by a, the difference scales as a^3 (slope 3).
    On the cuboid lattice (s = 2) the (3 cs2 - s^2) term is O(1): slope 1."""
    rng = np.random.default_rng(11)
    u0, d = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 27)
    kw = dict(omega_nu=1.6, omega_xi=1.2)

    def diff(r, s, a):
        f = U.feq_product(r, s, 1 / 3, 1.0, a * u0) * (1.0 + a * d)
        full = O.Oracle(2, 2, 2, r, s, 1 / 3, corrections=FULL, **kw).collide(f)
        off = O.Oracle(2, 2, 2, r, s, 1 / 3, corrections=OFF, **kw).collide(f)
        return np.abs(full - off).max()

    for a in (0.02, 0.01):
        assert np.log2(diff(1.0, 1.0, a) / diff(1.0, 1.0, a / 2)) == pytest.approx(3.0, abs=0.05)
        assert np.log2(diff(1.0, 2.0, a) / diff(1.0, 2.0, a / 2)) == pytest.approx(1.0, abs=0.05)


def test_corrections_active_on_cuboid_lattice():
    """At s = 2 the (3 cs2 - s^2) term is O(1): FULL/LOW differ from OFF at
    first order in the non-equilibrium, and not at equilibrium."""
    r, s, cs2 = 1.0, 2.0, 1 / 3
    rng = np.random.default_rng(4)
    f = _near_eq(r, s, cs2, rng, 0.05)
    outs = [O.Oracle(2, 2, 2, r, s, cs2, 1.6, corrections=c).collide(f) for c in (FULL, LOW, OFF)]
    assert np.abs(outs[0] - outs[2]).max() > 1e-5
    assert np.abs(outs[1] - outs[2]).max() > 1e-5
    # at exact equilibrium (no strain) the corrections vanish
    rho, u = 1.02, np.array([0.03, -0.02, 0.01])
    feq = U.feq_product(r, s, cs2, rho, u)
    for c in (FULL, LOW, OFF):
        assert np.allclose(O.Oracle(2, 2, 2, r, s, cs2, 1.6, corrections=c).collide(feq), feq, atol=1e-15)


@pytest.mark.parametrize("r,s,cs2", [(1.0, 1.0, 1 / 3), (1.0, 2.0, 1 / 3), (0.5, 1.0, 1 / 12),
                                     (0.406, 1.3, 0.04), (1.0, 0.5, 0.10)])
def test_eq69_lid_coefficients(r, s, cs2):
    """Eq. 69 (tests/golden/eq69_lid.txt, erratum E6 applied):
    the oracle derives the augmentation from f^eq = Q^-1 m^eq at the wall
    (P:L759); it must equal the paper's printed coefficients."""
    U_w = 0.05
    o = O.Oracle(2, 2, 2, r, s, cs2, 1.5, wall_u=U_w, bc=(1, 1, 1, 2, 1, 1))
    opp = O.opposite()
    edge = (cs2 - s * s) * cs2 / (2 * r * r * s * s)
    corner = cs2 * cs2 / (4 * r * r * s * s)
    tot = 0.0
    for rho in (1.0, 0.97):
        for q, a_printed, a_used, sign, kind in U.eq69_rows():
            assert opp[q] == a_used
            C = {"none": 0.0, "edge": edge, "corner": corner}[kind]
            got = o.lid_term(q, rho)
            assert np.isclose(got, sign * C * rho * U_w, rtol=1e-12, atol=1e-17), (q, got)
            tot += got
    # mass neutral (the nine terms cancel)
    assert abs(tot) < 1e-17
    # at r = s = 1, cs2 = 1/3 (textbook cubic moving wall, 2 w_a rho e_a.U / cs2):
    # f_9 (e_x = +1) gains U/9 (edge weight 1/54), f_21 gains U/36 (corner 1/216)
    if r == s == 1.0:
        assert np.isclose(o.lid_term(9, 1.0), U_w / 9)
        assert np.isclose(o.lid_term(10, 1.0), -U_w / 9)
        assert np.isclose(o.lid_term(21, 1.0), U_w / 36)
        assert np.isclose(o.lid_term(26, 1.0), -U_w / 36)
