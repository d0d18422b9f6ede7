"""Pins of the oracle's algebra (no GPU).  Each test names what fixes the value:
a paper-printed object (tests/golden/*, with citation), a closed form, an
invariant, or a textbook special case.  A transposed operand, a dropped term or
a wrong sign in oracle/cm_oracle.c fails at least one of these."""
import numpy as np
import pytest

import oracle as O
from tests import _util as U

RS = [(1.0, 1.0), (1.0, 2.0), (0.5, 1.0), (0.406, 1.3), (0.5, 0.33), (0.75, 1.0)]


def _cs2(r, s):
    return min(1.0, r * r, s * s) / 3.0


def test_velocity_set_and_opposites(golden_dir):
    """Eqs. 1a-1c: lattice symmetry; opposite pairs as listed at PAPER.md L753-757."""
    e = O.velocities(0.5, 2.0)
    assert e.shape == (27, 3)
    assert np.allclose(e.sum(axis=0), 0.0)
    # second moments: 18 directions have e_x != 0, etc. (Eq. 1)
    assert np.isclose((e[:, 0] ** 2).sum(), 18.0)
    assert np.isclose((e[:, 1] ** 2).sum(), 18.0 * 0.25)
    assert np.isclose((e[:, 2] ** 2).sum(), 18.0 * 4.0)
    opp = O.opposite()
    for a in range(27):
        assert np.allclose(e[opp[a]], -e[a])
    for qbar, q in U.opposite_pairs():
        assert opp[q] == qbar and opp[qbar] == q
    assert opp[0] == 0


def test_Q_at_unit_aspect_is_appendix_A(golden_dir):
    """App A prints m = P f; the oracle's Q(1,1) must be P."""
    assert np.array_equal(O.Q(1.0, 1.0), U.appendix_A())


@pytest.mark.parametrize("r,s", RS)
def test_Q_is_S_times_P(r, s):
    """Eq. 58/59: Q = S P with S = diag(r^n s^p) as printed."""
    S = U.eq59_S(r, s)
    assert np.allclose(O.Q(r, s), S[:, None] * U.appendix_A(), rtol=1e-15, atol=0)


def test_Qinv_at_unit_aspect_is_appendix_G():
    """App G prints P^-1; the oracle's numeric inverse of
    Q(1,1) reproduces every row except the printed f_4 row (erratum E1)."""
    Qi = O.invert27(O.Q(1.0, 1.0))
    assert np.allclose(Qi, U.appendix_G(), atol=1e-14)
    printed = U.appendix_G(printed_row4=True)
    assert not np.allclose(Qi[4], printed[4], atol=1e-3)
    assert np.allclose(np.delete(Qi, 4, 0), np.delete(printed, 4, 0), atol=1e-14)


@pytest.mark.parametrize("r,s", RS)
def test_Qinv_is_Pinv_Sinv(r, s):
    """Eq. 60/61: Q^-1 = P^-1 S^-1, and Q^-1 Q = I."""
    Q = O.Q(r, s)
    Qi = O.invert27(Q)
    assert np.allclose(Qi @ Q, np.eye(27), atol=1e-13)
    assert np.allclose(Qi, U.appendix_G() / U.eq59_S(r, s)[None, :], rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("seed", range(5))
def test_central_moments_literal_equals_binomial_of_raw(seed):
    """Eq. 3a (literal) = F(u) S P f (binomial transform of raw moments)."""
    rng = np.random.default_rng(seed)
    r, s = RS[seed % len(RS)]
    f = rng.uniform(0.0, 1.0, 27)
    u = rng.uniform(-0.3, 0.3, 3)
    e = O.velocities(r, s)
    k_lit = O.central_moments(e, f, u)
    k_bin = O.frame(O.Q(r, s) @ f, -u)
    assert np.allclose(k_lit, k_bin, rtol=1e-13, atol=1e-14)
    # u = 0: central = raw
    assert np.allclose(O.central_moments(e, f, np.zeros(3)), O.Q(r, s) @ f, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("seed", range(5))
def test_frame_inverse_is_minus_u(seed):
    """F^-1 = F(-u): round trip is the identity for |u| <= 0.3."""
    rng = np.random.default_rng(100 + seed)
    m = rng.normal(size=27)
    u = rng.uniform(-0.3, 0.3, 3)
    assert np.allclose(O.frame(O.frame(m, -u), u), m, rtol=1e-13, atol=1e-14)
    assert np.allclose(O.frame(O.frame(m, u), -u), m, rtol=1e-13, atol=1e-14)


def test_frame_is_lower_triangular_with_unit_diagonal():
    """F is lower triangular in the canonical order; unit diagonal."""
    u = np.array([0.1, -0.2, 0.15])
    F = np.stack([O.frame(np.eye(27)[j], -u) for j in range(27)], axis=1)
    order = [sum(map(int, m)) for m in U.MOMENTS]
    for i in range(27):
        for j in range(27):
            if order[j] > order[i]:
                assert F[i, j] == 0.0
    assert np.allclose(np.diag(F), 1.0)


@pytest.mark.parametrize("r,s", RS)
def test_feq_equals_closed_product_form(r, s):
    """f^eq = Q^-1 m^eq (Eq. 10) equals the per-axis product form."""
    rng = np.random.default_rng(7)
    cs2 = _cs2(r, s)
    o = O.Oracle(2, 2, 2, r, s, cs2, 1.5)
    for _ in range(5):
        rho = rng.uniform(0.9, 1.1)
        u = rng.uniform(-0.1, 0.1, 3)
        assert np.allclose(o.feq(rho, u), U.feq_product(r, s, cs2, rho, u), rtol=1e-13, atol=1e-16)


def test_feq_textbook_d3q27_weights():
    """r = s = 1, cs2 = 1/3, u = 0: the standard D3Q27 weights 8/27, 2/27, 1/54, 1/216."""
    o = O.Oracle(2, 2, 2, 1.0, 1.0, 1.0 / 3.0, 1.0)
    w = o.feq(1.0, np.zeros(3))
    nnz = np.array([abs(U.EX[a]) + abs(U.EY[a]) + abs(U.EZ[a]) for a in range(27)])
    expect = np.choose(nnz, [8 / 27, 2 / 27, 1 / 54, 1 / 216])
    assert np.allclose(w, expect, rtol=1e-14)


@pytest.mark.parametrize("r,s", RS)
def test_raw_equilibria_shift_to_maxwellian_central(r, s):
    """Eq. 10 is the binomial transform of Eq. 9: central moments of f^eq are
    rho, 0, cs2 rho, cs4 rho, cs6 rho."""
    cs2 = _cs2(r, s)
    rho, u = 1.03, np.array([0.04, -0.03, 0.02])
    o = O.Oracle(2, 2, 2, r, s, cs2, 1.5)
    k = O.central_moments(O.velocities(r, s), o.feq(rho, u), u)
    expect = np.zeros(27)
    for j, m in enumerate(U.MOMENTS):
        nd = [int(c) for c in m]
        if all(n % 2 == 0 for n in nd):
            expect[j] = rho * cs2 ** (sum(nd) // 2)
    assert np.allclose(k, expect, atol=2e-15)


def test_hydro_eq12():
    """Eq. 12: rho = sum f, rho u = sum f e + F/2."""
    rng = np.random.default_rng(3)
    e = O.velocities(0.5, 1.3)
    f = rng.uniform(0, 0.1, 27)
    F = np.array([1e-3, -2e-3, 5e-4])
    rho, u = O.hydro(e, f, F)
    assert np.isclose(rho, f.sum())
    assert np.allclose(rho * u, f @ e + F / 2)
