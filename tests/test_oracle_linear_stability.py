"""Linear stability of the oracle's scheme at the BASELINE configs (SURVEY §8(c)
P13; tests/linear_stability.py), no GPU.

* configs 2, 3 (Re 100 and 1000) and 4 are linearly stable: every Fourier mode
  of the linearised pull-streamed update has |lambda| <= 1;
* configs 1/5 (nu = 0.01 at r = 1, s = 2, omega_xi = 1) are weakly unstable at
  a z-Nyquist mode (|lambda| ~ 1.0036 on a 25^3 grid, as P13 predicts from an
  independent analysis), and stable with omega_xi = omega_nu or without the
  corrections;
* the least-damped transverse mode at long wavelength decays at nu k^2 (Eq. 53)
  along y and z, with k the physical wavenumber (kappa / r, kappa / s)."""
import numpy as np
import pytest

import synth
from tests import linear_stability as LS

N = 15  # odd: the grid holds the Nyquist wavenumber and never kappa = 0


def _growth(case):
    return LS.run_case(case, N)["max_abs_lambda"]


@pytest.mark.parametrize("case", ["config2_duct", "config3_cavity_re100", "config3_cavity_re1000",
                                  "config4_shear_layer", "config1_5_omega_xi_eq_omega_nu",
                                  "config1_5_corrections_off"])
def test_stable_configurations(case):
    assert _growth(case) <= 1.0 + 1e-9


def test_config1_5_weakly_unstable_at_z_nyquist():
    r = LS.run_case("config1_5_tgv", 25)
    assert 1.002 < r["max_abs_lambda"] < 1.01
    assert abs(abs(r["at_kappa"][2]) - np.pi) < 1e-12  # the z-Nyquist mode


@pytest.mark.parametrize("axis", [1, 2])
@pytest.mark.parametrize("r,s,nu", [(1.0, 2.0, 0.05), (0.5, 1.0, 0.01)])
def test_shear_eigenvalue_matches_viscosity(r, s, nu, axis):
    o, cs2 = LS.lattice(r, s, nu)
    J = LS.collision_jacobian(o, r, s)
    h = (1.0, r, s)[axis]
    kappa = np.zeros(3)
    kappa[axis] = 2 * np.pi / 64  # index-space wavenumber
    k = kappa[axis] / h           # physical wavenumber
    lam = LS.eigenvalues(J, kappa[None, :])[0]
    rates = -np.log(np.abs(lam))
    # the two transverse (shear) modes: real eigenvalues closest to exp(-nu k^2)
    best = rates[np.argmin(np.abs(rates - nu * k * k))]
    assert best / (nu * k * k) == pytest.approx(1.0, abs=0.01)


def test_central_moments_linearly_more_robust_than_raw_moments():
    """Section 7 of the paper: the central-moment scheme is more
    robust than the raw-moment one.  Linear counterpart on the (0.5, 1) lattice
    with cs2 = 0.08 and omega_nu = 1.6: the largest uniform flow speed for which
    every Fourier mode is damped is larger for 3DCCM than for 3DCRM."""
    cm = LS.max_stable_speed(0.5, 1.0, 0.08, 1.6, model=0, n=11, du=0.025)
    rm = LS.max_stable_speed(0.5, 1.0, 0.08, 1.6, model=1, n=11, du=0.025)
    assert cm is not None and rm is not None and cm > rm
