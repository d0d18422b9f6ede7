"""The weak linear instability of configs 1/5 (the oracle's von
Neumann analysis in tests/linear_stability.py) observed on
the GPU: config 1 (32x32x16, r = 1, s = 2, nu = 0.01) with omega_xi = 1 grows a
z-Nyquist mode at the rate the analysis predicts for this grid's wavenumbers
(max |lambda| = 1.0038), while omega_xi = omega_nu damps it."""
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


def _nyquist_z(u):
    sign = (-1.0) ** np.arange(u.shape[1])[None, :, None, None]
    return float(np.abs((u * sign).mean(axis=1)).max())


def _amplitudes(P, omega_xi):
    w = synth.CONFIGS["tgv"].scaled(omega_xi=omega_xi)
    g = P.Lattice(**w.params())
    rho, u = synth.initial_fields(w)
    g.init_fields(rho, u)
    amp = []
    for n in (1000, 1000):
        g.step(n)
        amp.append(_nyquist_z(g.get_macroscopic()[1]))
    g.close()
    return amp


def test_linear_instability_rate_matches_analysis(P):
    import sys, os  # noqa: E401

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tests import linear_stability as LS

    o, _ = LS.lattice(1.0, 2.0, 0.01)
    J = LS.collision_jacobian(o, 1.0, 2.0)
    k = [2 * np.pi * np.arange(n) / n for n in (32, 32, 16)]
    K = np.stack(np.meshgrid(*k, indexing="ij"), -1).reshape(-1, 3)
    lam_max = np.abs(LS.eigenvalues(J, K)).max()
    assert 1.003 < lam_max < 1.005
    a1, a2 = _amplitudes(P, 1.0)              # steps 1000 and 2000
    rate = (a2 / a1) ** (1.0 / 1000)          # measured growth factor per step
    assert 1.002 < rate <= lam_max + 1e-4, (rate, lam_max)
    cs2 = synth.auto_cs2(1.0, 2.0)
    b1, b2 = _amplitudes(P, synth.omega_from_nu(0.01, cs2))
    assert b2 < b1 < 1e-6


def test_check_every_reports_the_blow_up(P):
    """params.check_every (SURVEY §5 failure detection): the config-1 run with
    omega_xi = 1 blows up (see above); with check_every = 500 a later step() or
    sync() returns LBM_EUNSTABLE naming the step of the first failed check,
    without blocking the stepping in between.  The stable setting passes."""
    w = synth.CONFIGS["tgv"].scaled(omega_xi=1.0)
    g = P.Lattice(check_every=500, **w.params())
    rho, u = synth.initial_fields(w)
    g.init_fields(rho, u)
    with pytest.raises(P.LbmError) as e:
        for _ in range(40):
            g.step(500)
        g.sync()
    assert e.value.code == P.lbm.LBM_EUNSTABLE and "at step" in str(e.value)
    step = int(str(e.value).split("at step")[1].split()[0])
    assert 5000 < step <= 20000 and step % 500 == 0
    g.close()
    cs2 = synth.auto_cs2(1.0, 2.0)
    w2 = synth.CONFIGS["tgv"].scaled(omega_xi=synth.omega_from_nu(0.01, cs2))
    g2 = P.Lattice(check_every=500, **w2.params())
    g2.init_fields(rho, u)
    g2.step(20000)
    g2.sync()
    g2.close()
