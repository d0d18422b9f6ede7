"""Host logic of the GPU studies (no GPU): the bisection searches of
studies/stability.py with a mocked batch runner, and the analytic solutions."""
import numpy as np

from studies import analytic, stability


def test_bisection_finds_threshold(monkeypatch):
    thresholds = [0.123, 0.3, 0.0071]

    def fake(cases, steps, check_every=5000):
        return [c["wall_u"] <= t for c, t in zip(cases, thresholds)]

    monkeypatch.setattr(stability, "run_batch", fake)
    pts = [dict(model=0, grid=(4, 4, 4), r=1.0, s=1.0, omega_nu=1.5, omega_xi=1.0)] * 3
    lo, hi = stability.bisect(pts, 10, iters=12)
    for l, h, t in zip(lo, hi, thresholds):
        assert l <= t < h and h - l < 0.6 / 2 ** 11


def test_max_reynolds_search(monkeypatch):
    def fake(cases, steps, check_every=5000):
        return [c["omega_nu"] <= 1.9 for c in cases]

    monkeypatch.setattr(stability, "run_batch", fake)
    pts = [dict(model=1, grid=(40, 80, 40), r=0.5, s=1.0, omega_xi=1.0)]
    res = stability.max_reynolds(pts, 10, iters=14)
    assert abs(res[0]["omega_nu_max"] - 1.9) < 1e-3
    nu = 0.08 * (1 / res[0]["omega_nu_max"] - 0.5)
    assert abs(res[0]["Re_max"] - 0.2 * 40 / nu) < 1e-9


def test_womersley_pde_and_walls():
    a, Fm = 20.0, 1e-5
    om = 2 * np.pi / 10000
    nu = a * a * om / 3.09 ** 2

    def u(y, z, t):
        return analytic.womersley(y, z, t, a, Fm, om, nu)

    # u = 0 on the walls (the cosine series of 1 converges like 1/N there)
    scale = Fm / om
    assert abs(u(a, 0.3, 10.0)) < 1e-4 * scale and abs(u(-0.7, -a, 50.0)) < 1e-4 * scale
    y, z, t, h, ht = 3.0, -5.0, 777.0, 1e-2, 1.0
    lap = (u(y + h, z, t) + u(y - h, z, t) + u(y, z + h, t) + u(y, z - h, t) - 4 * u(y, z, t)) / h ** 2
    dt = (u(y, z, t + ht) - u(y, z, t - ht)) / (2 * ht)
    assert abs(dt - (Fm * np.cos(om * t) + nu * lap)) < 1e-3 * Fm
    # low-Wo limit: quasi-steady duct Poiseuille profile at the forcing peak
    om2 = 2 * np.pi / 1e9
    nu2 = 0.1
    ua = analytic.womersley(0.0, 0.0, 0.0, a, Fm, om2, nu2)
    up = analytic.duct_poiseuille(0.0, 0.0, 2 * a, Fm, 1.0, nu2)
    assert abs(ua - up) / up < 1e-4
