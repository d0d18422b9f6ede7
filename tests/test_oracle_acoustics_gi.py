"""Pins P10 and P11 of the oracle (no GPU).

P10 -- bulk viscosity and acoustic isotropy: a standing sound wave along each
axis is attenuated at k^2 (2 nu/3 + xi/2) (linearised Eq. 51 with xi from Eq. 53,
P:L433-440) equally along x, y and z, for several omega_xi; without the
corrections the stretched axes are off by > 3x.

P11 -- Galilean invariance of the aliasing terms (the 3u^2 parts of theta and C,
P:L1171-1196): a shear (2D Taylor-Green) mode riding a uniform flow U_b = 0.1
decays at the rate it has at rest with FULL_LOCAL; LOW_MACH (3u^2 terms dropped,
P:L448-465) shifts it by > 1.5 %.
"""
import numpy as np
import pytest

import oracle as O
import synth

FULL, LOW, OFF = 0, 1, 2


def _standing_sound_rate(corr, axis, r, s, wxi, nphys=64, nu=0.02, amp=1e-5, steps=400):
    cs2 = synth.auto_cs2(r, s)
    h = {"x": 1.0, "y": r, "z": s}[axis]
    n = int(round(nphys / h))
    shape = {"x": (1, 1, n), "y": (1, n, 1), "z": (n, 1, 1)}[axis]
    nz, ny, nx = shape
    o = O.Oracle(nx, ny, nz, r, s, cs2, synth.omega_from_nu(nu, cs2), omega_xi=wxi, corrections=corr)
    c = (np.arange(n) * h).reshape(shape)
    k = 2 * np.pi / nphys
    o.init_fields(1 + amp * np.cos(k * c), np.zeros((3,) + shape))
    basis = np.exp(-1j * k * c)
    d = "xyz".index(axis)
    cs = np.sqrt(cs2)
    ts, en = [], []
    for t in range(steps):
        o.step(1)
        if t >= 50:
            rho, u = o.macroscopic()
            a = ((rho - 1) * basis).sum()
            b = (u[d] * basis).sum() / cs  # acoustic energy ~ |rho'|^2 + |u'/cs|^2
            ts.append(t)
            en.append(np.log(abs(a) ** 2 + abs(b) ** 2))
    rate = -np.polyfit(ts, en, 1)[0] / 2
    xi = (2 * cs2 / 3) * (1 / wxi - 0.5)
    return rate / (k * k * (2 * nu / 3 + xi / 2))


@pytest.mark.parametrize("r,s", [(1.0, 2.0), (0.5, 1.0)])
def test_acoustic_attenuation_isotropic_with_bulk_viscosity(r, s):
    for wxi in (0.8, 1.6):
        rates = [_standing_sound_rate(FULL, ax, r, s, wxi) for ax in "xyz"]
        assert max(rates) - min(rates) < 0.01, rates
        assert all(abs(x - 1.0) < 0.03 for x in rates), rates
    stretched = "z" if (r, s) == (1.0, 2.0) else "x"
    assert _standing_sound_rate(OFF, stretched, r, s, 1.0) > 3.0


def _shear_rate_moving(corr, r, s, Ub, plane, nphys=32, nu=0.02, amp=1e-5, steps=300):
    cs2 = synth.auto_cs2(r, s)
    sp = {"x": 1.0, "y": r, "z": s}
    n = {d: (int(round(nphys / sp[d])) if d in plane else 1) for d in "xyz"}
    o = O.Oracle(n["x"], n["y"], n["z"], r, s, cs2, synth.omega_from_nu(nu, cs2), corrections=corr)
    k = 2 * np.pi / nphys
    Z, Y, X = np.meshgrid(np.arange(n["z"]) * s, np.arange(n["y"]) * r, np.arange(n["x"]) * 1.0,
                          indexing="ij")
    c = {"x": X, "y": Y, "z": Z}
    a, b = plane
    ia, ib = "xyz".index(a), "xyz".index(b)
    u = np.zeros((3,) + X.shape)
    u[ia] = Ub + amp * np.sin(k * c[a]) * np.cos(k * c[b])
    u[ib] = -amp * np.cos(k * c[a]) * np.sin(k * c[b])
    o.init_fields(np.ones(X.shape), u)
    basis = np.exp(-1j * k * (c[a] + c[b]))  # |mode| is invariant to advection
    ts, amps = [], []
    for t in range(steps):
        o.step(1)
        if t >= 50 and t % 10 == 0:
            ts.append(t)
            amps.append(np.log(abs((o.macroscopic()[1][ib] * basis).sum())))
    return -np.polyfit(ts, amps, 1)[0] / (2 * nu * k * k)


@pytest.mark.parametrize("r,s,plane", [(1.0, 1.0, "xy"), (1.0, 2.0, "xz")])
def test_galilean_invariance_of_aliasing_terms(r, s, plane):
    rest = _shear_rate_moving(FULL, r, s, 0.0, plane)
    full = _shear_rate_moving(FULL, r, s, 0.1, plane)
    low = _shear_rate_moving(LOW, r, s, 0.1, plane)
    assert abs(full - rest) < 0.002, (full, rest)
    assert abs(low - rest) > 0.015, (low, rest)
