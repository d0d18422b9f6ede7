"""Closed-form solutions the paper validates against (no method arithmetic).

womersley(): pulsatile flow in a square duct [-a, a]^2 driven by
F_x = F_m cos(omega t).  The printed series has a wrong
prefactor and coefficient (DESIGN.md erratum E14); re-derived from
d_t u = F/rho + nu lap u with u = 0 on the walls:
  u = Re[ (F_m/(i omega)) (1 - sum_n c_n {cosh(g_n y/a) cos(p_n z/a)
                                          + cosh(g_n z/a) cos(p_n y/a)} / cosh(g_n)) e^{i omega t} ],
  c_n = 2 (-1)^n / p_n,  p_n = (2n+1) pi/2,  g_n^2 = p_n^2 + i Wo^2,  Wo = a sqrt(omega/nu).
duct_poiseuille(): Eq. 70 with the exponent (-1)^((n-1)/2) (erratum E15).
"""
import numpy as np


def womersley(y, z, t, a, Fm, omega, nu, rho=1.0, nterms=400):
    y = np.asarray(y, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    Wo2 = a * a * omega / nu
    acc = np.zeros(np.broadcast(y, z).shape, dtype=np.complex128)
    for n in range(nterms):
        p = (2 * n + 1) * np.pi / 2
        g = np.sqrt(p * p + 1j * Wo2)
        c = 2.0 * (-1) ** n / p
        # cosh(g y/a)/cosh(g), written to avoid overflow for large |g|
        def ch(v):
            return (np.exp(g * (v / a - 1)) + np.exp(-g * (v / a + 1))) / (1 + np.exp(-2 * g))
        acc += c * (ch(y) * np.cos(p * z / a) + ch(z) * np.cos(p * y / a))
    U = (Fm / rho) / (1j * omega) * (1.0 - acc)
    return np.real(U * np.exp(1j * omega * t))


def duct_poiseuille(y, z, L, F, rho, nu, nmax=199):
    acc = 0.0
    for n in range(1, nmax + 1, 2):
        acc = acc + (-1) ** ((n - 1) // 2) * (1 - np.cosh(n * np.pi * z / L) / np.cosh(n * np.pi / 2)) \
            * np.cos(n * np.pi * y / L) / n ** 3
    return 4 * L * L * F / (np.pi ** 3 * rho * nu) * acc
