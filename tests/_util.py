"""Test-side helpers: golden-file parsers and closed forms derived independently
of the oracle (they are written from the mathematics, not copied from
oracle/cm_oracle.c)."""
import os
from fractions import Fraction

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# canonical raw-moment order of PAPER.md L606-609 as strings
MOMENTS = ["000", "100", "010", "001", "110", "101", "011", "200", "020", "002", "120", "102",
           "210", "012", "201", "021", "111", "220", "202", "022", "211", "121", "112", "122",
           "212", "221", "222"]


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        for ln in fh:
            ln = ln.split("#", 1)[0].strip()
            if ln:
                yield ln


def appendix_A():
    """27x27 matrix P as printed in App A (rows: moments, cols: populations)."""
    P = np.zeros((27, 27))
    for ln in _lines("appendix_A_P.txt"):
        key, rest = ln.split(":")
        j = MOMENTS.index(key.strip())
        for tok in rest.split():
            P[j, abs(int(tok))] += 1.0 if tok[0] == "+" else -1.0
    return P


def appendix_G(printed_row4=False):
    """27x27 matrix P^-1 as printed in App G (rows: populations, cols: moments)."""
    Pi = np.zeros((27, 27))
    for ln in _lines("appendix_G_Pinv.txt"):
        key, rest = ln.split(":")
        key = key.strip()
        toks = rest.split()
        fac = float(Fraction(toks[0]))
        if key == "4printed":
            if not printed_row4:
                continue
            a = 4
            Pi[a, :] = 0.0
        elif key == "4" and printed_row4:
            continue
        else:
            a = int(key)
        for tok in toks[1:]:
            Pi[a, MOMENTS.index(tok[1:])] += fac * (1.0 if tok[0] == "+" else -1.0)
    return Pi


def eq59_S(r, s):
    d = []
    for ln in _lines("eq59_S_diag.txt"):
        key, rest = ln.split(":")
        pr, ps = map(int, rest.split())
        d.append(r ** pr * s ** ps)
    return np.array(d)


def eq69_rows():
    rows = []
    for ln in _lines("eq69_lid.txt"):
        q, ap, au, sg, kind = ln.split()
        rows.append((int(q), int(ap), int(au), int(sg), kind))
    return rows


def opposite_pairs():
    return [tuple(map(int, ln.split())) for ln in _lines("opposite_pairs.txt")]


# integer velocity signs of Eqs. 1a-1c, re-typed here for the test-side closed
# forms (not imported from either implementation)
EX = [0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1]
EY = [0, 0, 0, 1, -1, 0, 0, 1, 1, -1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, 1, -1, -1, 1, 1, -1, -1]
EZ = [0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, 1, -1, -1, 1, 1, -1, -1, 1, 1, 1, 1, -1, -1, -1, -1]


def _axis_feq(c, cs2, u):
    """1D Maxwellian moments (1, u, cs2 + u^2) on the 3 speeds {0, +c, -c}:
    phi(0) = 1 - (cs2 + u^2)/c^2, phi(+-1) = ((cs2 + u^2)/c^2 +- u/c)/2."""
    a = (cs2 + u * u) / (c * c)
    return {0: 1.0 - a, 1: 0.5 * (a + u / c), -1: 0.5 * (a - u / c)}


def feq_product(r, s, cs2, rho, u):
    """Closed-form D3Q27 cuboid equilibrium: the raw equilibria of Eq. 10
    factorise into per-axis 1D Maxwellian moments, so f^eq is a product."""
    px = _axis_feq(1.0, cs2, u[0])
    py = _axis_feq(r, cs2, u[1])
    pz = _axis_feq(s, cs2, u[2])
    return np.array([rho * px[EX[a]] * py[EY[a]] * pz[EZ[a]] for a in range(27)])


def _axis_g0(c, u):
    a = u * u / (c * c)
    return {0: 1.0 - a, 1: 0.5 * (a + u / c), -1: 0.5 * (a - u / c)}


def _axis_g1(c, u):
    """d/du of g0: the 1D distribution with moments (0, 1, 2u)."""
    return {0: -2.0 * u / (c * c), 1: 0.5 * (2.0 * u / (c * c) + 1.0 / c), -1: 0.5 * (2.0 * u / (c * c) - 1.0 / c)}


def source_product(r, s, u, F):
    """Velocity-space source whose CENTRAL moments are sigma_100..001 = F and 0
    otherwise (Eq. 11c): per axis the raw moments of F_x are d/du_x (u_x^m) u_y^n u_z^p."""
    g0 = [_axis_g0(1.0, u[0]), _axis_g0(r, u[1]), _axis_g0(s, u[2])]
    g1 = [_axis_g1(1.0, u[0]), _axis_g1(r, u[1]), _axis_g1(s, u[2])]
    out = np.zeros(27)
    for a in range(27):
        e = (EX[a], EY[a], EZ[a])
        for d in range(3):
            term = F[d]
            for k in range(3):
                term *= (g1[k] if k == d else g0[k])[e[k]]
            out[a] += term
    return out
