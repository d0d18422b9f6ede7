"""GPU tests of two round-2 fixes:

* LBM_ESINGULAR (DESIGN reading R17): a node whose strain-rate
  system is singular in flight sets a device flag that
  lbm_cuboid_sync() / lbm_cuboid_check() report.  C_sy = [2cs2/omega_nu -
  (3cs2 - r^2)/2 - 3u_y^2/2] rho vanishes at u_y^2 = (4 cs2/omega_nu -
  (3cs2 - r^2))/3; a 3x3x3 block of nodes at equilibrium with that velocity
  makes the centre node (which pulls only from the block) singular.  The
  oracle counts the same node.
* AA streaming with the moving lid: the odd step's Eq. 69 density rho_f comes
  from a side array written by the even step (reading the node's 27 slots raced
  with the neighbour threads' pushes on multi-wave grids).  AA must equal the
  two-buffer path on the full 256x256x128 config-3 cavity.
"""
import numpy as np
import pytest

import synth
from tests import _util as U

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2107_14774_b200 as P

    P.load()
    return P


def _singular_state(r, s, cs2, omega_nu, frac=1.0, n=(9, 8, 7)):
    """Rest state with a 3x3x3 block at equilibrium with u_y = frac * u_y*."""
    uy2 = (4.0 * cs2 / omega_nu - (3.0 * cs2 - r * r)) / 3.0
    uy = frac * np.sqrt(uy2)
    nx, ny, nz = n
    f = np.empty((27, nz, ny, nx))
    f[...] = U.feq_product(r, s, cs2, 1.0, (0.0, 0.0, 0.0))[:, None, None, None]
    blk = U.feq_product(r, s, cs2, 1.0, (0.0, uy, 0.0))
    f[:, 2:5, 3:6, 3:6] = blk[:, None, None, None]
    return f


@pytest.mark.parametrize("kind", ["paper", "generic", "raw"])
def test_singular_node_is_reported(P, kind):
    import oracle as O

    r, s, cs2, wn = 1.0, 2.0, 1.0 / 3.0, 1.6
    kw = dict(nx=9, ny=8, nz=7, r=r, s=s, cs2=cs2, omega_nu=wn, omega_xi=1.0, corrections=0)
    if kind == "generic":
        kw.update(omega_1=1.2, omega_high=0.9)
    if kind == "raw":
        kw.update(model=1)
    f = _singular_state(r, s, cs2, wn)
    o = O.Oracle(**kw)
    O.singular_count(reset=True)
    o.set_populations(f)
    o.step(1)
    assert O.singular_count(reset=True) == 1  # the block's centre node only
    g = P.Lattice(**kw, graphs=1)
    g.set_populations(f)
    g.step(1)
    with pytest.raises(P.LbmError) as ei:
        g.sync()
    assert ei.value.code == P.lbm.LBM_ESINGULAR
    g.sync()  # reported once, then cleared
    g.close()
    # control: 0.9 u_y* is regular on both sides
    f = _singular_state(r, s, cs2, wn, frac=0.9)
    o.set_populations(f)
    o.step(1)
    assert O.singular_count(reset=True) == 0
    g = P.Lattice(**kw, graphs=1)
    g.set_populations(f)
    g.step(3)
    g.sync()
    g.check()
    g.close()


@pytest.mark.parametrize("prec", [0, 1])
def test_aa_equals_ab_on_full_config3_cavity(P, prec):
    """Config 3 at full size (256x256x128, six walls, Eq. 69 lid at U = 0.05),
    seeded rough start, 24 steps: AA in place == two-buffer AB (max|df| <= 1e-13
    fp64; the lid density rho_f differs only by the rounding of sum f~ vs the
    collision's rho)."""
    w = synth.CONFIGS["cavity1000"].scaled(precision=prec)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 77)
    a = P.Lattice(**w.params(), streaming=0)
    b = P.Lattice(**w.params(), streaming=1)
    a.init_fields(rho, u)
    b.init_fields(rho, u)
    for n in (1, 23):  # odd and even phase of AA
        a.step(n)
        b.step(n)
        fa, fb = a.get_populations(), b.get_populations()
        d = np.abs(fa - fb).max()
        assert d <= (1e-13 if prec == 0 else 2e-7), (n, d)
    a.close()
    b.close()
