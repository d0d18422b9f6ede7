"""The plane-shape specialisations of the paper-rate kernel
(k_collide_stream_paper_shape: nx, ny compile-time for the BASELINE config 3-5
planes, so the interior path's 27 load and 27 store offsets are immediates)
against the general kernel (LBM_SHAPE_SPEC=0), bit for bit: the same inlined
per-node code, only the address arithmetic differs.  Walls with the lid, free
slip, periodic wrap, fp64 and fp32 storage, CUDA graphs and the NCCL
ghost-plane path (strided boundary planes)."""
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


CASES = {
    "cavity_256x256": synth.CONFIGS["cavity1000"].scaled(nz=6),
    "shear_512x256": synth.CONFIGS["shear"].scaled(nz=4),
    "tgv_512x512": synth.CONFIGS["weak"].scaled(nz=4),
    "tgv_1024x1024": synth.CONFIGS["strong"].scaled(nz=2),
}


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("case", list(CASES))
def test_shape_kernel_bitwise_equal_general_kernel(P, case, prec, monkeypatch):
    w = CASES[case].scaled(precision=prec)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 88)
    monkeypatch.setenv("LBM_SHAPE_SPEC", "0")
    a = P.Lattice(**w.params(), graphs=1)
    monkeypatch.delenv("LBM_SHAPE_SPEC")
    hs = [P.Lattice(**w.params(), graphs=1), P.Lattice(**w.params(), graphs=2)]
    if w.bc[4] == synth.BC_PERIODIC:
        hs.append(P.Lattice(**w.params(), halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id()))
    for g in [a] + hs:
        g.init_fields(rho, u)
        g.step(6)
    fa = a.get_populations()
    a.close()
    for g in hs:
        assert np.array_equal(fa, g.get_populations())
        g.close()


@pytest.mark.parametrize("corr", [synth.CORR_FULL_FD, synth.CORR_FULL_FD_LAG])
@pytest.mark.parametrize("case", ["cavity_256x256", "tgv_512x512"])
def test_shape_kernel_with_density_gradient_terms(P, case, corr, monkeypatch):
    """FULL_FD (two-pass collide) and FULL_FD_LAG through the shape kernel: the
    26-neighbour density stencil with immediate offsets, bit for bit."""
    w = CASES[case].scaled(corrections=corr)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 89)
    monkeypatch.setenv("LBM_SHAPE_SPEC", "0")
    a = P.Lattice(**w.params(), graphs=1)
    monkeypatch.delenv("LBM_SHAPE_SPEC")
    b = P.Lattice(**w.params(), graphs=1)
    for g in (a, b):
        g.init_fields(rho, u)
        g.step(6)
    assert np.array_equal(a.get_populations(), b.get_populations())
    a.close()
    b.close()


def test_kernel_name_reports_the_launched_variant(P, monkeypatch):
    w = CASES["tgv_512x512"]
    g = P.Lattice(**w.params())
    assert g.kernel_name() == "k_collide_stream_paper_shape<double,512,512>"
    g.close()
    g = P.Lattice(**w.scaled(nx=96, ny=40, precision=1).params())
    assert g.kernel_name() == "k_collide_stream_paper<float>"
    g.close()
    g = P.Lattice(**w.scaled(nx=40, ny=40, corrections=synth.CORR_FULL_FD).params())
    assert g.kernel_name() == "k_collide_stream_paper<double> + k_density"
    g.close()
    g = P.Lattice(**w.scaled(nx=96, ny=40, corrections=synth.CORR_FULL_FD).params())
    assert g.kernel_name() == "k_collide_stream_fd_tma<double>"  # 9 of 10 tile rows staged
    g.close()
    monkeypatch.setenv("LBM_SHAPE_SPEC", "0")
    g = P.Lattice(**w.scaled(model=1).params())
    assert g.kernel_name() == "k_collide_stream_raw<double>"
    g.close()


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("case", ["cavity_256x256", "shear_512x256", "tgv_512x512"])
def test_shape_aa_kernels_bitwise_equal_general(P, case, prec, monkeypatch):
    """AA in-place streaming through k_aa_shape (interior warps pull reversed
    slots and push at constant offsets) against the general AA kernels, after
    an odd and an even number of steps (both layouts), lid included."""
    w = CASES[case].scaled(precision=prec)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 90)
    monkeypatch.setenv("LBM_SHAPE_SPEC", "0")
    a = P.Lattice(**w.params(), streaming=1, graphs=1)
    monkeypatch.delenv("LBM_SHAPE_SPEC")
    b = P.Lattice(**w.params(), streaming=1, graphs=1)
    assert b.kernel_name().startswith("k_aa_shape<")
    for g in (a, b):
        g.init_fields(rho, u)
    for n in (5, 6):
        a.step(n)
        b.step(n)
        assert np.array_equal(a.get_populations(), b.get_populations()), n
    a.close()
    b.close()
