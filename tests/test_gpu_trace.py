"""The event trace of the step structure (lbm_cuboid_trace / _trace_read): one
record per launch on its stream, boundary planes before the exchange, interior
after, NCCL exchange on the halo stream; P2P boundary launch on the halo stream."""
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


@pytest.mark.parametrize("halo", ["nccl", "p2p", "none"])
def test_trace_records_the_step_structure(P, halo):
    w = synth.CONFIGS["tgv"].scaled(nx=64, ny=32, nz=16)
    kw = w.params()
    if halo == "nccl":
        g = P.Lattice(**kw, halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id())
    elif halo == "p2p":
        g = P.Lattice(**kw, halo=P.HALO_P2P)
    else:
        g = P.Lattice(**kw)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 1)
    g.init_fields(rho, u)
    g.trace(True)
    g.step(4)
    rows = g.trace_read()
    g.trace(False)
    assert g.trace_read() == []
    g.close()
    kinds = [r["kind"] for r in rows]
    if halo == "none":
        assert kinds == ["collide"] * 4
    else:
        assert kinds.count("boundary") == 4 and kinds.count("collide") == 4
        assert kinds.count("nccl_halo") == (4 if halo == "nccl" else 0)
        b = [r for r in rows if r["kind"] == "boundary"]
        assert all(r["stream"] == ("halo" if halo == "p2p" else "compute") for r in b)
        assert all(r["zbeg"] == 0 for r in b)
        i = [r for r in rows if r["kind"] == "collide"]
        assert all(r["stream"] == "compute" and r["zbeg"] == 1 and r["nplanes"] == w.nz - 2 for r in i)
        assert all(r["stream"] == "halo" for r in rows if r["kind"] == "nccl_halo")
    assert all(r["t1_ms"] >= r["t0_ms"] >= 0.0 for r in rows)
