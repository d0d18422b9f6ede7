"""Fused peer-memory halo (LBM_HALO_P2P) on the B200.

The boundary-plane collide-stream kernel stores the outgoing directions into
the neighbours' ghost planes and publishes an epoch flag; the neighbour's halo
stream waits on the flag.  Checked here:

* one GPU, periodic z (the slab is its own neighbour): bitwise equal to the
  in-kernel wrap, for every collision kernel and both precisions;
* z-slab decompositions over world = 2, 3, 4, 8 slabs driven from ONE process on
  ONE GPU (direct pointers instead of IPC), bitwise equal to the undecomposed
  lattice ("1 vs 2/4/8 ranks ... must be bitwise-equal"), with
  periodic and walled z, and against the oracle.  The slabs are stepped one at
  a time with a host synchronisation after each call, so every flag a stream
  waits on is already set when the wait is enqueued: no slab's work ever
  waits on another slab's work in flight (no cross-stream dependency on one
  GPU; B200_PROFILING.md on ranks sharing a GPU);
* error paths of the wiring.
"""
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


def _lat(P, w, **kw):
    d = w.params()
    d.update(kw)
    return P.Lattice(**d)


def _slabs(P, w, world, **kw):
    """world slabs of w on cuda:0, wired to each other with direct pointers."""
    hs = [_lat(P, w, rank=r, world=world, halo=P.HALO_P2P, **kw) for r in range(world)]
    blobs = [h.p2p_export() for h in hs]
    for h in hs:
        h.p2p_connect(*P.lbm.p2p_neighbour_blobs(P.lbm.halo_plan(h.p), blobs))
    return hs


def _serial(hs, fn):
    for h in hs:
        fn(h)
        h.sync()


def _split_init(hs, rho, u, f=None):
    n = hs[0].nzl
    for r, h in enumerate(hs):
        if f is None:
            h.init_fields(np.ascontiguousarray(rho[r * n:(r + 1) * n]),
                          np.ascontiguousarray(u[:, r * n:(r + 1) * n]))
        else:
            h.set_populations(np.ascontiguousarray(f[:, r * n:(r + 1) * n]))
        h.sync()


def _gather(hs):
    return np.concatenate([h.get_populations() for h in hs], axis=1)


def _close(hs):
    for h in hs:
        h.close()


KERNELS = {
    "paper_fp64": {},
    "paper_fp32": {"precision": 1},
    "generic_force": {"omega_1": 1.3, "omega_high": 1.1, "omega_xi": 1.2, "force": (1e-5, -2e-5, 3e-5)},
    "raw_model": {"model": 1},
    "full_fd": {"corrections": 3},
    "full_fd_raw_fp32": {"corrections": 3, "model": 1, "precision": 1},
}


@pytest.mark.parametrize("kname", list(KERNELS))
def test_p2p_self_halo_matches_wrap(P, kname):
    w = synth.CONFIGS["weak"].scaled(nx=40, ny=24, nz=12)
    kw = KERNELS[kname]
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 31)
    a = _lat(P, w, **kw)
    b = _lat(P, w, halo=P.HALO_P2P, **kw)
    assert b.info()["halo"] == 2 and a.info()["halo"] == 0
    a.init_fields(rho, u)
    b.init_fields(rho, u)
    a.step(40)
    b.step(40)
    assert np.array_equal(a.get_populations(), b.get_populations())
    a.close()
    b.close()


CASES = {
    # periodic z (ring of slabs), TGV physics
    "tgv_periodic": (synth.CONFIGS["tgv"].scaled(nx=24, ny=13, nz=16), {}),
    # bounce-back z walls + moving lid on +y (cavity), ragged plane
    "cavity_walls": (synth.CONFIGS["cavity100"].scaled(nx=19, ny=11, nz=8), {}),
    # free-slip y walls, periodic z (shear layer geometry), generic rates
    "shear_generic": (synth.CONFIGS["shear"].scaled(nx=16, ny=10, nz=8), {"omega_1": 1.2, "omega_high": 0.9}),
    # duct: force, walls in y and z
    "duct_fp32": (synth.CONFIGS["duct"].scaled(nx=6, ny=14, nz=8), {"precision": 1}),
}
# FULL_FD is not in the slab cases: its step exchanges twice (boundary-plane
# density, then populations), so slab r's step waits for slab r+1's density of
# the SAME step and the slabs cannot be stepped one at a time; on one GPU the
# FULL_FD P2P path is covered by the self-neighbour cases above.


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("case", list(CASES))
def test_p2p_slabs_bitwise_equal_single_lattice(P, case, world):
    w, kw = CASES[case]
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 57)
    ref = _lat(P, w, **kw)
    ref.init_fields(rho, u)
    ref.step(25)
    f_ref = ref.get_populations()
    ref.close()
    hs = _slabs(P, w, world, **kw)
    assert all(h.info()["halo"] == 2 for h in hs)
    _split_init(hs, rho, u)
    for _ in range(25):
        _serial(hs, lambda h: h.step(1))
    f = _gather(hs)
    _close(hs)
    assert np.array_equal(f, f_ref)


def test_p2p_slabs_match_oracle_nonequilibrium(P):
    """world 3 (nz_l = 3), non-equilibrium populations through set_populations,
    walls on every face, against the CPU oracle (fp64 bar 1e-12)."""
    import oracle as O

    w = synth.CONFIGS["cavity1000"].scaled(nx=13, ny=10, nz=9)
    o = O.Oracle(**w.params())
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 91)
    o.init_fields(rho, u)
    f0 = o.get_populations() * (1.0 + 1e-3 * synth.noise((27, w.nz, w.ny, w.nx), 92))
    o.set_populations(f0)
    hs = _slabs(P, w, 3)
    _split_init(hs, None, None, f=f0)
    for _ in range(30):
        _serial(hs, lambda h: h.step(1))
    o.step(30)
    err = np.abs(_gather(hs) - o.get_populations()).max()
    _close(hs)
    assert err <= 1e-12, err


def test_p2p_one_plane_slabs(P):
    """nz_l = 1 (every plane its own slab, both faces in one plane) and nz_l = 2
    (no interior launch)."""
    w = synth.CONFIGS["tgv"].scaled(nx=9, ny=7, nz=4)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 5)
    ref = _lat(P, w)
    ref.init_fields(rho, u)
    ref.step(12)
    f_ref = ref.get_populations()
    ref.close()
    for world in (4, 2):
        hs = _slabs(P, w, world)
        _split_init(hs, rho, u)
        for _ in range(12):
            _serial(hs, lambda h: h.step(1))
        assert np.array_equal(_gather(hs), f_ref), world
        _close(hs)


def test_p2p_timing_and_launch_counts(P):
    w = synth.CONFIGS["weak"].scaled(nx=32, ny=32, nz=16)
    g = _lat(P, w, halo=P.HALO_P2P)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 3)
    g.init_fields(rho, u)
    i0 = g.info()
    g.timing(True)
    g.step(10)
    t = g.timing_read()
    i1 = g.info()
    assert t["launches"] == 10 and t["node_updates"] == 10 * w.nodes and t["kernel_ms"] > 0
    assert i1["collide_stream_launches"] - i0["collide_stream_launches"] == 20  # boundary + interior
    g.close()


def test_p2p_wiring_errors(P):
    w = synth.CONFIGS["tgv"].scaled(nx=8, ny=8, nz=8)
    hs = [_lat(P, w, rank=r, world=2, halo=P.HALO_P2P) for r in range(2)]
    rho, u = synth.random_fields(w.nx, w.ny, 4, 1)
    with pytest.raises(P.LbmError) as e:  # not connected yet
        hs[0].init_fields(rho, u)
    assert e.value.code == P.lbm.LBM_EINVAL
    with pytest.raises(P.LbmError):  # blob of the wrong rank
        hs[0].p2p_connect(hs[0].p2p_export(), hs[0].p2p_export())
    other = _lat(P, w.scaled(nx=9), rank=1, world=2, halo=P.HALO_P2P)
    with pytest.raises(P.LbmError):  # another geometry
        hs[0].p2p_connect(other.p2p_export(), other.p2p_export())
    other.close()
    fd = _lat(P, w, rank=1, world=2, halo=P.HALO_P2P, corrections=3)
    with pytest.raises(P.LbmError):  # another correction mode (density field)
        hs[0].p2p_connect(fd.p2p_export(), fd.p2p_export())
    fd.close()
    b1 = hs[1].p2p_export()
    hs[0].p2p_connect(b1, b1)
    with pytest.raises(P.LbmError):  # twice
        hs[0].p2p_connect(b1, b1)
    with pytest.raises(P.LbmError) as e:
        _lat(P, w, halo=P.HALO_P2P, streaming=1)
    assert e.value.code == P.lbm.LBM_ENOTSUP
    nohalo = _lat(P, w)
    with pytest.raises(P.LbmError):  # no ghost exchange: nothing to export
        nohalo.p2p_export()
    nohalo.close()
    # hs[0] is connected but hs[1] is not: close without publishing (epoch 0)
    _close(hs)


@pytest.mark.parametrize("world,case", [(2, "periodic"), (3, "walls"), (4, "periodic")])
def test_p2p_cuda_ipc_between_processes(P, world, case):
    """The CUDA-IPC wiring (cudaIpcGetMemHandle / cudaIpcOpenMemHandle of the
    torch-allocated buffers and the flag words) between `world` processes on one
    GPU, stepped one rank at a time (scripts/p2p_ipc_check.py)."""
    import os
    import socket
    import subprocess
    import sys

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "scripts", "p2p_ipc_check.py"), "--case", case]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert '"bitwise_equal": true' in r.stdout, r.stdout


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config5_geometry_64cubed_slabs_bitwise(P, world):
    """1 vs 2/4/8 ranks on 64x64x64 bitwise-equal (config 5
    physics: periodic TGV, r = 1, s = 2, nu = 0.01), 30 steps, P2P slabs."""
    w = synth.CONFIGS["weak"].scaled(nx=64, ny=64, nz=64)
    rho, u = synth.initial_fields(w)
    ref = _lat(P, w)
    ref.init_fields(rho, u)
    ref.step(30)
    f_ref = ref.get_populations()
    ref.close()
    hs = _slabs(P, w, world)
    _split_init(hs, rho, u)
    for _ in range(30):
        _serial(hs, lambda h: h.step(1))
    f = _gather(hs)
    _close(hs)
    assert np.array_equal(f, f_ref)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", ["tgv_periodic", "cavity_walls"])
def test_p2p_slabs_run_concurrently_within_a_step(P, case, world):
    """The slabs' steps in flight together: every slab's step(1) is enqueued
    before any is synchronised, so one slab's boundary kernel stores into its
    neighbours' ghost planes and publishes its flag while the neighbours'
    interior and boundary kernels run (4-8 streams on the GPU at once).  Every
    flag wait is on the PREVIOUS step (host-synchronised between steps), so no
    stream waits on another slab's work that is still queued behind it
    (B200_PROFILING.md on ranks sharing a GPU).  Bitwise equal to the
    undecomposed lattice; large enough planes that the launches overlap."""
    w0, kw = CASES[case]
    w = w0.scaled(nx=160, ny=96, nz=8 * world)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 58)
    ref = _lat(P, w, **kw)
    ref.init_fields(rho, u)
    ref.step(20)
    f_ref = ref.get_populations()
    ref.close()
    hs = _slabs(P, w, world, **kw)
    _split_init(hs, rho, u)
    for _ in range(20):
        for h in hs:
            h.step(1)
        for h in hs:
            h.sync()
    f = _gather(hs)
    _close(hs)
    assert np.array_equal(f, f_ref)
