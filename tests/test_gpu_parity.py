"""GPU parity: the CUDA path (through the C ABI via the thin binding) against the
CPU oracle, element by element, on the same seeded inputs.

Tolerances: fp64 max|df| <= 1e-12 after 100 steps
(BASELINE.json north_star); fp32 storage max |df|/|f| <= 1e-5 (reading R12).
Sizes: small enough for the oracle (~0.6 MLUPS) to finish in seconds, chosen to
span several 128-thread blocks with ragged tails (nx*ny not a multiple of 128).
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2107_14774_b200 as P

    P.load()
    return P


def _oracle(w):
    import oracle as O

    return O.Oracle(**w.params())


def _gpu(P, w, **kw):
    d = w.params()
    d.update(kw)
    return P.Lattice(**d)


def _init_both(P, w, seed=None, noneq=0.0, **kw):
    o = _oracle(w)
    g = _gpu(P, w, **kw)
    if seed is None:
        rho, u = synth.initial_fields(w)
    else:
        rho, u = synth.random_fields(w.nx, w.ny, w.nz, seed)
    o.init_fields(rho, u)
    if noneq:
        f = o.get_populations() * (1.0 + noneq * synth.noise((27, w.nz, w.ny, w.nx), 1000 + (seed or 0)))
        o.set_populations(f)
        g.set_populations(f)
    else:
        g.init_fields(rho, u)
    return o, g


def _cmp(o, g, prec=0):
    fo = o.get_populations()
    fg = g.get_populations()
    assert np.all(np.isfinite(fg))
    if prec == 0:
        err = np.abs(fg - fo).max()
        assert err <= TOL64, err
    else:
        err = (np.abs(fg - fo) / np.abs(fo)).max()
        assert err <= TOL32, err
    return err


CASES = {
    # name: (workload, reduced grid)
    "tgv_full": synth.CONFIGS["tgv"],
    "duct": synth.CONFIGS["duct"].scaled(nx=5, ny=37, nz=19),
    "cavity100": synth.CONFIGS["cavity100"].scaled(nx=21, ny=19, nz=11),
    "cavity1000": synth.CONFIGS["cavity1000"].scaled(nx=17, ny=23, nz=9),
    "shear": synth.CONFIGS["shear"].scaled(nx=16, ny=29, nz=12),
    "weak_tgv": synth.CONFIGS["weak"].scaled(nx=40, ny=24, nz=12),
}


@pytest.mark.parametrize("name", list(CASES))
def test_parity_fp64_100_steps(P, name):
    w = CASES[name]
    o, g = _init_both(P, w, seed=7)
    _cmp(o, g)  # initialisation (reading R8)
    o.step(100)
    g.step(100)
    _cmp(o, g)


def test_parity_config2_duct_full_size(P):
    """BASELINE config 2 at its full size (8x128x64, force, walls in y and z),
    100 steps from non-equilibrium populations, element by element (the oracle
    needs ~10 s for these 6.6 M node updates)."""
    w = synth.CONFIGS["duct"]
    o, g = _init_both(P, w, seed=17, noneq=1e-3)
    o.step(100)
    g.step(100)
    _cmp(o, g)
    g.close()


@pytest.mark.parametrize("name", ["tgv_full", "cavity100", "shear", "duct"])
def test_parity_fp32_storage(P, name):
    w = CASES[name].scaled(precision=synth.PREC_FP32)
    o, g = _init_both(P, w, seed=3)
    # the GPU stores fp32: compare after the same 100 steps relative to the fp64 oracle
    o.step(100)
    g.step(100)
    _cmp(o, g, prec=1)


@pytest.mark.parametrize("corr", [synth.CORR_LOW_MACH, synth.CORR_OFF])
def test_parity_correction_modes(P, corr):
    w = CASES["weak_tgv"].scaled(corrections=corr)
    o, g = _init_both(P, w, seed=11, noneq=1e-3)
    o.step(50)
    g.step(50)
    _cmp(o, g)


def test_parity_generic_rates_and_force(P):
    """omega_1, omega_high != 1 (all App D relaxations active), body force, OFF-axis
    aspect ratios."""
    w = synth.Workload("generic", 19, 13, 10, r=0.75, s=1.3, nu=0.02, omega_xi=1.4, omega_1=1.2,
                       omega_high=0.9, force=(2e-5, -1e-5, 5e-6), init="random", seed=5)
    o, g = _init_both(P, w, seed=5, noneq=1e-3)
    o.step(60)
    g.step(60)
    _cmp(o, g)


def test_parity_nonequilibrium_walls(P):
    """All wall kinds with a non-equilibrium start: moving lid + bounce-back box."""
    w = CASES["cavity100"]
    o, g = _init_both(P, w, seed=13, noneq=2e-3)
    o.step(80)
    g.step(80)
    _cmp(o, g)


@pytest.mark.parametrize("shape", [(1, 1, 1), (1, 7, 5), (3, 1, 4), (6, 5, 1), (130, 1, 2)])
def test_parity_degenerate_grids(P, shape):
    """Degenerate extents (1 node along an axis wraps onto itself)."""
    nx, ny, nz = shape
    w = synth.CONFIGS["weak"].scaled(nx=nx, ny=ny, nz=nz, init="random")
    o, g = _init_both(P, w, seed=17, noneq=1e-3)
    o.step(30)
    g.step(30)
    _cmp(o, g)


def test_parity_duct_walls_thin(P):
    """Walls on both faces of a 1-node-thick axis (bounce-back twice per link)."""
    w = synth.CONFIGS["duct"].scaled(nx=3, ny=1, nz=6)
    o, g = _init_both(P, w, seed=19, noneq=1e-3)
    o.step(30)
    g.step(30)
    _cmp(o, g)


def test_nccl_self_halo_matches_wrap(P):
    """LBM_HALO_NCCL on one GPU (send-to-self ghost planes) gives bitwise the
    same result as the in-kernel z wrap."""
    w = CASES["weak_tgv"]
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 23)
    a = _gpu(P, w)
    uid = P.nccl_unique_id()
    b = _gpu(P, w, halo=P.HALO_NCCL, nccl_uid=uid)
    assert b.info()["halo"] == 1 and a.info()["halo"] == 0
    a.init_fields(rho, u)
    b.init_fields(rho, u)
    a.step(40)
    b.step(40)
    assert np.array_equal(a.get_populations(), b.get_populations())


def test_zero_steps_and_roundtrips(P):
    w = CASES["shear"]
    g = _gpu(P, w)
    rho, u = synth.initial_fields(w)
    g.init_fields(rho, u)
    r2, u2 = g.get_macroscopic()
    assert np.abs(r2 - rho).max() < 1e-14 and np.abs(u2 - u).max() < 1e-15
    f = g.get_populations()
    g.step(0)
    assert np.array_equal(f, g.get_populations())
    f2 = f * (1 + 1e-3 * synth.noise(f.shape, 4))
    g.set_populations(f2)
    assert np.array_equal(f2, g.get_populations())
    fp = g.get_populations_planes(3, 4)
    assert np.array_equal(fp, f2[:, 3:7])


def test_device_init_and_macroscopic(P):
    import torch

    w = CASES["weak_tgv"]
    g = _gpu(P, w)
    rho, u = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0, xp=torch, device="cuda")
    g.init_fields(rho, u)
    g.step(5)
    rd, ud = g.get_macroscopic(device=True)
    torch.cuda.synchronize()
    rh, uh = g.get_macroscopic()
    assert np.array_equal(rd.cpu().numpy(), rh) and np.array_equal(ud.cpu().numpy(), uh)


def test_conservation_and_check(P):
    w = CASES["cavity1000"]
    g = _gpu(P, w)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 29, rho_amp=1e-3, u_amp=1e-3)
    g.init_fields(rho, u)
    m0 = g.check()["mass"]
    g.step(300)
    d = g.check()
    assert abs(d["mass"] - m0) / m0 < 1e-12
    assert d["bad_nodes"] == 0 and d["max_speed"] < 0.2
    f = g.get_populations()
    f[5, 1, 2, 3] = np.nan
    g.set_populations(f)
    with pytest.raises(P.LbmError):
        g.check()


def test_invalid_parameters_raise(P):
    w = CASES["tgv_full"]
    with pytest.raises(P.LbmError):
        _gpu(P, w, omega_nu=2.5)
    with pytest.raises(P.LbmError):
        _gpu(P, w, bc=(2, 2, 0, 0, 0, 0))  # moving wall off the +y face
    with pytest.raises(P.LbmError):
        _gpu(P, w, cs2=1.5)


def _tgv_patch_oracle(w, nx, ny, nz, xs, ys, zs):
    """Oracle update of single nodes of the full-size periodic TGV after one
    step: a 3x3x3 periodic patch of the initial fields around each node
    reproduces exactly the node's 27 pull sources."""
    import oracle as O

    out = []
    d = w.params()
    d.update(nx=3, ny=3, nz=3)
    o = O.Oracle(**d)
    for x, y, z in zip(xs, ys, zs):
        X = 2 * np.pi * (((x + np.arange(-1, 2)) % nx) / nx)
        Y = 2 * np.pi * (((y + np.arange(-1, 2)) % ny) / ny)
        Z = 2 * np.pi * (((z + np.arange(-1, 2)) % nz) / nz)
        Zg, Yg, Xg = np.meshgrid(Z, Y, X, indexing="ij")
        u = np.zeros((3, 3, 3, 3))
        u[0] = w.u0 * np.sin(Xg) * np.cos(Yg) * np.cos(Zg)
        u[1] = -w.u0 * np.cos(Xg) * np.sin(Yg) * np.cos(Zg)
        rho = 1.0 + (w.u0 ** 2 / 16) * (np.cos(2 * Xg) + np.cos(2 * Yg)) * (np.cos(2 * Zg) + 2.0) / w.cs2_value
        o.init_fields(rho, u)
        o.step(1)
        out.append(o.get_populations()[:, 1, 1, 1])
    return np.array(out)


@pytest.mark.parametrize("precision", [0, 1])
def test_full_size_bench_config_sampled(P, precision):
    """BASELINE config 5 (weak, 512^3 per GPU, r=1, s=2) in the launch
    configuration bench.py times: one step on the full grid, sampled nodes
    (incl. all faces/edges/corners of the periodic box) against the oracle."""
    import torch

    w = synth.CONFIGS["weak"].scaled(precision=precision)
    g = _gpu(P, w)
    rho, u = synth.tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0, xp=torch, device="cuda")
    g.init_fields(rho, u)
    del rho, u
    g.step(1)
    rng = np.random.default_rng(1)
    planes = [0, 1, 255, 510, 511]
    for z in planes:
        fz = g.get_populations_planes(z, 1)[:, 0]
        xs = np.concatenate([[0, w.nx - 1, 0, w.nx - 1], rng.integers(0, w.nx, 6)])
        ys = np.concatenate([[0, 0, w.ny - 1, w.ny - 1], rng.integers(0, w.ny, 6)])
        ref = _tgv_patch_oracle(w, w.nx, w.ny, w.nz, xs, ys, [z] * len(xs))
        got = fz[:, ys, xs].T
        if precision == 0:
            assert np.abs(got - ref).max() <= TOL64
        else:
            assert (np.abs(got - ref) / np.abs(ref)).max() <= TOL32
    d = g.check()
    assert d["bad_nodes"] == 0


# ------------------------------------------------------------ 3DCRM (raw moments)
@pytest.mark.parametrize("name", ["tgv_full", "cavity100", "shear", "duct"])
def test_parity_raw_model_fp64(P, name):
    w = CASES[name].scaled(model=synth.MODEL_RM)
    o, g = _init_both(P, w, seed=31)
    o.step(100)
    g.step(100)
    _cmp(o, g)


def test_parity_raw_model_generic_rates_fp32(P):
    w = synth.Workload("rm-generic", 17, 11, 9, r=0.5, s=1.0, nu=0.02, omega_xi=0.7, omega_1=1.3,
                       omega_high=1.1, force=(1e-5, 2e-5, -1e-5), init="random", seed=8, model=synth.MODEL_RM)
    o, g = _init_both(P, w, seed=8, noneq=1e-3)
    o.step(60)
    g.step(60)
    _cmp(o, g)
    w32 = w.scaled(precision=synth.PREC_FP32)
    o, g = _init_both(P, w32, seed=8)
    o.step(60)
    g.step(60)
    _cmp(o, g, prec=1)


# ------------------------------------------------------------------- CUDA graphs
@pytest.mark.parametrize("model", [0, 1])
def test_graphs_bitwise_equal_to_stream_launches(P, model):
    """step(n) replays captured 32-step graphs on small grids (graphs=0 auto);
    the result is bitwise the one of plain launches (graphs=1)."""
    w = CASES["tgv_full"].scaled(model=model)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 41)
    a = _gpu(P, w, graphs=1)
    b = _gpu(P, w, graphs=0)
    a.init_fields(rho, u)
    b.init_fields(rho, u)
    for n in (100, 7, 64):  # 3 graphs + 4 launches, 7 launches, 2 graphs
        a.step(n)
        b.step(n)
    assert a.info()["steps"] == b.info()["steps"] == 171
    assert np.array_equal(a.get_populations(), b.get_populations())
    b.set_force((1e-5, 0.0, 0.0))  # invalidates the captured graphs
    a.set_force((1e-5, 0.0, 0.0))
    a.step(40)
    b.step(40)
    assert np.array_equal(a.get_populations(), b.get_populations())


def test_parity_time_periodic_force(P):
    """Per-step force updates (F = F_m cos(omega t)) through
    lbm_cuboid_set_force on both sides, walls in y and z."""
    w = synth.CONFIGS["duct"].scaled(nx=4, ny=22, nz=11, force=(0.0, 0.0, 0.0))
    o, g = _init_both(P, w, seed=43)
    for n in range(1, 61):
        F = (1e-4 * np.cos(2 * np.pi * n / 40), 0.0, 2e-5 * np.sin(2 * np.pi * n / 40))
        o.set_force(F)
        g.set_force(F)
        o.step(1)
        g.step(1)
    _cmp(o, g)
    ro, uo = o.macroscopic()
    rg, ug = g.get_macroscopic()
    assert np.abs(ro - rg).max() < 1e-12 and np.abs(uo - ug).max() < 1e-12


# ------------------------------------------------- FULL_FD (density-gradient terms)
@pytest.mark.parametrize("model", [0, 1])
@pytest.mark.parametrize("name", ["tgv_full", "cavity100", "shear", "duct"])
def test_parity_full_fd(P, name, model):
    w = CASES[name].scaled(corrections=synth.CORR_FULL_FD, model=model)
    o, g = _init_both(P, w, seed=53)
    o.step(60)
    g.step(60)
    _cmp(o, g)


def test_parity_full_fd_generic_rates_fp32(P):
    w = synth.Workload("fd-generic", 15, 9, 8, r=0.75, s=1.3, nu=0.02, omega_xi=1.3, omega_1=1.2,
                       omega_high=0.9, force=(1e-5, 0.0, -2e-5), corrections=synth.CORR_FULL_FD,
                       init="random", seed=9)
    o, g = _init_both(P, w, seed=9, noneq=1e-3)
    o.step(40)
    g.step(40)
    _cmp(o, g)
    w32 = w.scaled(precision=synth.PREC_FP32)
    o, g = _init_both(P, w32, seed=9)
    o.step(40)
    g.step(40)
    _cmp(o, g, prec=1)


def test_full_fd_nccl_halo_and_graphs_bitwise(P):
    """FULL_FD through the ghost-plane path (density planes exchanged by NCCL,
    send to self) and through CUDA graphs equals the plain single-GPU launches."""
    w = CASES["weak_tgv"].scaled(corrections=synth.CORR_FULL_FD)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 57)
    a = _gpu(P, w, graphs=1)
    b = _gpu(P, w, halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id())
    c = _gpu(P, w, graphs=2)
    for g in (a, b, c):
        g.init_fields(rho, u)
        g.step(70)
    fa = a.get_populations()
    assert np.array_equal(fa, b.get_populations())
    assert np.array_equal(fa, c.get_populations())


def _patch_update(w, rho_g, u_g, x, y, z):
    """Oracle value after ONE step of node (x, y, z) of the full grid: a 3x3x3
    patch of the initial fields holding all the node's pull sources.  Along a
    periodic axis the patch wraps around the node; along an axis where the node
    touches a wall the patch starts at that wall and keeps its boundary type."""
    import oracle as O

    n = (w.nx, w.ny, w.nz)
    pos = (x, y, z)
    idx, centre, bc = [], [], list(w.bc)
    for d in range(3):
        lo_wall = w.bc[2 * d] != synth.BC_PERIODIC
        if lo_wall and pos[d] == 0:
            ids, c = [0, 1, 2], 0
        elif lo_wall and pos[d] == n[d] - 1:
            ids, c = [n[d] - 3, n[d] - 2, n[d] - 1], 2
        else:
            ids, c = [(pos[d] + k) % n[d] for k in (-1, 0, 1)], 1
            bc[2 * d] = bc[2 * d + 1] = synth.BC_PERIODIC
        idx.append(ids)
        centre.append(c)
    d = w.params()
    d.update(nx=3, ny=3, nz=3, bc=tuple(bc))
    o = O.Oracle(**d)
    sel = np.ix_(idx[2], idx[1], idx[0])
    o.init_fields(rho_g[sel], np.stack([u_g[k][sel] for k in range(3)]))
    o.step(1)
    return o.get_populations()[:, centre[2], centre[1], centre[0]]


def test_full_size_config4_shear_layer_sampled(P):
    """BASELINE config 4 at full size (512x256x512, r=0.5, s=1, free-slip y walls,
    tanh profile + seeded noise): one step on the GPU, sampled nodes including
    both free-slip walls against the oracle's patch update."""
    w = synth.CONFIGS["shear"]
    rho, u = synth.initial_fields(w)
    g = _gpu(P, w)
    g.init_fields(rho, u)
    g.step(1)
    rng = np.random.default_rng(2)
    for z in (0, 300, 511):
        fz = g.get_populations_planes(z, 1)[:, 0]
        ys = np.concatenate([[0, 0, w.ny - 1, w.ny - 1, 1, w.ny - 2], rng.integers(0, w.ny, 4)])
        xs = np.concatenate([[0, w.nx - 1, 0, w.nx - 1, 7, 9], rng.integers(0, w.nx, 4)])
        for x, y in zip(xs, ys):
            ref = _patch_update(w, rho, u, x, y, z)
            assert np.abs(fz[:, y, x] - ref).max() <= TOL64
    d = g.check()
    assert d["bad_nodes"] == 0


def test_full_size_config3_cavity_properties(P):
    """BASELINE config 3 at full size (256x256x128, s = 2, Re = 1000): properties
    that hold at any size -- total mass is conserved to round-off with all walls,
    and the z-mirror symmetry of the lid-driven box is kept (u_z odd, u_x, u_y
    even about the mid-plane) after 2000 steps."""
    w = synth.CONFIGS["cavity1000"]
    g = _gpu(P, w)
    rho, u = synth.rest_fields(w.nx, w.ny, w.nz)
    g.init_fields(rho, u)
    m0 = g.check()["mass"]
    g.step(2000)
    d = g.check()
    assert d["bad_nodes"] == 0 and abs(d["mass"] - m0) / m0 < 1e-11
    assert 0.3 * w.wall_u < d["max_speed"] < 1.5 * w.wall_u
    _, uu = g.get_macroscopic()
    mir = uu[:, ::-1]
    scale = w.wall_u
    assert np.abs(uu[0] - mir[0]).max() < 1e-9 * scale
    assert np.abs(uu[1] - mir[1]).max() < 1e-9 * scale
    assert np.abs(uu[2] + mir[2]).max() < 1e-9 * scale


# ----------------------------------------------------- AA in-place streaming
def _run_ab_aa(P, w, steps, seed=61, **kw):
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, seed)
    a = _gpu(P, w, **kw)
    b = _gpu(P, w, streaming=P.STREAM_AA, **kw)
    a.init_fields(rho, u)
    b.init_fields(rho, u)
    a.step(steps)
    b.step(steps)
    return a, b


@pytest.mark.parametrize("steps", [1, 2, 37, 64])
@pytest.mark.parametrize("name", ["weak_tgv", "duct", "shear"])
def test_aa_equals_ab_bitwise(P, name, steps):
    """AA in-place streaming (one buffer) reproduces the two-buffer scheme bit for
    bit (same per-node arithmetic, same values gathered) after odd and even step
    counts, with periodic, bounce-back and free-slip faces."""
    w = CASES[name]
    a, b = _run_ab_aa(P, w, steps)
    fa, fb = a.get_populations(), b.get_populations()
    assert np.array_equal(fa, fb)
    ra, ua = a.get_macroscopic()
    rb, ub = b.get_macroscopic()
    assert np.array_equal(ra, rb) and np.array_equal(ua, ub)
    assert a.check()["mass"] == pytest.approx(b.check()["mass"], rel=1e-15)


@pytest.mark.parametrize("model", [0, 1])
@pytest.mark.parametrize("steps", [1, 30, 31])
def test_aa_lid_cavity_and_models(P, model, steps):
    """Moving lid (the push uses rho_f = rho of the node, equal to sum f~ up to
    rounding): AA vs AB within 1e-14, and AA vs the oracle within the parity bar."""
    w = CASES["cavity100"].scaled(model=model)
    a, b = _run_ab_aa(P, w, steps)
    assert np.abs(a.get_populations() - b.get_populations()).max() < 1e-14
    o, _ = _init_both(P, w, seed=61)
    o.step(steps)
    _cmp(o, b)


def test_aa_fp32_generic_rates_graphs_and_set_populations(P):
    w = synth.Workload("aa-generic", 13, 11, 9, r=0.75, s=1.3, nu=0.02, omega_xi=1.3, omega_1=1.2,
                       omega_high=0.9, force=(1e-5, 0.0, -2e-5), bc=(0, 0, 1, 2, 0, 0), wall_u=0.03,
                       init="random", seed=4)
    for prec in (0, 1):
        ww = w.scaled(precision=prec)
        a, b = _run_ab_aa(P, ww, 45, seed=4)
        d = np.abs(a.get_populations() - b.get_populations()).max()
        assert d < (1e-14 if prec == 0 else 1e-6), d
    # graphs (32-step replays) and a set_populations restart in layout R
    ww = w.scaled(nx=21, ny=19, nz=11)
    a, b = _run_ab_aa(P, ww, 70, seed=5, graphs=2)
    c = _gpu(P, ww, streaming=P.STREAM_AA, graphs=1)
    rho, u = synth.random_fields(ww.nx, ww.ny, ww.nz, 5)
    c.init_fields(rho, u)
    c.step(70)
    assert np.array_equal(b.get_populations(), c.get_populations())
    f = b.get_populations()
    b.set_populations(f)
    a.set_populations(f)
    a.step(9)
    b.step(9)
    assert np.abs(a.get_populations() - b.get_populations()).max() < 1e-14


def test_aa_rejects_multi_gpu_and_fd(P):
    w = CASES["weak_tgv"]
    with pytest.raises(P.LbmError):
        _gpu(P, w, streaming=P.STREAM_AA, halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id())
    with pytest.raises(P.LbmError):
        _gpu(P, w.scaled(corrections=synth.CORR_FULL_FD), streaming=P.STREAM_AA)


PERSIST_CASES = {
    "tgv_paper": (synth.CONFIGS["tgv"], {}),
    "cavity_generic": (synth.CONFIGS["cavity100"].scaled(nx=21, ny=19, nz=11), {"omega_1": 1.2, "omega_high": 1.1}),
    "shear_raw_fp32": (synth.CONFIGS["shear"].scaled(nx=16, ny=29, nz=12), {"model": 1, "precision": 1}),
    "duct_fd": (synth.CONFIGS["duct"].scaled(nx=5, ny=37, nz=19), {"corrections": 3}),
    "tgv_fd_fp32": (synth.CONFIGS["tgv"].scaled(nx=24, ny=20, nz=10), {"corrections": 3, "precision": 1}),
}


@pytest.mark.parametrize("case", list(PERSIST_CASES))
def test_persistent_kernel_bitwise_equal_to_launches(P, case):
    """graphs = 3 (one cooperative launch for many steps, grid barrier between
    steps) gives bitwise the per-step launches' result; odd step counts."""
    w, kw = PERSIST_CASES[case]
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 41)
    a = _gpu(P, w, graphs=1, **kw)
    b = _gpu(P, w, graphs=3, **kw)
    for g in (a, b):
        g.init_fields(rho, u)
        g.step(37)
        g.step(0)
        g.step(2)
    assert np.array_equal(a.get_populations(), b.get_populations())
    assert b.info()["steps"] == 39 and b.info()["collide_stream_launches"] == 2
    a.close()
    b.close()


def test_persistent_kernel_long_run_chunks_and_oracle(P):
    """More steps than one persistent launch holds (1024): chunked launches,
    buffer parity across chunks, against the oracle on config 1."""
    w = synth.CONFIGS["tgv"].scaled(nx=12, ny=10, nz=6)
    o, g = _init_both(P, w, seed=8, noneq=1e-3, graphs=3)
    g.timing(True)
    g.step(1031)
    t = g.timing_read()
    assert t["launches"] == 2 and t["node_updates"] == 1031 * w.nodes
    o.step(1031)
    _cmp(o, g)
    g.close()


FD_FUSED_CASES = {
    # ragged tiles (nx % 32, ny % 8 != 0) and z-chunks (nz % 16 != 0)
    "tgv_ragged": (synth.CONFIGS["tgv"].scaled(nx=45, ny=13, nz=37), {}),
    "cavity_lid_walls": (synth.CONFIGS["cavity100"].scaled(nx=33, ny=17, nz=20), {}),
    "shear_slip_raw_fp32": (synth.CONFIGS["shear"].scaled(nx=40, ny=9, nz=18), {"model": 1, "precision": 1}),
    "duct_generic": (synth.CONFIGS["duct"].scaled(nx=7, ny=26, nz=17), {"omega_1": 1.3, "omega_high": 0.8}),
    "thin": (synth.CONFIGS["tgv"].scaled(nx=3, ny=2, nz=2), {}),
}


@pytest.mark.parametrize("case", list(FD_FUSED_CASES))
def test_full_fd_fused_kernel_equals_two_pass(P, case, monkeypatch):
    """The fused FULL_FD kernel (2.5D tiles, shared-memory density ring) equals
    the two-pass path (density pass + collide): the same densities and the same
    per-node arithmetic, inlined into two different kernels, where ptxas may
    fuse a multiply and an add differently (seen on the generic-rate duct after
    the singular-system predicate was added), so to rounding: max|df| <= 1e-14
    (fp64), relative <= 1e-6 (fp32 storage) after 23 steps.  The fused kernel
    through the NCCL ghost-plane path (boundary-plane density exchanged, planes
    next to the ghost faces read from the density field) equals the
    single-launch fused kernel bit for bit."""
    w, kw = FD_FUSED_CASES[case]
    w = w.scaled(corrections=synth.CORR_FULL_FD)
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 61)
    monkeypatch.setenv("LBM_FD_FUSED", "0")
    a = _gpu(P, w, graphs=1, **kw)
    monkeypatch.setenv("LBM_FD_FUSED", "1")
    b = _gpu(P, w, graphs=1, **kw)
    monkeypatch.delenv("LBM_FD_FUSED")
    hs = [a, b, _gpu(P, w, graphs=1, **kw)]  # and the default for this precision
    if w.bc[4] == synth.BC_PERIODIC:
        monkeypatch.setenv("LBM_FD_FUSED", "1")
        hs.append(_gpu(P, w, halo=P.HALO_NCCL, nccl_uid=P.nccl_unique_id(), **kw))
        monkeypatch.delenv("LBM_FD_FUSED")
    for g in hs:
        g.init_fields(rho, u)
        g.step(23)
    fa, fb = a.get_populations(), b.get_populations()
    for g in hs[1:]:
        fg = g.get_populations()
        if kw.get("precision", 0) == 0:
            assert np.abs(fg - fa).max() <= 1e-14
        else:
            assert (np.abs(fg - fa) / np.abs(fa)).max() <= 1e-6
    for g in hs[3:]:  # NCCL ghost path, fused kernel
        assert np.array_equal(fb, g.get_populations())
    for g in hs:
        g.close()


def test_max_plane_size_int32_offsets(P):
    """The largest plane the ABI accepts (27 nx ny < 2^31: int32 offsets within a
    plane): 8191 x 9710 nodes per plane, nz = 2 periodic, fp32 storage (69 GB in
    two buffers).  One step from rough random fields; sampled nodes including all
    four plane corners and the last node against the oracle's patch update.  The
    populations are read straight from the device buffer (layout of DESIGN.md
    section 6: [(z_local + 1) * 27 + q][y][x], q = (ex+1) + 3(ey+1) + 9(ez+1))."""
    import oracle as O
    import torch

    nx, ny, nz = 8191, 9710, 2
    assert 27 * nx * ny < 2 ** 31
    w = synth.CONFIGS["tgv"].scaled(nx=nx, ny=ny, nz=nz, precision=synth.PREC_FP32)
    free, _ = torch.cuda.mem_get_info()
    if free < 80e9:
        pytest.skip("needs ~75 GB of free device memory")
    rho, u = synth.random_fields(nx, ny, nz, 4242)
    g = _gpu(P, w)
    g.init_fields(rho, u)
    g.step(1)
    g.sync()
    buf = g._bufs[g.info()["steps"] % 2].view(torch.float32)  # the state after one step
    e = O.velocities(1.0, 1.0).round().astype(int)           # paper order, unit components
    qint = (e[:, 0] + 1) + 3 * (e[:, 1] + 1) + 9 * (e[:, 2] + 1)
    nxy = nx * ny
    rng = np.random.default_rng(5)
    pts = [(0, 0), (nx - 1, 0), (0, ny - 1), (nx - 1, ny - 1), (nx // 2, ny // 2)]
    pts += [(int(a), int(b)) for a, b in zip(rng.integers(0, nx, 4), rng.integers(0, ny, 4))]
    for z in (0, nz - 1):
        for x, y in pts:
            off = torch.tensor([((z + 1) * 27 + int(q)) * nxy + y * nx + x for q in qint], device=buf.device)
            fg = buf[off].double().cpu().numpy()
            ref = _patch_update(w, rho, u, x, y, z)
            assert (np.abs(fg - ref) / np.abs(ref)).max() <= TOL32, (x, y, z)
    g.close()


@pytest.mark.parametrize("kw", [{}, {"streaming": 1}, {"precision": 1}, {"corrections": 3}])
def test_checkpoint_resume_is_exact(P, kw):
    """Checkpoint / resume: 24 steps in one run equal n steps,
    get_populations, a NEW lattice set_populations, 24 - n more steps -- bit for
    bit (the state is the stored populations; the update is deterministic).
    AA checkpoints after an even step, where the buffer holds the canonical
    post-collision state; after an odd step reading it back undoes the Eq. 69
    lid term with rho_f = sum f~ of the read values, exact only to rounding."""
    w = CASES["cavity100"]
    n = 12 if kw.get("streaming") else 11
    rho, u = synth.random_fields(w.nx, w.ny, w.nz, 77)
    a = _gpu(P, w, **kw)
    a.init_fields(rho, u)
    a.step(24)
    ref = a.get_populations()
    a.close()
    b = _gpu(P, w, **kw)
    b.init_fields(rho, u)
    b.step(n)
    ck = b.get_populations()
    b.close()
    c = _gpu(P, w, **kw)
    c.set_populations(ck)
    c.step(24 - n)
    assert np.array_equal(c.get_populations(), ref)
    c.close()
