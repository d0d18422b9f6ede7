"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no moment transforms, no
collision, no equilibria).  It only produces:

  * the five workload presets of BASELINE.json (grid, aspect ratios, physical
    parameters, boundary types) and the plain parameter mapping the paper states
    between viscosities and relaxation rates (Eq. 53), and
  * seeded macroscopic initial fields (rho, u) and seeded noise arrays.

Both sides receive identical numbers from here; each then computes its own
populations.  Layouts: scalar fields are C-ordered [z][y][x]; vector fields are
[3][z][y][x] (component-major), x fastest.
"""
from __future__ import annotations

import dataclasses

import numpy as np

# boundary types (same integer codes as include/lbm_cuboid.h and the oracle)
BC_PERIODIC, BC_BOUNCE_BACK, BC_MOVING_WALL, BC_FREE_SLIP = 0, 1, 2, 3
# correction modes (readings R1)
CORR_FULL_LOCAL, CORR_LOW_MACH, CORR_OFF, CORR_FULL_FD, CORR_FULL_FD_LAG = 0, 1, 2, 3, 4
# storage precision
PREC_FP64, PREC_FP32 = 0, 1
# collision model
MODEL_CM, MODEL_RM = 0, 1


def auto_cs2(r: float, s: float) -> float:
    """Speed of sound rule.  PAPER.md L545 gives cs2 = min(r^2, s^2)/3; DESIGN.md
    reading R3 uses min(1, r^2, s^2)/3, identical at every (r, s) of the configs."""
    return min(1.0, r * r, s * s) / 3.0


def omega_from_nu(nu: float, cs2: float) -> float:
    """Eq. 53: nu = cs2 (1/omega_nu - 1/2)."""
    return 1.0 / (nu / cs2 + 0.5)


def omega_from_xi(xi: float, cs2: float) -> float:
    """Eq. 53: xi = (2 cs2 / 3)(1/omega_xi - 1/2)."""
    return 1.0 / (xi / (2.0 * cs2 / 3.0) + 0.5)


@dataclasses.dataclass
class Workload:
    name: str
    nx: int
    ny: int
    nz: int
    r: float
    s: float
    nu: float
    cs2: float | None = None
    omega_xi: float = 1.0      # all rates other than shear set to 1.0
    omega_1: float = 1.0
    omega_high: float = 1.0
    force: tuple = (0.0, 0.0, 0.0)
    bc: tuple = (0, 0, 0, 0, 0, 0)   # faces -x,+x,-y,+y,-z,+z
    wall_u: float = 0.0
    corrections: int = CORR_FULL_LOCAL
    precision: int = PREC_FP64
    steps: int = 100
    init: str = "rest"          # 'rest' | 'tgv' | 'shear_layer' | 'random'
    u0: float = 0.0
    seed: int = 2107
    model: int = 0              # 0: 3DCCM (central moments), 1: 3DCRM (raw moments)

    @property
    def cs2_value(self) -> float:
        return auto_cs2(self.r, self.s) if self.cs2 is None else self.cs2

    @property
    def omega_nu(self) -> float:
        return omega_from_nu(self.nu, self.cs2_value)

    @property
    def nodes(self) -> int:
        return self.nx * self.ny * self.nz

    def scaled(self, nx=None, ny=None, nz=None, **kw) -> "Workload":
        """Same physics at another grid size."""
        d = dataclasses.asdict(self)
        d.update({k: v for k, v in (("nx", nx), ("ny", ny), ("nz", nz)) if v is not None})
        d.update(kw)
        return Workload(**d)

    def params(self) -> dict:
        """The problem statement as both sides consume it (PAPER.md L56, L438-440,
        L545, L746-751, L1235-1239)."""
        return dict(nx=self.nx, ny=self.ny, nz=self.nz, r=self.r, s=self.s,
                    cs2=self.cs2_value, omega_nu=self.omega_nu, omega_xi=self.omega_xi,
                    omega_1=self.omega_1, omega_high=self.omega_high,
                    force=tuple(self.force), bc=tuple(self.bc), wall_u=self.wall_u,
                    corrections=self.corrections, precision=self.precision, model=self.model)


P = BC_PERIODIC
BB = BC_BOUNCE_BACK
MW = BC_MOVING_WALL
FS = BC_FREE_SLIP

# BASELINE.json configs[0..4]; unspecified details are DESIGN.md readings R9-R15.
CONFIGS = {
    "tgv": Workload("config1-tgv-32x32x16", 32, 32, 16, r=1.0, s=2.0, nu=0.01,
                    init="tgv", u0=0.02, steps=200),
    "duct": Workload("config2-duct-8x128x64", 8, 128, 64, r=1.0, s=2.0, nu=0.05,
                     force=(1e-6, 0.0, 0.0), bc=(P, P, BB, BB, BB, BB), init="rest",
                     steps=300000),
    "cavity100": Workload("config3-cavity-Re100-256x256x128", 256, 256, 128, r=1.0, s=2.0,
                          nu=0.05 * 256 / 100.0, bc=(BB, BB, BB, MW, BB, BB), wall_u=0.05,
                          init="rest", steps=20000),
    "cavity1000": Workload("config3-cavity-Re1000-256x256x128", 256, 256, 128, r=1.0, s=2.0,
                           nu=0.05 * 256 / 1000.0, bc=(BB, BB, BB, MW, BB, BB), wall_u=0.05,
                           init="rest", steps=20000),
    "shear": Workload("config4-shear-layer-512x256x512", 512, 256, 512, r=0.5, s=1.0, nu=0.01,
                      bc=(P, P, FS, FS, P, P), init="shear_layer", u0=0.04, steps=1000),
    "weak": Workload("config5-weak-tgv-512^3-per-gpu", 512, 512, 512, r=1.0, s=2.0, nu=0.01,
                     init="tgv", u0=0.02, steps=500),
    "strong": Workload("config5-strong-tgv-1024x1024x512", 1024, 1024, 512, r=1.0, s=2.0,
                       nu=0.01, init="tgv", u0=0.02, steps=500),
}


def slab_range(nz: int, rank: int, world: int) -> tuple[int, int]:
    """z-slab decomposition: rank owns planes [z0, z1).  nz % world must be 0."""
    if world < 1 or nz % world:
        raise ValueError(f"nz={nz} not divisible by world={world}")
    n = nz // world
    return rank * n, (rank + 1) * n


def tgv_fields(nx, ny, nz, cs2, u0, z0=0, z1=None, nz_global=None, xp=np, device=None):
    """Decaying Taylor-Green vortex initial fields (reading R9):
    u = u0 (sin x cos y cos z, -cos x sin y cos z, 0) and
    rho = 1 + (u0^2/16)(cos 2x + cos 2y)(cos 2z + 2)/cs2, at node phases
    x = 2 pi i/nx, y = 2 pi j/ny, z = 2 pi k/nz_global.  Returns the slab
    [z0, z1) of the global field.  xp = numpy (host arrays) or torch (arrays
    on `device`, fp64, same values) for device-resident bench inputs."""
    nz_global = nz if nz_global is None else nz_global
    z1 = nz_global if z1 is None else z1
    kw = {} if xp is np else {"dtype": xp.float64, "device": device}
    x = 2 * np.pi * xp.arange(nx, **kw) / nx
    y = 2 * np.pi * xp.arange(ny, **kw) / ny
    z = 2 * np.pi * xp.arange(z0, z1, **kw) / nz_global
    X, Y, Z = x[None, None, :], y[None, :, None], z[:, None, None]
    shape = (z1 - z0, ny, nx)
    u = xp.zeros((3,) + shape, **kw)
    u[0] = u0 * xp.sin(X) * xp.cos(Y) * xp.cos(Z)
    u[1] = -u0 * xp.cos(X) * xp.sin(Y) * xp.cos(Z)
    rho = 1.0 + (u0 * u0 / 16.0) * (xp.cos(2 * X) + xp.cos(2 * Y)) * (xp.cos(2 * Z) + 2.0) / cs2
    rho = rho + xp.zeros(shape, **kw)
    if xp is np:
        return np.ascontiguousarray(rho), np.ascontiguousarray(u)
    return rho.contiguous(), u.contiguous()


def rest_fields(nx, ny, nz):
    return np.ones((nz, ny, nx)), np.zeros((3, nz, ny, nx))


def shear_layer_fields(nx, ny, nz, u0, thickness=16.0, amp=1e-3, seed=2107, z0=0, z1=None):
    """Config 4 (reading R10): u_x = u0 tanh((j - ny/2 + 1/2)/thickness),
    every velocity component += amp * xi, xi ~ U(-1,1) from PCG64(seed) drawn in C
    order (z, y, x, component) over the GLOBAL grid; rho = 1."""
    z1 = nz if z1 is None else z1
    rng = np.random.Generator(np.random.PCG64(seed))
    xi = rng.uniform(-1.0, 1.0, size=(nz, ny, nx, 3))[z0:z1]
    j = np.arange(ny)
    prof = u0 * np.tanh((j - ny / 2 + 0.5) / thickness)
    u = np.zeros((3, z1 - z0, ny, nx))
    u[0] += prof[None, :, None]
    u += amp * np.moveaxis(xi, -1, 0)
    return np.ones((z1 - z0, ny, nx)), np.ascontiguousarray(u)


def random_fields(nx, ny, nz, seed, rho_amp=0.01, u_amp=0.02):
    """Seeded, rough (per-node independent) macroscopic fields for parity tests:
    rho = 1 + rho_amp * xi, u = u_amp * xi, xi ~ U(-1,1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rho = 1.0 + rho_amp * rng.uniform(-1.0, 1.0, size=(nz, ny, nx))
    u = u_amp * rng.uniform(-1.0, 1.0, size=(3, nz, ny, nx))
    return rho, u


def noise(shape, seed):
    """xi ~ U(-1, 1) of the given shape from PCG64(seed)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-1.0, 1.0, size=shape)


def initial_fields(w: Workload, z0=0, z1=None, nz_global=None):
    """Initial (rho, u) for a workload (slab [z0, z1) of the global grid)."""
    nzg = w.nz if nz_global is None else nz_global
    z1 = nzg if z1 is None else z1
    if w.init == "tgv":
        return tgv_fields(w.nx, w.ny, w.nz, w.cs2_value, w.u0, z0, z1, nzg)
    if w.init == "shear_layer":
        return shear_layer_fields(w.nx, w.ny, nzg, w.u0, seed=w.seed, z0=z0, z1=z1)
    if w.init == "random":
        rho, u = random_fields(w.nx, w.ny, nzg, w.seed)
        return np.ascontiguousarray(rho[z0:z1]), np.ascontiguousarray(u[:, z0:z1])
    return rest_fields(w.nx, w.ny, z1 - z0)


def reynolds(w: Workload, length: float, speed: float) -> float:
    return speed * length / w.nu


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("np", "dataclasses", "annotations")]
