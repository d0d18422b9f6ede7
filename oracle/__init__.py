"""ctypes wrapper around the plain-C CPU oracle (oracle/cm_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may use this.  The product path
(paper_2107_14774_b200/) never imports it.

Array layouts: populations [27][nz][ny][nx] in the paper's direction order
(Eqs. 1a-1c); scalar fields [nz][ny][nx]; vector fields
[3][nz][ny][nx].
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cm_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no contraction, no SIMD intrinsics)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, SRC, "-o", tmp, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class _Params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("r", ctypes.c_double), ("s", ctypes.c_double), ("cs2", ctypes.c_double),
                ("omega_nu", ctypes.c_double), ("omega_xi", ctypes.c_double),
                ("omega_1", ctypes.c_double), ("omega_high", ctypes.c_double),
                ("force", ctypes.c_double * 3), ("bc", ctypes.c_int32 * 6),
                ("wall_u", ctypes.c_double), ("corrections", ctypes.c_int32), ("model", ctypes.c_int32)]


_lib = None
_D = ctypes.POINTER(ctypes.c_double)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.oracle_create.restype = ctypes.c_void_p
        L.oracle_create.argtypes = [ctypes.POINTER(_Params)]
        L.oracle_destroy.argtypes = [ctypes.c_void_p]
        L.oracle_set_force.argtypes = [ctypes.c_void_p, _D]
        L.oracle_ctx_Qinv.restype = _D
        L.oracle_ctx_Qinv.argtypes = [ctypes.c_void_p]
        L.oracle_velocities.argtypes = [ctypes.c_double, ctypes.c_double, _D]
        L.oracle_opposite.argtypes = [ctypes.POINTER(ctypes.c_int)]
        L.oracle_Q.argtypes = [ctypes.c_double, ctypes.c_double, _D]
        L.oracle_invert27.argtypes = [_D, _D]
        L.oracle_invert27.restype = ctypes.c_int
        L.oracle_hydro.argtypes = [_D, _D, _D, _D, _D]
        L.oracle_central_moments.argtypes = [_D, _D, _D, _D]
        L.oracle_frame.argtypes = [_D, _D, _D]
        L.oracle_raw_equilibria.argtypes = [ctypes.c_double, _D, ctypes.c_double, _D]
        L.oracle_feq.argtypes = [ctypes.c_void_p, ctypes.c_double, _D, _D]
        L.oracle_collide.argtypes = [ctypes.c_void_p, _D, _D]
        L.oracle_collide_raw.argtypes = [ctypes.c_void_p, _D, _D]
        L.oracle_collide_g.argtypes = [ctypes.c_void_p, _D, _D, _D]
        L.oracle_collide_raw_g.argtypes = [ctypes.c_void_p, _D, _D, _D]
        L.oracle_density_gradient.argtypes = [ctypes.c_void_p, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
        L.oracle_raw_source.argtypes = [_D, _D, _D]
        L.oracle_lid_term.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_double]
        L.oracle_lid_term.restype = ctypes.c_double
        L.oracle_step.argtypes = [ctypes.c_void_p, _D, _D]
        L.oracle_run.argtypes = [ctypes.c_void_p, _D, _D, ctypes.c_int64]
        L.oracle_init.argtypes = [ctypes.c_void_p, _D, _D, _D]
        L.oracle_macroscopic.argtypes = [ctypes.c_void_p, _D, _D, _D]
        L.oracle_singular_count.restype = ctypes.c_int64
        L.oracle_singular_count.argtypes = []
        L.oracle_singular_reset.argtypes = []
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def _arr(x, n=None):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if n is not None:
        assert a.size == n, (a.shape, n)
    return a


# ---------------------------------------------------------------- pure functions

def velocities(r, s):
    e = np.zeros((27, 3))
    lib().oracle_velocities(r, s, _p(e))
    return e


def opposite():
    o = (ctypes.c_int * 27)()
    lib().oracle_opposite(o)
    return np.array(list(o))


def Q(r, s):
    m = np.zeros((27, 27))
    lib().oracle_Q(r, s, _p(m))
    return m


def invert27(a):
    a = _arr(a, 729)
    out = np.zeros((27, 27))
    if lib().oracle_invert27(_p(a), _p(out)) != 0:
        raise np.linalg.LinAlgError("singular")
    return out


def hydro(e, f, F):
    rho = np.zeros(1)
    u = np.zeros(3)
    lib().oracle_hydro(_p(_arr(e, 81)), _p(_arr(f, 27)), _p(_arr(F, 3)), _p(rho), _p(u))
    return rho[0], u


def central_moments(e, f, u):
    k = np.zeros(27)
    lib().oracle_central_moments(_p(_arr(e, 81)), _p(_arr(f, 27)), _p(_arr(u, 3)), _p(k))
    return k


def frame(m, a):
    """Binomial transform with shift a: a = -u maps raw->central, a = +u central->raw."""
    out = np.zeros(27)
    lib().oracle_frame(_p(_arr(m, 27)), _p(_arr(a, 3)), _p(out))
    return out


def raw_source(u, F):
    phi = np.zeros(27)
    lib().oracle_raw_source(_p(_arr(u, 3)), _p(_arr(F, 3)), _p(phi))
    return phi


def singular_count(reset=False):
    """Nodes whose strain-rate system was singular (reading R17)
    since the last reset."""
    n = int(lib().oracle_singular_count())
    if reset:
        lib().oracle_singular_reset()
    return n


def raw_equilibria(rho, u, cs2):
    m = np.zeros(27)
    lib().oracle_raw_equilibria(float(rho), _p(_arr(u, 3)), float(cs2), _p(m))
    return m


# ---------------------------------------------------------------- lattice object

class Oracle:
    """One periodic/walled grid of the 3DCCM-LBM, run on the CPU, fp64."""

    def __init__(self, nx, ny, nz, r, s, cs2, omega_nu, omega_xi=1.0, omega_1=1.0,
                 omega_high=1.0, force=(0.0, 0.0, 0.0), bc=(0,) * 6, wall_u=0.0,
                 corrections=0, precision=0, model=0, **ignored):
        del precision, ignored  # the oracle is always fp64; GPU-only knobs (halo, graphs, ...) ignored
        p = _Params()
        p.nx, p.ny, p.nz = nx, ny, nz
        p.r, p.s, p.cs2 = r, s, cs2
        p.omega_nu, p.omega_xi, p.omega_1, p.omega_high = omega_nu, omega_xi, omega_1, omega_high
        for i in range(3):
            p.force[i] = force[i]
        for i in range(6):
            p.bc[i] = bc[i]
        p.wall_u = wall_u
        p.corrections = corrections
        p.model = model
        self.model = model
        self._params = p
        self.shape = (nz, ny, nx)
        self.nx, self.ny, self.nz = nx, ny, nz
        self.r, self.s, self.cs2 = r, s, cs2
        self.force = np.array(force, dtype=np.float64)
        self._ctx = lib().oracle_create(ctypes.byref(p))
        if not self._ctx:
            raise ValueError("oracle_create failed (singular Q)")
        self.f = np.zeros((27, nz, ny, nx))
        self._tmp = np.zeros_like(self.f)

    @classmethod
    def from_params(cls, d: dict):
        return cls(**d)

    def __del__(self):
        if getattr(self, "_ctx", None) and _lib is not None:
            _lib.oracle_destroy(self._ctx)
            self._ctx = None

    @property
    def Qinv(self):
        ptr = lib().oracle_ctx_Qinv(self._ctx)
        return np.ctypeslib.as_array(ptr, shape=(27 * 27,)).reshape(27, 27).copy()

    def feq(self, rho, u):
        out = np.zeros(27)
        lib().oracle_feq(self._ctx, float(rho), _p(_arr(u, 3)), _p(out))
        return out

    def collide(self, f, grad_rho=None):
        out = np.zeros(27)
        if grad_rho is None:
            fn = lib().oracle_collide_raw if self.model == 1 else lib().oracle_collide
            fn(self._ctx, _p(_arr(f, 27)), _p(out))
        else:
            fn = lib().oracle_collide_raw_g if self.model == 1 else lib().oracle_collide_g
            fn(self._ctx, _p(_arr(f, 27)), _p(_arr(grad_rho, 3)), _p(out))
        return out

    def density_gradient(self, rho, x, y, z):
        g = np.zeros(3)
        lib().oracle_density_gradient(self._ctx, _p(_arr(rho, self.f[0].size)), int(x), int(y), int(z), _p(g))
        return g

    def set_force(self, F):
        self.force = _arr(F, 3).copy()
        lib().oracle_set_force(self._ctx, _p(self.force))

    def lid_term(self, q, rho_f):
        return lib().oracle_lid_term(self._ctx, int(q), float(rho_f))

    def init_fields(self, rho, u):
        rho = _arr(rho, self.f[0].size)
        u = _arr(u, 3 * self.f[0].size)
        lib().oracle_init(self._ctx, _p(rho), _p(u), _p(self.f))

    def set_populations(self, f):
        self.f[...] = np.asarray(f, dtype=np.float64).reshape(self.f.shape)

    def get_populations(self):
        return self.f.copy()

    def step(self, n: int = 1):
        lib().oracle_run(self._ctx, _p(self.f), _p(self._tmp), int(n))

    def macroscopic(self):
        rho = np.zeros(self.shape)
        u = np.zeros((3,) + self.shape)
        lib().oracle_macroscopic(self._ctx, _p(self.f), _p(rho), _p(u))
        return rho, u
