"""Thin ctypes binding of the C ABI in include/lbm_cuboid.h.

Argument marshalling only: every step of the hot path runs in the CUDA kernels
of liblbm_cuboid.so.  PyTorch provides device memory (the two population
buffers are torch tensors), the compute stream (torch's current stream) and,
for several GPUs, the process group used to broadcast the NCCL unique id.

There is no CPU fallback: if the shared library is missing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# LBM_CUBOID_LIB selects an alternative build (kernel-variant sweeps); default in-tree
LIB_PATH = os.environ.get("LBM_CUBOID_LIB", os.path.join(_PKG, "liblbm_cuboid.so"))

LBM_OK, LBM_EINVAL, LBM_ENOMEM, LBM_ECUDA, LBM_ENCCL, LBM_EUNSTABLE, LBM_ESINGULAR, LBM_ENOTSUP = (
    0, -1, -2, -3, -4, -5, -6, -7)
BC_PERIODIC, BC_BOUNCE_BACK, BC_MOVING_WALL, BC_FREE_SLIP = 0, 1, 2, 3
CORR_FULL_LOCAL, CORR_LOW_MACH, CORR_OFF, CORR_FULL_FD, CORR_FULL_FD_LAG = 0, 1, 2, 3, 4
FP64, FP32_STORAGE = 0, 1
HALO_AUTO, HALO_NCCL, HALO_P2P = 0, 1, 2
P2P_BLOB_BYTES = 512
MODEL_CM, MODEL_RM = 0, 1
STREAM_AB, STREAM_AA = 0, 1

# every symbol include/lbm_cuboid.h declares
EXPORTS = ["lbm_cuboid_default_params", "lbm_cuboid_buffer_bytes", "lbm_cuboid_halo_plan",
           "lbm_cuboid_nccl_unique_id", "lbm_cuboid_p2p_export", "lbm_cuboid_p2p_connect",
           "lbm_cuboid_create", "lbm_cuboid_init_fields", "lbm_cuboid_init_fields_device",
           "lbm_cuboid_step", "lbm_cuboid_sync", "lbm_cuboid_get_macroscopic",
           "lbm_cuboid_get_macroscopic_device", "lbm_cuboid_get_populations",
           "lbm_cuboid_get_populations_planes", "lbm_cuboid_set_populations", "lbm_cuboid_check", "lbm_cuboid_set_force",
           "lbm_cuboid_info", "lbm_cuboid_stream", "lbm_cuboid_comm_ranks", "lbm_cuboid_kernel_name", "lbm_cuboid_timing", "lbm_cuboid_timing_read",
           "lbm_cuboid_trace", "lbm_cuboid_trace_read",
           "lbm_cuboid_destroy", "lbm_cuboid_last_error"]


class LbmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("r", ctypes.c_double), ("s", ctypes.c_double), ("cs2", ctypes.c_double),
                ("omega_nu", ctypes.c_double), ("omega_xi", ctypes.c_double),
                ("omega_1", ctypes.c_double), ("omega_high", ctypes.c_double),
                ("force", ctypes.c_double * 3), ("bc", ctypes.c_int32 * 6),
                ("wall_u", ctypes.c_double), ("corrections", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("device", ctypes.c_int32), ("halo", ctypes.c_int32), ("graphs", ctypes.c_int32),
                ("model", ctypes.c_int32), ("streaming", ctypes.c_int32),
                ("nccl_uid", ctypes.c_void_p), ("stream", ctypes.c_void_p),
                ("buf_a", ctypes.c_void_p), ("buf_b", ctypes.c_void_p), ("check_every", ctypes.c_int32)]


_lib = None
_D = ctypes.POINTER(ctypes.c_double)
_VP = ctypes.c_void_p


def load():
    """Load liblbm_cuboid.so (build it with paper_2107_14774_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2107_14774_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.lbm_cuboid_default_params.argtypes = [ctypes.POINTER(Params)]
    L.lbm_cuboid_default_params.restype = None
    L.lbm_cuboid_buffer_bytes.argtypes = [ctypes.POINTER(Params), ctypes.POINTER(ctypes.c_int64)]
    L.lbm_cuboid_halo_plan.argtypes = [ctypes.POINTER(Params), ctypes.POINTER(ctypes.c_int64)]
    L.lbm_cuboid_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.lbm_cuboid_create.argtypes = [ctypes.POINTER(Params), ctypes.POINTER(_VP)]
    L.lbm_cuboid_p2p_export.argtypes = [_VP, ctypes.c_char_p]
    L.lbm_cuboid_p2p_connect.argtypes = [_VP, ctypes.c_char_p, ctypes.c_char_p]
    for n in ("lbm_cuboid_init_fields", "lbm_cuboid_init_fields_device", "lbm_cuboid_get_macroscopic",
              "lbm_cuboid_get_macroscopic_device"):
        getattr(L, n).argtypes = [_VP, _VP, _VP]
    L.lbm_cuboid_step.argtypes = [_VP, ctypes.c_int64]
    L.lbm_cuboid_sync.argtypes = [_VP]
    L.lbm_cuboid_get_populations.argtypes = [_VP, _VP]
    L.lbm_cuboid_get_populations_planes.argtypes = [_VP, ctypes.c_int32, ctypes.c_int32, _VP]
    L.lbm_cuboid_set_populations.argtypes = [_VP, _VP]
    L.lbm_cuboid_check.argtypes = [_VP, _D]
    L.lbm_cuboid_set_force.argtypes = [_VP, _D]
    L.lbm_cuboid_info.argtypes = [_VP, ctypes.POINTER(ctypes.c_int64)]
    L.lbm_cuboid_stream.argtypes = [_VP]
    L.lbm_cuboid_stream.restype = _VP
    L.lbm_cuboid_comm_ranks.argtypes = [_VP, ctypes.POINTER(ctypes.c_int32)]
    L.lbm_cuboid_comm_ranks.restype = ctypes.c_int
    L.lbm_cuboid_kernel_name.argtypes = [_VP]
    L.lbm_cuboid_kernel_name.restype = ctypes.c_char_p
    L.lbm_cuboid_trace.argtypes = [_VP, ctypes.c_int]
    L.lbm_cuboid_trace.restype = ctypes.c_int
    L.lbm_cuboid_trace_read.argtypes = [_VP, _D, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
    L.lbm_cuboid_trace_read.restype = ctypes.c_int
    L.lbm_cuboid_timing.argtypes = [_VP, ctypes.c_int]
    L.lbm_cuboid_timing_read.argtypes = [_VP, _D]
    L.lbm_cuboid_destroy.argtypes = [_VP]
    L.lbm_cuboid_last_error.argtypes = []
    L.lbm_cuboid_last_error.restype = ctypes.c_char_p
    for name in EXPORTS:
        getattr(L, name)
    for n in ("lbm_cuboid_buffer_bytes", "lbm_cuboid_halo_plan", "lbm_cuboid_nccl_unique_id", "lbm_cuboid_create",
              "lbm_cuboid_p2p_export", "lbm_cuboid_p2p_connect",
              "lbm_cuboid_init_fields", "lbm_cuboid_init_fields_device", "lbm_cuboid_step",
              "lbm_cuboid_sync", "lbm_cuboid_get_macroscopic", "lbm_cuboid_get_macroscopic_device",
              "lbm_cuboid_get_populations", "lbm_cuboid_get_populations_planes",
              "lbm_cuboid_set_populations", "lbm_cuboid_check",
              "lbm_cuboid_set_force", "lbm_cuboid_info", "lbm_cuboid_timing", "lbm_cuboid_timing_read",
              "lbm_cuboid_destroy"):
        getattr(L, n).restype = ctypes.c_int
    _lib = L
    return L


def _check(rc):
    if rc != LBM_OK:
        raise LbmError(rc, load().lbm_cuboid_last_error().decode())


def make_params(nx, ny, nz, r, s, cs2=0.0, omega_nu=1.0, omega_xi=1.0, omega_1=1.0, omega_high=1.0,
                force=(0.0, 0.0, 0.0), bc=(0,) * 6, wall_u=0.0, corrections=0, precision=0,
                rank=0, world=1, device=0, halo=0, graphs=0, model=0, streaming=0, check_every=0) -> Params:
    p = Params()
    load().lbm_cuboid_default_params(ctypes.byref(p))
    p.nx, p.ny, p.nz = int(nx), int(ny), int(nz)
    p.r, p.s, p.cs2 = float(r), float(s), float(cs2)
    p.omega_nu, p.omega_xi = float(omega_nu), float(omega_xi)
    p.omega_1, p.omega_high = float(omega_1), float(omega_high)
    for i in range(3):
        p.force[i] = float(force[i])
    for i in range(6):
        p.bc[i] = int(bc[i])
    p.wall_u = float(wall_u)
    p.corrections, p.precision = int(corrections), int(precision)
    p.rank, p.world, p.device, p.halo = int(rank), int(world), int(device), int(halo)
    p.graphs = int(graphs)
    p.model = int(model)
    p.streaming = int(streaming)
    p.check_every = int(check_every)
    return p


def buffer_bytes(p: Params) -> int:
    b = ctypes.c_int64()
    _check(load().lbm_cuboid_buffer_bytes(ctypes.byref(p), ctypes.byref(b)))
    return b.value


def halo_plan(p: Params) -> dict:
    a = (ctypes.c_int64 * 8)()
    _check(load().lbm_cuboid_halo_plan(ctypes.byref(p), a))
    keys = ["ghost", "peer_up", "peer_down", "count", "send_up", "recv_down", "send_down", "recv_up"]
    return dict(zip(keys, list(a)))


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().lbm_cuboid_nccl_unique_id(buf))
    return buf.raw


def _host_ptr(a: np.ndarray, n: int):
    assert a.dtype == np.float64 and a.flags.c_contiguous and a.size == n, (a.dtype, a.shape, n)
    return a.ctypes.data_as(_VP)


class Lattice:
    """One z-slab of the cuboid D3Q27 lattice on one GPU (a lbm_cuboid_t handle).

    Parameters are those of lbm_cuboid_params (include/lbm_cuboid.h).  The two
    population buffers are torch uint8 tensors on `device`; the compute stream
    is torch's current stream of that device unless `stream` is given.
    """

    def __init__(self, nx, ny, nz, r, s, cs2=0.0, omega_nu=1.0, omega_xi=1.0, omega_1=1.0,
                 omega_high=1.0, force=(0.0, 0.0, 0.0), bc=(0,) * 6, wall_u=0.0, corrections=0,
                 precision=0, rank=0, world=1, device=0, halo=0, graphs=0, model=0, streaming=0,
                 nccl_uid: bytes | None = None, stream=None, check_every=0):
        import torch  # noqa: PLC0415  (device memory / streams only)

        L = load()
        self._torch = torch
        self.p = make_params(nx, ny, nz, r, s, cs2, omega_nu, omega_xi, omega_1, omega_high, force,
                             bc, wall_u, corrections, precision, rank, world, device, halo, graphs, model,
                             streaming, check_every)
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.world, self.rank = int(world), int(rank)
        self.nzl = self.nz // self.world
        self.r, self.s = float(r), float(s)
        self.device = torch.device("cuda", int(device))
        nbytes = buffer_bytes(self.p)
        nbuf = 1 if int(streaming) == STREAM_AA else 2
        if int(halo) == HALO_P2P and int(world) > 1:
            # buffers shared with other processes through CUDA IPC: plain cudaMalloc
            # allocations owned by the library (torch's allocator may hand out
            # memory that cannot be exported, e.g. expandable segments)
            self._bufs = []
        else:
            self._bufs = [torch.empty(nbytes, dtype=torch.uint8, device=self.device) for _ in range(nbuf)]
            self.p.buf_a = self._bufs[0].data_ptr()
            self.p.buf_b = self._bufs[1].data_ptr() if nbuf == 2 else None
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
            if stream.cuda_stream == 0:
                # the ABI reads a NULL stream as "library-owned"; give the handle a
                # real torch stream so callers can time and order work on it
                stream = torch.cuda.Stream(self.device)
        self.stream = stream
        self.p.stream = stream.cuda_stream
        self._uid = ctypes.create_string_buffer(nccl_uid, 128) if nccl_uid is not None else None
        self.p.nccl_uid = ctypes.cast(self._uid, _VP) if self._uid is not None else None
        h = _VP()
        _check(L.lbm_cuboid_create(ctypes.byref(self.p), ctypes.byref(h)))
        self._h = h

    # stream ordering between torch's current stream and the handle's stream
    def _consume_after_torch(self):
        cur = self._torch.cuda.current_stream(self.device)
        if cur.cuda_stream != self.stream.cuda_stream:
            self.stream.wait_stream(cur)

    def _produce_for_torch(self):
        cur = self._torch.cuda.current_stream(self.device)
        if cur.cuda_stream != self.stream.cuda_stream:
            cur.wait_stream(self.stream)

    # ---------------------------------------------------------------- fields
    @property
    def local_shape(self):
        return (self.nzl, self.ny, self.nx)

    def init_fields(self, rho, u):
        """rho [nz_l][ny][nx], u [3][nz_l][ny][nx]: numpy (host) or torch CUDA fp64 tensors."""
        n = self.nzl * self.ny * self.nx
        if hasattr(rho, "is_cuda") and rho.is_cuda:
            assert rho.dtype == self._torch.float64 and u.dtype == self._torch.float64
            assert rho.is_contiguous() and u.is_contiguous() and rho.numel() == n and u.numel() == 3 * n
            self._consume_after_torch()
            _check(load().lbm_cuboid_init_fields_device(self._h, rho.data_ptr(), u.data_ptr()))
            self._produce_for_torch()
        else:
            rho = np.ascontiguousarray(rho, dtype=np.float64)
            u = np.ascontiguousarray(u, dtype=np.float64)
            _check(load().lbm_cuboid_init_fields(self._h, _host_ptr(rho, n), _host_ptr(u, 3 * n)))

    def step(self, n: int = 1):
        _check(load().lbm_cuboid_step(self._h, int(n)))

    def sync(self):
        _check(load().lbm_cuboid_sync(self._h))

    def get_macroscopic(self, out=None, device=False):
        """(rho, u) of the stored state; host numpy arrays, or CUDA tensors if device=True."""
        n = self.nzl * self.ny * self.nx
        if device:
            t = self._torch
            rho, u = out if out is not None else (
                t.empty(self.local_shape, dtype=t.float64, device=self.device),
                t.empty((3,) + self.local_shape, dtype=t.float64, device=self.device))
            self._consume_after_torch()
            _check(load().lbm_cuboid_get_macroscopic_device(self._h, rho.data_ptr(), u.data_ptr()))
            self._produce_for_torch()
            return rho, u
        rho, u = out if out is not None else (np.empty(self.local_shape), np.empty((3,) + self.local_shape))
        _check(load().lbm_cuboid_get_macroscopic(self._h, _host_ptr(rho, n), _host_ptr(u, 3 * n)))
        return rho, u

    def get_populations(self):
        f = np.empty((27,) + self.local_shape)
        _check(load().lbm_cuboid_get_populations(self._h, _host_ptr(f, f.size)))
        return f

    def get_populations_planes(self, z_begin: int, n_planes: int):
        f = np.empty((27, n_planes, self.ny, self.nx))
        _check(load().lbm_cuboid_get_populations_planes(self._h, int(z_begin), int(n_planes),
                                                        _host_ptr(f, f.size)))
        return f

    def set_populations(self, f):
        f = np.ascontiguousarray(f, dtype=np.float64)
        _check(load().lbm_cuboid_set_populations(self._h, _host_ptr(f, 27 * self.nzl * self.ny * self.nx)))

    def check(self, raise_on_unstable=True):
        out = np.zeros(7)
        rc = load().lbm_cuboid_check(self._h, out.ctypes.data_as(_D))
        if rc != LBM_OK and (rc != LBM_EUNSTABLE or raise_on_unstable):
            _check(rc)
        return {"mass": out[0], "momentum": out[1:4].copy(), "kinetic_energy": out[4],
                "max_speed": out[5], "bad_nodes": int(out[6])}

    def set_force(self, force):
        a = np.ascontiguousarray(force, dtype=np.float64)
        _check(load().lbm_cuboid_set_force(self._h, a.ctypes.data_as(_D)))

    def info(self):
        a = (ctypes.c_int64 * 8)()
        _check(load().lbm_cuboid_info(self._h, a))
        keys = ["launches", "collide_stream_launches", "steps", "bytes_per_node_update",
                "local_nodes", "buffer_bytes", "halo", "paper_rate_kernel"]
        return dict(zip(keys, list(a)))

    def trace(self, enable: bool):
        """Start (and clear) / stop the event trace of the step structure."""
        _check(load().lbm_cuboid_trace(self._h, 1 if enable else 0))

    def trace_read(self):
        """Recorded launches: list of dicts kind/stream/zbeg/nplanes/t0_ms/t1_ms."""
        n = ctypes.c_int32(0)
        _check(load().lbm_cuboid_trace_read(self._h, None, 0, ctypes.byref(n)))
        a = np.zeros((max(n.value, 1), 6))
        _check(load().lbm_cuboid_trace_read(self._h, a.ctypes.data_as(_D), n.value, ctypes.byref(n)))
        kinds = {0: "collide", 1: "boundary", 2: "nccl_halo", 3: "density"}
        return [{"kind": kinds[int(r[0])], "stream": "compute" if r[1] == 0 else "halo", "zbeg": int(r[2]),
                 "nplanes": int(r[3]), "t0_ms": float(r[4]), "t1_ms": float(r[5])} for r in a[:n.value]]

    def kernel_name(self) -> str:
        """The collide-stream kernel this lattice's steps launch."""
        return load().lbm_cuboid_kernel_name(self._h).decode()

    def comm_ranks(self):
        """(nranks, rank) of the library's NCCL communicator, (-1, -1) without one."""
        a = (ctypes.c_int32 * 2)()
        _check(load().lbm_cuboid_comm_ranks(self._h, a))
        return int(a[0]), int(a[1])

    def p2p_export(self) -> bytes:
        """This slab's LBM_HALO_P2P descriptor (IPC handles + addresses), for its neighbours."""
        buf = ctypes.create_string_buffer(P2P_BLOB_BYTES)
        _check(load().lbm_cuboid_p2p_export(self._h, buf))
        return buf.raw

    def p2p_connect(self, blob_down: bytes | None, blob_up: bytes | None):
        """Map the neighbours' buffers (None where halo_plan has no neighbour)."""
        _check(load().lbm_cuboid_p2p_connect(self._h, blob_down, blob_up))

    def timing(self, enable: bool):
        """Enable/disable (and clear) per-launch CUDA-event timing of the collide-stream kernel."""
        _check(load().lbm_cuboid_timing(self._h, 1 if enable else 0))

    def timing_read(self):
        a = np.zeros(3)
        _check(load().lbm_cuboid_timing_read(self._h, a.ctypes.data_as(_D)))
        return {"launches": int(a[0]), "kernel_ms": float(a[1]), "node_updates": int(a[2])}

    def close(self):
        if getattr(self, "_h", None):
            load().lbm_cuboid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def p2p_neighbour_blobs(plan: dict, blobs: list) -> tuple:
    """(blob_down, blob_up) for lbm_cuboid_p2p_connect from every rank's blob
    (index = rank) and this rank's halo plan."""
    dn, up = int(plan["peer_down"]), int(plan["peer_up"])
    return (blobs[dn] if dn >= 0 else None, blobs[up] if up >= 0 else None)


def distributed_lattice(**kw) -> Lattice:
    """Create this rank's slab under an initialised torch.distributed process
    group.  NCCL halo: rank 0 makes the NCCL unique id, the group broadcasts
    it.  P2P halo (halo=HALO_P2P): every rank exports its descriptor, the group
    all-gathers them and each rank maps its two neighbours."""
    import torch.distributed as dist  # noqa: PLC0415

    world, rank = dist.get_world_size(), dist.get_rank()
    if int(kw.get("halo", HALO_AUTO)) == HALO_P2P:
        lat = Lattice(rank=rank, world=world, **kw)
        if world > 1:
            blobs = [None] * world
            dist.all_gather_object(blobs, lat.p2p_export())
            lat.p2p_connect(*p2p_neighbour_blobs(halo_plan(lat.p), blobs))
        return lat
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Lattice(rank=rank, world=world, nccl_uid=obj[0], **kw)
