// lbm_cuboid.cu -- runtime and C ABI (include/lbm_cuboid.h) of the B200
// 3D cuboid central-moment LBM.  One handle = one z-slab on one GPU.
//
// Per time step:
//   single GPU, periodic or walled z : one fused collide-stream launch over all
//                                      planes (z wrap inside the kernel)
//   ghost-plane mode (world > 1, or LBM_HALO_NCCL):
//     compute stream: wait(halo[t-1]) -> boundary planes {0, nz_l-1} -> record(bnd)
//     comm stream   : wait(bnd) -> NCCL send/recv of the 9 outgoing directions of
//                     the two boundary planes into the neighbours' ghost planes
//                     -> record(halo[t])
//     compute stream: interior planes 1..nz_l-2 (overlaps the exchange)
//   fused P2P halo (LBM_HALO_P2P):
//     halo stream   : wait(compute) -> wait(neighbours' epoch flags >= e) ->
//                     boundary planes, storing the outgoing directions into the
//                     neighbours' ghost planes and publishing epoch e + 1
//     compute stream: interior planes 1..nz_l-2 (concurrent) -> wait(halo stream)
#include "../../include/lbm_cuboid.h"
#include "cm_kernels.cuh"
#include "cm_tma.cuh"

#include <cuda.h>  // driver types only; entry points come from cudaGetDriverEntryPointByVersion
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges for nsys (no-ops without a tool)
#include <cuda_runtime.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

using lbm::Consts;

namespace {

thread_local std::string g_err;

// NVTX range for the scope of a host call (step phases show up in nsys timelines)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) return fail(LBM_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,         \
                                       cudaGetErrorString(e_));                                      \
  } while (0)

#define NC(call)                                                                                     \
  do {                                                                                               \
    ncclResult_t r_ = (call);                                                                        \
    if (r_ != ncclSuccess) return fail(LBM_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call,         \
                                       ncclGetErrorString(r_));                                      \
  } while (0)

constexpr size_t kStageBytes = size_t(256) << 20;  // host<->device staging chunk
constexpr size_t kMaxTimedLaunches = 1 << 16;
constexpr int kGraphSteps = 32;                 // steps per captured graph (even: ends on the same buffer)
constexpr int64_t kGraphMaxNodes = 4 << 20;     // auto mode: graphs below this many local nodes
constexpr int64_t kPersistMaxNodes = 0;          // auto mode: persistent kernel up to this many nodes
constexpr int kPersistChunk = 1024;              // steps per persistent launch

}  // namespace

struct lbm_cuboid {
  lbm_cuboid_params p{};
  int nzl = 0, z0 = 0;
  int64_t nxy = 0, plane = 0, buf_elems = 0;
  size_t elem = 8;
  void* buf[2] = {nullptr, nullptr};
  bool own_buf = false;
  int cur = 0;  // buf[cur] holds the stored state
  cudaStream_t stream = nullptr, comm_stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_bnd = nullptr, ev_halo = nullptr;
  bool halo_pending = false;
  bool ghost = false;  // ghost-plane mode (NCCL or fused P2P halo)
  bool paper_rates = false;  // omega_1 = omega_high = 1 -> k_collide_stream_paper
  bool fd = false;           // FULL_FD / FULL_FD_LAG: density-gradient (lambda, e_rho) terms
  bool fd_lag = false;       // FULL_FD_LAG: gradient of the stored state's density (d_rho double-buffered,
                             // written by the collision of the previous step; reading R16b)
  bool fd_fused = true;      // FULL_FD: fused 2.5D kernel or density pass + collide (default since round 2);
                             // env LBM_FD_FUSED=0/1 forces the two-pass / fused path
  std::string kname;         // lbm_cuboid_kernel_name
  bool shape_spec = false;   // plane shape compiled in (k_collide_stream_paper_shape); env LBM_SHAPE_SPEC=0 disables
  bool tma = false;          // TMA-staged collide-stream kernel (cm_tma.cuh); opt-in LBM_TMA=1
  lbm::TmaMaps tmaps[2];     // buf[i] as the 3D tensor (x, y, 27 (nz_l + 2)) for the TMA unit
  bool fd_tma = false;       // FULL_FD: TMA-staged fused kernel (cm_tma.cuh, k_collide_stream_fd_tma)
  lbm::FdTmaMaps fdmaps[2];  // its tile + ring boxes (and x-seam wrap boxes) of buf[i]
  int tma_grid = 0;          // persistent grid size of the TMA kernel (resident CTAs)
  bool xpair = false;        // fp32 storage, nx even: x-pair kernel (float2 loads/stores); opt-in LBM_XPAIR=1
  bool aa = false;           // AA in-place streaming: one buffer; cur = 0 layout R, cur = 1 layout N
  double* d_rho = nullptr;   // FULL_FD density field, population-buffer plane structure (ghost planes)
  cudaEvent_t ev_rho = nullptr;
  ncclComm_t comm = nullptr;
  int peer_down = -1, peer_up = -1;  // ranks owning the planes below / above, -1 none
  // fused P2P halo (LBM_HALO_P2P); comm_stream is the (high-priority) halo stream
  bool p2p = false, p2p_ready = false;
  unsigned int* d_sig = nullptr;  // [0] epoch from the down neighbour, [1] from the up one, [2] CTA counter
  void* peer_buf_up[2] = {nullptr, nullptr};  // neighbours' population buffers, mapped
  void* peer_buf_dn[2] = {nullptr, nullptr};
  double* peer_rho_up = nullptr;         // neighbours' FULL_FD density fields, mapped
  double* peer_rho_dn = nullptr;
  unsigned int* peer_flag_up = nullptr;  // my slot in the up neighbour's flag words ([0])
  unsigned int* peer_flag_dn = nullptr;  // my slot in the down neighbour's flag words ([1])
  std::vector<void*> ipc_open;           // IPC mappings to close
  uint32_t epoch = 0;                    // halo publishes enqueued so far
  void* wait32 = nullptr;                // cuStreamWaitValue32 (driver entry point, resolved at create)
  cudaEvent_t ev_fork = nullptr;
  Consts c{};
  double* stage = nullptr;
  size_t stage_bytes = 0;
  double* d_check = nullptr;
  // opt-in stability watch (params.check_every): the check of step watch_step
  // lands in pinned host memory and is looked at by the next step()/sync()
  double* h_watch = nullptr;
  cudaEvent_t ev_watch = nullptr;
  int64_t watch_step = -1;
  unsigned int* d_dbg = nullptr;  // [0] bounds-check flag (LBM_DEBUG_BOUNDS builds), [1] singular-system flag
  double* d_aa_lid = nullptr;     // AA + moving lid: rho of the lid-row nodes (Consts::aa_lid_rho)
  int64_t launches = 0, cs_launches = 0, steps = 0;
  // CUDA graphs of kGraphSteps steps, one per starting buffer
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  bool capturing = false;
  // optional per-launch timing of the collide-stream kernel (lbm_cuboid_timing)
  bool timing = false;
  // optional trace of the step structure (lbm_cuboid_trace): an event pair per
  // launch / halo exchange on the stream it runs on, relative to trace_base
  bool tracing = false;
  cudaEvent_t trace_base = nullptr;
  struct TraceRec {
    int kind, stream, zbeg, nplanes;
    cudaEvent_t a, b;
  };
  std::vector<TraceRec> trace;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_t;
  std::vector<int64_t> ev_t_nodes;
};

namespace {

// trace record kinds (lbm_cuboid_trace_read)
enum { TR_COLLIDE = 0, TR_BOUNDARY = 1, TR_NCCL = 2, TR_DENSITY = 3 };
constexpr size_t kMaxTrace = 1 << 16;

// event pair around work enqueued on stream s (no-op unless tracing)
struct TraceScope {
  lbm_cuboid* h;
  cudaStream_t s;
  int idx = -1;
  TraceScope(lbm_cuboid* hh, cudaStream_t ss, int kind, int zbeg, int nplanes) : h(hh), s(ss) {
    if (!h->tracing || h->capturing || h->trace.size() >= kMaxTrace) return;
    lbm_cuboid::TraceRec r{kind, s == h->stream ? 0 : 1, zbeg, nplanes, nullptr, nullptr};
    if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return;
    cudaEventRecord(r.a, s);
    h->trace.push_back(r);
    idx = int(h->trace.size()) - 1;
  }
  ~TraceScope() {
    if (idx >= 0) cudaEventRecord(h->trace[idx].b, s);
  }
};

int set_device(const lbm_cuboid* h) {
  CU(cudaSetDevice(h->p.device));
  return LBM_OK;
}

int validate(const lbm_cuboid_params* p) {
  if (!p) return fail(LBM_EINVAL, "params is NULL");
  if (p->nx < 1 || p->ny < 1 || p->nz < 1) return fail(LBM_EINVAL, "nx, ny, nz must be >= 1");
  if (p->world < 1 || p->rank < 0 || p->rank >= p->world) return fail(LBM_EINVAL, "rank/world out of range");
  if (p->nz % p->world) return fail(LBM_EINVAL, "nz (%d) must be divisible by world (%d)", p->nz, p->world);
  if (!(p->r > 0) || !(p->s > 0) || !std::isfinite(p->r) || !std::isfinite(p->s))
    return fail(LBM_EINVAL, "aspect ratios r, s must be finite and > 0");
  const double lim = std::min({1.0, p->r * p->r, p->s * p->s});
  const double cs2 = p->cs2 > 0 ? p->cs2 : lim / 3.0;
  if (!(cs2 > 0 && cs2 < lim)) return fail(LBM_EINVAL, "cs2 = %g must satisfy 0 < cs2 < min(1, r^2, s^2) = %g", cs2, lim);
  auto bad_w = [](double w) { return !(w > 0.0 && w < 2.0); };
  if (bad_w(p->omega_nu) || bad_w(p->omega_xi)) return fail(LBM_EINVAL, "omega_nu, omega_xi must lie in (0, 2)");
  if (!(p->omega_1 > 0 && p->omega_1 <= 2) || !(p->omega_high > 0 && p->omega_high <= 2))
    return fail(LBM_EINVAL, "omega_1, omega_high must lie in (0, 2]");
  for (int f = 0; f < 6; ++f)
    if (p->bc[f] < 0 || p->bc[f] > 3) return fail(LBM_EINVAL, "bc[%d] = %d is not an lbm_bc", f, p->bc[f]);
  for (int d = 0; d < 3; ++d)
    if ((p->bc[2 * d] == LBM_BC_PERIODIC) != (p->bc[2 * d + 1] == LBM_BC_PERIODIC))
      return fail(LBM_EINVAL, "faces %d and %d must be both periodic or both non-periodic", 2 * d, 2 * d + 1);
  for (int f = 0; f < 6; ++f)
    if (p->bc[f] == LBM_BC_MOVING_WALL && f != 3)
      return fail(LBM_EINVAL, "configuration error: a moving wall is supported on the +y face only (P:L751)");
  if (p->corrections < 0 || p->corrections > 4) return fail(LBM_EINVAL, "corrections must be an lbm_corr");
  if (p->precision < 0 || p->precision > 1) return fail(LBM_EINVAL, "precision must be an lbm_prec");
  if (p->halo < 0 || p->halo > 2) return fail(LBM_EINVAL, "halo must be an lbm_halo");
  if (p->graphs < 0 || p->graphs > 3) return fail(LBM_EINVAL, "graphs must be 0, 1, 2 or 3");
  if (p->model < 0 || p->model > 1) return fail(LBM_EINVAL, "model must be an lbm_model");
  if (p->streaming < 0 || p->streaming > 1) return fail(LBM_EINVAL, "streaming must be an lbm_streaming");
  if (p->check_every < 0) return fail(LBM_EINVAL, "check_every must be >= 0");
  if (p->streaming == LBM_STREAM_AA) {
    if (p->world > 1 || p->halo != LBM_HALO_AUTO)
      return fail(LBM_ENOTSUP, "AA in-place streaming is single-GPU only (no ghost-plane exchange)");
    if (p->corrections == LBM_CORR_FULL_FD || p->corrections == LBM_CORR_FULL_FD_LAG)
      return fail(LBM_ENOTSUP, "AA in-place streaming does not support FULL_FD / FULL_FD_LAG");
  }
  for (int d = 0; d < 3; ++d)
    if (!std::isfinite(p->force[d])) return fail(LBM_EINVAL, "force must be finite");
  if (!std::isfinite(p->wall_u)) return fail(LBM_EINVAL, "wall_u must be finite");
  const int64_t nxy = int64_t(p->nx) * p->ny;
  if (27 * nxy >= (int64_t(1) << 31)) return fail(LBM_EINVAL, "nx*ny too large (27*nx*ny must fit int32)");
  if (p->nz / p->world > 65535) return fail(LBM_EINVAL, "nz/world must be <= 65535");
  if (p->corrections != LBM_CORR_OFF) {
    // the 3x3 strain-rate system of App D at rest must be
    // regular (a singular system is an error), C / rho at u = 0
    const double csn = 2.0 * cs2 / p->omega_nu, csx = 2.0 * cs2 / p->omega_xi;
    const double gx = 3.0 * cs2 - 1.0, gy = 3.0 * cs2 - p->r * p->r, gz = 3.0 * cs2 - p->s * p->s;
    const double Csx = -csn + 0.5 * gx, Cbx = -csx + 0.5 * gx, Csy = csn - 0.5 * gy, Cby = -csx + 0.5 * gy,
                 Csz = csn - 0.5 * gz, Cbz = -csx + 0.5 * gz;
    // the in-flight predicate of reading R17 (note_singular) at rho = 1, u = 0; no
    // valid (r, s, cs2, omega) was found where it holds at rest (DESIGN R17), so
    // in practice the system only degenerates in flight, through the 3u^2/2 terms
    const double det = -Csx * Csz * Cby - Csy * (Csx * Cbz - Csz * Cbx);
    const double thr = 1e-12 * cs2;
    if (!(std::fabs(det) >= thr && std::fabs(Csy) >= thr && std::fabs(Csz) >= thr))
      return fail(LBM_ESINGULAR, "the strain-rate system of the corrections is singular at rest (det = %g) for these "
                  "r, s, cs2, omega_nu, omega_xi", det);
  }
  return LBM_OK;
}

void fill_consts(lbm_cuboid* h) {
  const lbm_cuboid_params& p = h->p;
  Consts& c = h->c;
  c.nx = p.nx;
  c.ny = p.ny;
  c.nzl = h->nzl;
  c.nxy = int(h->nxy);
  c.plane = h->plane;
  const double cs2 = p.cs2 > 0 ? p.cs2 : std::min({1.0, p.r * p.r, p.s * p.s}) / 3.0;
  c.r = p.r;
  c.s = p.s;
  c.cs2 = cs2;
  c.r2 = p.r * p.r;
  c.s2 = p.s * p.s;
  c.h1y = 0.5 / p.r;
  c.h2y = 0.5 / (p.r * p.r);
  c.h1z = 0.5 / p.s;
  c.h2z = 0.5 / (p.s * p.s);
  c.wn = p.omega_nu;
  c.wx = p.omega_xi;
  c.w1 = p.omega_1;
  c.wh = p.omega_high;
  c.an = 1.0 / p.omega_nu - 0.5;
  c.ab = 1.0 / p.omega_xi - 0.5;
  c.gx = 3.0 * cs2 - 1.0;
  c.gy = 3.0 * cs2 - c.r2;
  c.gz = 3.0 * cs2 - c.s2;
  c.galias = (p.corrections == LBM_CORR_FULL_LOCAL || p.corrections == LBM_CORR_FULL_FD ||
              p.corrections == LBM_CORR_FULL_FD_LAG) ? 1.0 : 0.0;
  c.corr_on = (p.corrections != LBM_CORR_OFF);
  c.csn = 2.0 * cs2 / p.omega_nu;
  c.csx = 2.0 * cs2 / p.omega_xi;
  for (int d = 0; d < 3; ++d) c.F[d] = p.force[d];
  c.c4 = cs2 * cs2;
  c.c6 = cs2 * cs2 * cs2;
  c.lid_u = (p.bc[3] == LBM_BC_MOVING_WALL) ? p.wall_u : 0.0;
  // Eq. 69 coefficients: f^eq_a - f^eq_abar at the wall (u = (U,0,0)) is
  // rho U e_x * cs2/(2 r^2) * phi_z(e_z), phi_z(0) = 1 - cs2/s^2, phi_z(+-1) = cs2/(2 s^2)
  const double py = cs2 / (2.0 * c.r2);
  c.lid_c[0] = py * cs2 / (2.0 * c.s2);
  c.lid_c[1] = py * (1.0 - cs2 / c.s2);
  c.lid_c[2] = py * cs2 / (2.0 * c.s2);
  // local faces
  auto kind = [](int bc) {
    switch (bc) {
      case LBM_BC_BOUNCE_BACK: return int(lbm::FK_BOUNCE);
      case LBM_BC_MOVING_WALL: return int(lbm::FK_MOVING);
      case LBM_BC_FREE_SLIP: return int(lbm::FK_SLIP);
      default: return int(lbm::FK_WRAP);
    }
  };
  for (int f = 0; f < 4; ++f) c.face[f] = kind(p.bc[f]);
  const bool zper = (p.bc[4] == LBM_BC_PERIODIC);
  if (h->ghost) {
    c.face[4] = (p.rank == 0 && !zper) ? kind(p.bc[4]) : int(lbm::FK_GHOST);
    c.face[5] = (p.rank == p.world - 1 && !zper) ? kind(p.bc[5]) : int(lbm::FK_GHOST);
  } else {
    c.face[4] = kind(p.bc[4]);
    c.face[5] = kind(p.bc[5]);
  }
  c.buf_elems = h->buf_elems;
  c.sing_thr = 1e-12 * cs2;
  // fast division by nx for idx < 2^31: m = ceil(2^p / nx), p = 31 + ceil(log2 nx),
  // idx / nx = umulhi(idx, m) >> (p - 32)  (nx = 1: no division)
  if (p.nx > 1) {
    int l = 0;
    while ((1u << l) < unsigned(p.nx)) ++l;
    const int pw = 31 + l;
    c.nx_mul = unsigned(((uint64_t(1) << pw) + uint64_t(p.nx) - 1) / uint64_t(p.nx));
    c.nx_shift = pw - 32;
  } else {
    c.nx_mul = 0;
    c.nx_shift = 0;
  }
  // rest weights of the isotropic density gradient (FULL_FD): f^eq at rho = 1, u = 0 per axis
  const double cc[3] = {1.0, c.r2, c.s2};
  double* ph[3] = {c.phx, c.phy, c.phz};
  for (int d = 0; d < 3; ++d) {
    ph[d][0] = cs2 / (2.0 * cc[d]);
    ph[d][1] = 1.0 - cs2 / cc[d];
    ph[d][2] = cs2 / (2.0 * cc[d]);
  }
  c.has_walls = 0;
  c.has_slip = 0;
  for (int f = 0; f < 6; ++f)
    if (c.face[f] == lbm::FK_SLIP) c.has_slip = 1;
  for (int f = 0; f < 6; ++f)
    if (c.face[f] >= lbm::FK_BOUNCE && c.face[f] <= lbm::FK_SLIP) c.has_walls = 1;
}

dim3 grid_for(const lbm_cuboid* h, int nplanes) {
  return dim3(unsigned((h->nxy + lbm::kBlock - 1) / lbm::kBlock), unsigned(nplanes), 1);
}

// P2P halo arguments of a boundary launch / halo push into the neighbours'
// buffer `which`, publishing `epoch`
template <typename T>
lbm::P2PArgs<T> p2p_args(const lbm_cuboid* h, int which, uint32_t epoch) {
  lbm::P2PArgs<T> a;
  a.up = (T*)h->peer_buf_up[which];
  a.dn = (T*)h->peer_buf_dn[which];
  a.counter = h->d_sig + 2;
  a.flag_up = h->peer_flag_up;
  a.flag_dn = h->peer_flag_dn;
  a.epoch = epoch;
  // FULL_FD_LAG: the neighbours' density fields of buffer `which` (their ghost planes
  // receive this slab's boundary-plane densities)
  const size_t half = size_t(h->nzl + 2) * size_t(h->nxy);
  a.rho_up = (h->fd_lag && h->peer_rho_up) ? h->peer_rho_up + which * half : nullptr;
  a.rho_dn = (h->fd_lag && h->peer_rho_dn) ? h->peer_rho_dn + which * half : nullptr;
  return a;
}

// FULL_FD_LAG: the density field of the state in buf[i] (the lower / upper half
// of d_rho; population-buffer plane structure with ghost planes)
double* rho_field(const lbm_cuboid* h, int i) { return h->d_rho + size_t(i) * size_t(h->nzl + 2) * size_t(h->nxy); }

// p2p_which >= 0: fused P2P boundary launch storing into the neighbours' buffer
// p2p_which and publishing p2p_epoch (LBM_HALO_P2P)
int launch_cs(lbm_cuboid* h, const void* src, void* dst, int zbeg, int nplanes, int zstride, cudaStream_t s,
              int p2p_which = -1, uint32_t p2p_epoch = 0, bool allow_timing = true) {
  if (nplanes <= 0) return LBM_OK;
  // ghost-plane mode: the boundary-plane launch starts at plane 0, the interior at 1
  TraceScope trace_scope(h, s, (h->ghost && zbeg == 0) ? TR_BOUNDARY : TR_COLLIDE, zbeg, nplanes);
  dim3 g = grid_for(h, nplanes);
  const bool fp64 = (h->p.precision == LBM_FP64);
  const bool timed = allow_timing && h->timing && h->ev_t.size() < kMaxTimedLaunches;
  if (timed) {
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    h->ev_t.push_back({a, b});
    CU(cudaEventRecord(a, s));
  }
  // FULL_FD_LAG: read the density field of the source state, write the collision's
  // density into the destination state's field
  const double* rf = h->d_rho;
  Consts cc = h->c;
  if (h->fd_lag) {
    rf = rho_field(h, src == h->buf[0] ? 0 : 1);
    cc.rf_out = rho_field(h, src == h->buf[0] ? 1 : 0);
  }
#define LBM_LAUNCH(KERNEL)                                                                                   \
  do {                                                                                                       \
    if (fp64) {                                                                                              \
      if (h->fd)                                                                                             \
        lbm::KERNEL<double, true><<<g, lbm::kBlock, 0, s>>>((const double*)src, (double*)dst, rf, cc, zbeg, \
                                                             zstride);                                       \
      else                                                                                                   \
        lbm::KERNEL<double, false><<<g, lbm::kBlock, 0, s>>>((const double*)src, (double*)dst, rf, cc, zbeg, \
                                                              zstride);                                      \
    } else {                                                                                                 \
      if (h->fd)                                                                                             \
        lbm::KERNEL<float, true><<<g, lbm::kBlock, 0, s>>>((const float*)src, (float*)dst, rf, cc, zbeg,    \
                                                            zstride);                                        \
      else                                                                                                   \
        lbm::KERNEL<float, false><<<g, lbm::kBlock, 0, s>>>((const float*)src, (float*)dst, rf, cc, zbeg,   \
                                                             zstride);                                       \
    }                                                                                                        \
  } while (0)
#define LBM_P2P(T)                                                                                           \
  do {                                                                                                       \
    const lbm::P2PArgs<T> a = p2p_args<T>(h, p2p_which, p2p_epoch);                                          \
    if (h->fd)                                                                                               \
      LBM_P2PK(T, true, a);                                                                                  \
    else                                                                                                     \
      LBM_P2PK(T, false, a);                                                                                 \
  } while (0)
#define LBM_P2PK(T, FD, a)                                                                                   \
  do {                                                                                                       \
    if (h->p.model == LBM_MODEL_RM)                                                                          \
      lbm::k_collide_stream_p2p<T, lbm::CORE_RAW, FD><<<g, lbm::kBlock, 0, s>>>((const T*)src, (T*)dst, rf,  \
                                                                                cc, zbeg, zstride, a);     \
    else if (h->paper_rates)                                                                                 \
      lbm::k_collide_stream_p2p<T, lbm::CORE_PAPER, FD><<<g, lbm::kBlock, 0, s>>>((const T*)src, (T*)dst, rf, \
                                                                                  cc, zbeg, zstride, a);   \
    else                                                                                                     \
      lbm::k_collide_stream_p2p<T, lbm::CORE_GENERIC, FD><<<g, lbm::kBlock, 0, s>>>(                         \
          (const T*)src, (T*)dst, rf, cc, zbeg, zstride, a);                                               \
  } while (0)
  if (p2p_which >= 0) {
    if (fp64)
      LBM_P2P(double);
    else
      LBM_P2P(float);
  } else if (h->fd && h->fd_fused) {
    // contiguous planes [zbeg, zbeg + nplanes) in z-chunks; strided single planes otherwise
    const int zlen = (zstride == 1) ? lbm::kFdZc : 1;
    const int zst = (zstride == 1) ? lbm::kFdZc : zstride;
    const int zend = zbeg + (nplanes - 1) * zstride + 1;
    const int nchunks = (zstride == 1) ? (nplanes + lbm::kFdZc - 1) / lbm::kFdZc : nplanes;
    const dim3 gf(unsigned((h->p.nx + lbm::kFdTx - 1) / lbm::kFdTx), unsigned((h->p.ny + lbm::kFdTy - 1) / lbm::kFdTy),
                  unsigned(nchunks));
    const int kind = (h->p.model == LBM_MODEL_RM) ? lbm::CORE_RAW : (h->paper_rates ? lbm::CORE_PAPER : lbm::CORE_GENERIC);
#define LBM_FDF(T, K)                                                                                          \
  do {                                                                                                         \
    if (h->fd_tma && zstride == 1)                                                                             \
      lbm::k_collide_stream_fd_tma<T, K><<<gf, lbm::kFdTmaThreads, lbm::TmaFdLayout<T>::kSmem, s>>>(           \
          h->fdmaps[(src == h->buf[0]) ? 0 : 1], (const T*)src, (T*)dst, rf, cc, zbeg, zst, zlen, zend);       \
    else                                                                                                       \
      lbm::k_collide_stream_fd<T, K><<<gf, lbm::kFdThreads, 0, s>>>((const T*)src, (T*)dst, rf, cc, zbeg, zst, \
                                                                    zlen, zend);                               \
  } while (0)
    if (fp64) {
      if (kind == lbm::CORE_PAPER) LBM_FDF(double, lbm::CORE_PAPER);
      else if (kind == lbm::CORE_RAW) LBM_FDF(double, lbm::CORE_RAW);
      else LBM_FDF(double, lbm::CORE_GENERIC);
    } else {
      if (kind == lbm::CORE_PAPER) LBM_FDF(float, lbm::CORE_PAPER);
      else if (kind == lbm::CORE_RAW) LBM_FDF(float, lbm::CORE_RAW);
      else LBM_FDF(float, lbm::CORE_GENERIC);
    }
#undef LBM_FDF
  } else if (h->tma && !h->fd) {
    const int ntx = int((h->p.nx + lbm::kTmaTx - 1) / lbm::kTmaTx);
    const lbm::TmaTiles tl{zbeg, zstride, nplanes, ntx, (long long)nplanes * h->p.ny * ntx};
    const unsigned grid = unsigned(std::min<long long>(tl.count, h->tma_grid));
    const lbm::TmaMaps& maps = h->tmaps[(src == h->buf[0]) ? 0 : 1];
    const int kind = (h->p.model == LBM_MODEL_RM) ? lbm::CORE_RAW : (h->paper_rates ? lbm::CORE_PAPER : lbm::CORE_GENERIC);
#define LBM_TMAK(T, K)                                                                                          \
  lbm::k_collide_stream_tma<T, K><<<grid, lbm::kTmaThreads, lbm::tma_smem_bytes<T>(), s>>>(maps, (const T*)src, \
                                                                                          (T*)dst, cc, tl)
    if (fp64) {
      if (kind == lbm::CORE_PAPER) LBM_TMAK(double, lbm::CORE_PAPER);
      else if (kind == lbm::CORE_RAW) LBM_TMAK(double, lbm::CORE_RAW);
      else LBM_TMAK(double, lbm::CORE_GENERIC);
    } else {
      if (kind == lbm::CORE_PAPER) LBM_TMAK(float, lbm::CORE_PAPER);
      else if (kind == lbm::CORE_RAW) LBM_TMAK(float, lbm::CORE_RAW);
      else LBM_TMAK(float, lbm::CORE_GENERIC);
    }
#undef LBM_TMAK
  } else if (h->xpair && !fp64 && !h->fd) {
    const dim3 gp(unsigned((h->nxy / 2 + lbm::kBlock - 1) / lbm::kBlock), unsigned(nplanes), 1);
    if (h->p.model == LBM_MODEL_RM)
      lbm::k_collide_stream_xpair<lbm::CORE_RAW><<<gp, lbm::kBlock, 0, s>>>((const float*)src, (float*)dst, cc, zbeg, zstride);
    else if (h->paper_rates)
      lbm::k_collide_stream_xpair<lbm::CORE_PAPER><<<gp, lbm::kBlock, 0, s>>>((const float*)src, (float*)dst, cc, zbeg, zstride);
    else
      lbm::k_collide_stream_xpair<lbm::CORE_GENERIC><<<gp, lbm::kBlock, 0, s>>>((const float*)src, (float*)dst, cc, zbeg, zstride);
  } else if (h->shape_spec && (!h->fd || !h->fd_fused) && h->paper_rates && h->p.model == LBM_MODEL_CM) {
    // compile-time plane shape (k_collide_stream_paper_shape); FULL_FD two-pass and FULL_FD_LAG too
#define LBM_SHAPE(T, NX, NY)                                                                                     \
  do {                                                                                                           \
    if (h->fd)                                                                                                   \
      lbm::k_collide_stream_paper_shape<T, NX, NY, true><<<g, lbm::kBlock, 0, s>>>((const T*)src, (T*)dst, rf,  \
                                                                                  cc, zbeg, zstride);          \
    else                                                                                                         \
      lbm::k_collide_stream_paper_shape<T, NX, NY, false><<<g, lbm::kBlock, 0, s>>>((const T*)src, (T*)dst, rf, \
                                                                                   cc, zbeg, zstride);         \
  } while (0)
#define LBM_SHAPES(T)                                                              \
  do {                                                                             \
    const int nx_ = h->p.nx, ny_ = h->p.ny;                                        \
    if (nx_ == 512 && ny_ == 512) LBM_SHAPE(T, 512, 512);                          \
    else if (nx_ == 256 && ny_ == 256) LBM_SHAPE(T, 256, 256);                     \
    else if (nx_ == 512 && ny_ == 256) LBM_SHAPE(T, 512, 256);                     \
    else LBM_SHAPE(T, 1024, 1024);                                                 \
  } while (0)
    if (fp64)
      LBM_SHAPES(double);
    else
      LBM_SHAPES(float);
#undef LBM_SHAPES
#undef LBM_SHAPE
  } else if (h->p.model == LBM_MODEL_RM)
    LBM_LAUNCH(k_collide_stream_raw);
  else if (h->paper_rates)
    LBM_LAUNCH(k_collide_stream_paper);
  else
    LBM_LAUNCH(k_collide_stream);
#undef LBM_LAUNCH
#undef LBM_P2P
#undef LBM_P2PK
  CU(cudaGetLastError());
  if (timed) {
    CU(cudaEventRecord(h->ev_t.back().second, s));
    h->ev_t_nodes.push_back(int64_t(nplanes) * h->nxy);
  }
  if (!h->capturing) {
    h->launches++;
    h->cs_launches++;
  }
  return LBM_OK;
}

// AA in-place step over the whole slab: odd kernel from layout R (cur == 0),
// even kernel from layout N (cur == 1)
int launch_aa(lbm_cuboid* h, cudaStream_t s) {
  dim3 g = grid_for(h, h->nzl);
  const bool fp64 = (h->p.precision == LBM_FP64), odd = (h->cur == 0);
  const int kind = (h->p.model == LBM_MODEL_RM) ? lbm::CORE_RAW : (h->paper_rates ? lbm::CORE_PAPER : lbm::CORE_GENERIC);
  const bool timed = h->timing && h->ev_t.size() < kMaxTimedLaunches;
  if (timed) {
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    h->ev_t.push_back({a, b});
    CU(cudaEventRecord(a, s));
  }
#define LBM_AA(T, K)                                                                                   \
  do {                                                                                                 \
    if (odd)                                                                                           \
      lbm::k_aa<T, K, true><<<g, lbm::kBlock, 0, s>>>((T*)h->buf[0], h->c, 0, 1);                    \
    else                                                                                               \
      lbm::k_aa<T, K, false><<<g, lbm::kBlock, 0, s>>>((T*)h->buf[0], h->c, 0, 1);                   \
  } while (0)
#define LBM_AAS(T, NX, NY)                                                                              \
  do {                                                                                                  \
    if (odd)                                                                                            \
      lbm::k_aa_shape<T, true, NX, NY><<<g, lbm::kBlock, 0, s>>>((T*)h->buf[0], h->c, 0, 1);          \
    else                                                                                                \
      lbm::k_aa_shape<T, false, NX, NY><<<g, lbm::kBlock, 0, s>>>((T*)h->buf[0], h->c, 0, 1);         \
  } while (0)
#define LBM_AASHAPES(T)                                                                                 \
  do {                                                                                                  \
    if (h->p.nx == 512 && h->p.ny == 512) LBM_AAS(T, 512, 512);                                         \
    else if (h->p.nx == 256 && h->p.ny == 256) LBM_AAS(T, 256, 256);                                    \
    else if (h->p.nx == 512 && h->p.ny == 256) LBM_AAS(T, 512, 256);                                    \
    else LBM_AAS(T, 1024, 1024);                                                                        \
  } while (0)
  if (h->shape_spec && kind == lbm::CORE_PAPER && h->p.model == LBM_MODEL_CM) {
    if (fp64)
      LBM_AASHAPES(double);
    else
      LBM_AASHAPES(float);
  } else if (fp64) {
    if (kind == lbm::CORE_PAPER) LBM_AA(double, lbm::CORE_PAPER);
    else if (kind == lbm::CORE_RAW) LBM_AA(double, lbm::CORE_RAW);
    else LBM_AA(double, lbm::CORE_GENERIC);
  } else {
    if (kind == lbm::CORE_PAPER) LBM_AA(float, lbm::CORE_PAPER);
    else if (kind == lbm::CORE_RAW) LBM_AA(float, lbm::CORE_RAW);
    else LBM_AA(float, lbm::CORE_GENERIC);
  }
#undef LBM_AASHAPES
#undef LBM_AAS
#undef LBM_AA
  CU(cudaGetLastError());
  if (timed) {
    CU(cudaEventRecord(h->ev_t.back().second, s));
    h->ev_t_nodes.push_back(int64_t(h->nzl) * h->nxy);
  }
  if (!h->capturing) {
    h->launches++;
    h->cs_launches++;
  }
  return LBM_OK;
}

// layout selector of the diagnostic kernels: 0 two-buffer, 1 AA layout R, 2 AA layout N
int aa_mode(const lbm_cuboid* h) { return h->aa ? (h->cur == 0 ? 1 : 2) : 0; }

// FULL_FD density pass over planes zbeg + i*zstride of the local slab
int launch_density(lbm_cuboid* h, const void* src, int zbeg, int nplanes, int zstride, cudaStream_t s) {
  if (nplanes <= 0) return LBM_OK;
  TraceScope trace_scope(h, s, TR_DENSITY, zbeg, nplanes);
  dim3 g = grid_for(h, nplanes);
  if (h->p.precision == LBM_FP64)
    lbm::k_density<double><<<g, lbm::kBlock, 0, s>>>((const double*)src, h->d_rho, h->c, zbeg, zstride);
  else
    lbm::k_density<float><<<g, lbm::kBlock, 0, s>>>((const float*)src, h->d_rho, h->c, zbeg, zstride);
  CU(cudaGetLastError());
  if (!h->capturing) h->launches++;
  return LBM_OK;
}

// TMA kernel: tensor maps of both buffers, shared-memory opt-in, persistent grid
typedef CUresult (*PfnEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
template <typename F>
int driver_fn(const char* name, F* out);

template <typename T>
int tma_kernel_setup(lbm_cuboid* h, const void* fn) {
  const int smem = int(lbm::tma_smem_bytes<T>());
  CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0, sms = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, lbm::kTmaThreads, smem));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->p.device));
  if (per_sm < 1) return fail(LBM_ECUDA, "TMA kernel cannot be resident");
  h->tma_grid = per_sm * sms;
  return LBM_OK;
}

int tma_setup(lbm_cuboid* h) {
  PfnEncodeTiled enc = nullptr;
  int rc;
  if ((rc = driver_fn("cuTensorMapEncodeTiled", &enc))) return rc;
  const bool fp64 = (h->p.precision == LBM_FP64);
  const cuuint64_t e = fp64 ? 8 : 4;
  const cuuint64_t dims[3] = {cuuint64_t(h->p.nx), cuuint64_t(h->p.ny), cuuint64_t(27) * cuuint64_t(h->nzl + 2)};
  const cuuint64_t strides[2] = {cuuint64_t(h->p.nx) * e, cuuint64_t(h->nxy) * e};
  // boxes: the tile (e_x = 0), the tile widened by 16 bytes on both sides (e_x
  // = +-1: a box must start on a 16-byte boundary), 16 bytes (the x-wrap column)
  const cuuint32_t V = cuuint32_t(16 / e);
  const cuuint32_t boxes[3][3] = {{cuuint32_t(lbm::kTmaTx), 1, 1}, {cuuint32_t(lbm::kTmaTx) + 2 * V, 1, 1}, {V, 1, 1}};
  const cuuint32_t estr[3] = {1, 1, 1};
  for (int i = 0; i < 2; ++i) {
    CUtensorMap* maps[3] = {&h->tmaps[i].center, &h->tmaps[i].shift, &h->tmaps[i].wrap};
    for (int w = 0; w < 3; ++w) {
      CUresult r = enc(maps[w], fp64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, h->buf[i],
                       dims, strides, boxes[w], estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(LBM_ECUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
    }
  }
  using namespace lbm;
  const int kind = (h->p.model == LBM_MODEL_RM) ? CORE_RAW : (h->paper_rates ? CORE_PAPER : CORE_GENERIC);
  const void* fn;
  if (fp64)
    fn = kind == CORE_PAPER ? (const void*)k_collide_stream_tma<double, CORE_PAPER>
         : kind == CORE_RAW ? (const void*)k_collide_stream_tma<double, CORE_RAW>
                            : (const void*)k_collide_stream_tma<double, CORE_GENERIC>;
  else
    fn = kind == CORE_PAPER ? (const void*)k_collide_stream_tma<float, CORE_PAPER>
         : kind == CORE_RAW ? (const void*)k_collide_stream_tma<float, CORE_RAW>
                            : (const void*)k_collide_stream_tma<float, CORE_GENERIC>;
  return fp64 ? tma_kernel_setup<double>(h, fn) : tma_kernel_setup<float>(h, fn);
}

// Fraction of the FULL_FD tiles (kFdTx x kFdTy) that the TMA kernel stages
// (the predicate of k_collide_stream_fd_tma)
double fd_tma_staged_fraction(int nx, int ny, bool xper) {
  const int ntx = (nx + lbm::kFdTx - 1) / lbm::kFdTx, nty = (ny + lbm::kFdTy - 1) / lbm::kFdTy;
  const bool seam_ok = xper && nx % lbm::kFdTx == 0 && nx >= 2 * lbm::kFdTx;
  int sx = 0, sy = 0;
  for (int b = 0; b < ntx; ++b) {
    const int x0 = b * lbm::kFdTx;
    sx += (seam_ok && (x0 == 0 || x0 + lbm::kFdTx == nx)) || (x0 >= lbm::kFdTx && x0 + lbm::kFdTx + 2 <= nx);
  }
  for (int b = 0; b < nty; ++b) {
    const int y0 = b * lbm::kFdTy;
    sy += y0 >= 2 && y0 + lbm::kFdTy + 2 <= ny;
  }
  return double(sx) * double(sy) / (double(ntx) * double(nty));
}

// FULL_FD TMA kernel: one tensor map per buffer (box kFdTx + 2V columns x
// kFdTy + 2 rows x 1 slot), shared-memory opt-in of the instantiation in use
int fd_tma_setup(lbm_cuboid* h) {
  PfnEncodeTiled enc = nullptr;
  int rc;
  if ((rc = driver_fn("cuTensorMapEncodeTiled", &enc))) return rc;
  const bool fp64 = (h->p.precision == LBM_FP64);
  const cuuint64_t e = fp64 ? 8 : 4;
  const cuuint64_t dims[3] = {cuuint64_t(h->p.nx), cuuint64_t(h->p.ny), cuuint64_t(27) * cuuint64_t(h->nzl + 2)};
  const cuuint64_t strides[2] = {cuuint64_t(h->p.nx) * e, cuuint64_t(h->nxy) * e};
  const cuuint32_t V = cuuint32_t(16 / e);
  const cuuint32_t boxes[2][3] = {{cuuint32_t(lbm::kFdTx) + 2 * V, cuuint32_t(lbm::kFdTy + 2), 1},
                                  {V, cuuint32_t(lbm::kFdTy + 2), 1}};
  const cuuint32_t estr[3] = {1, 1, 1};
  for (int i = 0; i < 2; ++i) {
    CUtensorMap* maps[2] = {&h->fdmaps[i].box, &h->fdmaps[i].wrap};
    for (int w = 0; w < 2; ++w) {
      CUresult r = enc(maps[w], fp64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                       h->buf[i], dims, strides, boxes[w], estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(LBM_ECUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
    }
  }
  using namespace lbm;
  const int kind = (h->p.model == LBM_MODEL_RM) ? CORE_RAW : (h->paper_rates ? CORE_PAPER : CORE_GENERIC);
  const void* fn;
  int smem;
  if (fp64) {
    fn = kind == CORE_PAPER ? (const void*)k_collide_stream_fd_tma<double, CORE_PAPER>
         : kind == CORE_RAW ? (const void*)k_collide_stream_fd_tma<double, CORE_RAW>
                            : (const void*)k_collide_stream_fd_tma<double, CORE_GENERIC>;
    smem = int(TmaFdLayout<double>::kSmem);
  } else {
    fn = kind == CORE_PAPER ? (const void*)k_collide_stream_fd_tma<float, CORE_PAPER>
         : kind == CORE_RAW ? (const void*)k_collide_stream_fd_tma<float, CORE_RAW>
                            : (const void*)k_collide_stream_fd_tma<float, CORE_GENERIC>;
    smem = int(TmaFdLayout<float>::kSmem);
  }
  CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // all of the unified L1 / shared memory as shared memory (2-3 CTAs per SM)
  CU(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, int(cudaSharedmemCarveoutMaxShared)));
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kFdTmaThreads, smem));
  if (per_sm < 1) return fail(LBM_ECUDA, "FULL_FD TMA kernel cannot be resident");
  return LBM_OK;
}

void drop_graphs(lbm_cuboid* h) {
  if (h->gexec[0] || h->gexec[1]) cudaStreamSynchronize(h->stream);  // a replay may still be running
  for (auto& g : h->gexec)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
}

bool use_persistent(const lbm_cuboid* h) {
  if (h->ghost || h->aa || h->fd_lag) return false;
  return h->p.graphs == 3 || (h->p.graphs == 0 && h->nxy * h->nzl <= kPersistMaxNodes);
}

bool use_graphs(const lbm_cuboid* h) {
  if (h->ghost || h->timing || h->tracing || h->p.graphs == 1 || h->p.graphs == 3) return false;
  return h->p.graphs == 2 || h->nxy * h->nzl < kGraphMaxNodes;
}

template <typename T>
const void* persistent_fn(int kind, bool fd) {
  using namespace lbm;
  if (kind == CORE_PAPER) return fd ? (const void*)k_persistent<T, CORE_PAPER, true> : (const void*)k_persistent<T, CORE_PAPER, false>;
  if (kind == CORE_RAW) return fd ? (const void*)k_persistent<T, CORE_RAW, true> : (const void*)k_persistent<T, CORE_RAW, false>;
  return fd ? (const void*)k_persistent<T, CORE_GENERIC, true> : (const void*)k_persistent<T, CORE_GENERIC, false>;
}

// nsteps steps in cooperative launches of at most kPersistChunk steps, each with
// as many CTAs as can be co-resident (capped at one node per thread)
int launch_persistent(lbm_cuboid* h, int64_t nsteps) {
  const int kind = (h->p.model == LBM_MODEL_RM) ? lbm::CORE_RAW : (h->paper_rates ? lbm::CORE_PAPER : lbm::CORE_GENERIC);
  const bool fp64 = (h->p.precision == LBM_FP64);
  const void* fn = fp64 ? persistent_fn<double>(kind, h->fd) : persistent_fn<float>(kind, h->fd);
  int per_sm = 0, sms = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, lbm::kBlock, 0));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->p.device));
  const int64_t nodes = h->nxy * h->nzl;
  const int64_t want = (nodes + lbm::kBlock - 1) / lbm::kBlock;
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(per_sm) * sms)));
  if (per_sm < 1) return fail(LBM_ECUDA, "persistent kernel cannot be resident");
  while (nsteps > 0) {
    int n = int(std::min<int64_t>(nsteps, kPersistChunk));
    int cur = h->cur;
    void* b0 = h->buf[0];
    void* b1 = h->buf[1];
    double* rf = h->d_rho;
    void* args[] = {&b0, &b1, &rf, (void*)&h->c, &cur, &n};
    const bool timed = h->timing && h->ev_t.size() < kMaxTimedLaunches;
    if (timed) {
      cudaEvent_t a, b;
      CU(cudaEventCreate(&a));
      CU(cudaEventCreate(&b));
      h->ev_t.push_back({a, b});
      CU(cudaEventRecord(a, h->stream));
    }
    CU(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(lbm::kBlock), args, 0, h->stream));
    if (timed) {
      CU(cudaEventRecord(h->ev_t.back().second, h->stream));
      h->ev_t_nodes.push_back(int64_t(n) * nodes);
    }
    h->launches++;
    h->cs_launches++;
    h->steps += n;
    if (n & 1) h->cur ^= 1;
    nsteps -= n;
  }
  return LBM_OK;
}

int step_once(lbm_cuboid* h);

// capture kGraphSteps single-GPU steps starting from buffer `start`
int capture_graph(lbm_cuboid* h, int start) {
  cudaGraph_t g = nullptr;
  CU(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  h->capturing = true;
  int rc = LBM_OK;
  const int cur0 = h->cur;
  h->cur = start;
  for (int t = 0; t < kGraphSteps && rc == LBM_OK; ++t) {
    rc = step_once(h);
    h->cur ^= 1;  // kGraphSteps is even: ends on `start`
  }
  h->cur = cur0;
  h->capturing = false;
  cudaError_t e = cudaStreamEndCapture(h->stream, &g);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) return fail(LBM_ECUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&h->gexec[start], g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    h->gexec[start] = nullptr;
    return fail(LBM_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
  }
  return LBM_OK;
}

// Halo plan (element offsets into one buffer): see lbm_cuboid_halo_plan().
struct HaloPlan {
  bool ghost;
  int peer_up, peer_down;
  int64_t count, send_up, recv_dn, send_dn, recv_up;
};

HaloPlan make_plan(const lbm_cuboid_params* p) {
  HaloPlan hp{};
  const bool zper = (p->bc[4] == LBM_BC_PERIODIC);
  hp.ghost = (p->world > 1) || (p->halo != LBM_HALO_AUTO && zper);
  hp.peer_up = hp.peer_down = -1;
  if (hp.ghost) {
    hp.peer_up = (p->rank < p->world - 1 || zper) ? (p->rank + 1) % p->world : -1;
    hp.peer_down = (p->rank > 0 || zper) ? (p->rank - 1 + p->world) % p->world : -1;
  }
  const int64_t nxy = int64_t(p->nx) * p->ny, plane = 27 * nxy, nzl = p->nz / p->world;
  hp.count = 9 * nxy;
  // internal q = (ex+1) + 3(ey+1) + 9(ez+1): q 0..8 have e_z = -1, q 18..26 e_z = +1
  hp.send_up = nzl * plane + 18 * nxy;        // plane p = nz_l (z = nz_l - 1)
  hp.recv_dn = 0 * plane + 18 * nxy;          // ghost p = 0, pulled by z = 0
  hp.send_dn = 1 * plane + 0 * nxy;           // plane p = 1 (z = 0)
  hp.recv_up = (nzl + 1) * plane + 0 * nxy;   // ghost p = nz_l + 1, pulled by z = nz_l - 1
  return hp;
}

int p2p_push(lbm_cuboid* h, int which);

// NCCL exchange of buffer `which`'s boundary planes into the neighbours' ghost
// planes, on the comm stream, after the work already enqueued on the compute stream.
int exchange(lbm_cuboid* h, int which) {
  if (!h->ghost) return LBM_OK;
  NvtxRange nv("lbm halo exchange");
  if (h->p2p) return p2p_push(h, which);
  CU(cudaEventRecord(h->ev_bnd, h->stream));
  CU(cudaStreamWaitEvent(h->comm_stream, h->ev_bnd, 0));
  const HaloPlan hp = make_plan(&h->p);
  const ncclDataType_t dt = (h->p.precision == LBM_FP64) ? ncclDouble : ncclFloat;
  TraceScope trace_scope(h, h->comm_stream, TR_NCCL, 0, 2);
  char* b = (char*)h->buf[which];
  const size_t e = h->elem, cnt = size_t(hp.count);
  // NCCL matches the sends and recvs between one pair of ranks in issue order;
  // this order is right also when both neighbours are one rank (world 2,
  // periodic) or this rank itself (world 1): the k-th send meets the k-th recv.
  NC(ncclGroupStart());
  if (hp.peer_up >= 0) NC(ncclSend(b + hp.send_up * e, cnt, dt, hp.peer_up, h->comm, h->comm_stream));
  if (hp.peer_down >= 0) NC(ncclRecv(b + hp.recv_dn * e, cnt, dt, hp.peer_down, h->comm, h->comm_stream));
  if (hp.peer_down >= 0) NC(ncclSend(b + hp.send_dn * e, cnt, dt, hp.peer_down, h->comm, h->comm_stream));
  if (hp.peer_up >= 0) NC(ncclRecv(b + hp.recv_up * e, cnt, dt, hp.peer_up, h->comm, h->comm_stream));
  if (h->fd_lag) {
    // FULL_FD_LAG: the boundary planes of the new state's density field (written by
    // the boundary launch) into the neighbours' density ghost planes, same order
    double* r = rho_field(h, which);
    const size_t n = size_t(h->nxy), nzl = size_t(h->nzl);
    if (hp.peer_up >= 0) NC(ncclSend(r + nzl * n, n, ncclDouble, hp.peer_up, h->comm, h->comm_stream));
    if (hp.peer_down >= 0) NC(ncclRecv(r, n, ncclDouble, hp.peer_down, h->comm, h->comm_stream));
    if (hp.peer_down >= 0) NC(ncclSend(r + n, n, ncclDouble, hp.peer_down, h->comm, h->comm_stream));
    if (hp.peer_up >= 0) NC(ncclRecv(r + (nzl + 1) * n, n, ncclDouble, hp.peer_up, h->comm, h->comm_stream));
  }
  NC(ncclGroupEnd());
  CU(cudaEventRecord(h->ev_halo, h->comm_stream));
  h->halo_pending = true;
  return LBM_OK;
}

// FULL_FD: the density of the two boundary planes into the neighbours' ghost
// planes (same peers and order as the population exchange), then the compute
// stream waits for it.
int exchange_rho(lbm_cuboid* h) {
  if (!h->ghost) return LBM_OK;
  CU(cudaEventRecord(h->ev_bnd, h->stream));
  CU(cudaStreamWaitEvent(h->comm_stream, h->ev_bnd, 0));
  const HaloPlan hp = make_plan(&h->p);
  const size_t n = size_t(h->nxy), nzl = size_t(h->nzl);
  double* r = h->d_rho;
  NC(ncclGroupStart());
  if (hp.peer_up >= 0) NC(ncclSend(r + nzl * n, n, ncclDouble, hp.peer_up, h->comm, h->comm_stream));
  if (hp.peer_down >= 0) NC(ncclRecv(r, n, ncclDouble, hp.peer_down, h->comm, h->comm_stream));
  if (hp.peer_down >= 0) NC(ncclSend(r + n, n, ncclDouble, hp.peer_down, h->comm, h->comm_stream));
  if (hp.peer_up >= 0) NC(ncclRecv(r + (nzl + 1) * n, n, ncclDouble, hp.peer_up, h->comm, h->comm_stream));
  NC(ncclGroupEnd());
  CU(cudaEventRecord(h->ev_rho, h->comm_stream));
  CU(cudaStreamWaitEvent(h->stream, h->ev_rho, 0));
  return LBM_OK;
}

int wait_halo(lbm_cuboid* h) {
  if (h->halo_pending) {
    CU(cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
    h->halo_pending = false;
  }
  return LBM_OK;
}

// ------------------------------------------------------- fused P2P halo (LBM_HALO_P2P)
typedef CUresult (*PfnWaitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PfnAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

template <typename F>
int driver_fn(const char* name, F* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
  CU(cudaGetDriverEntryPointByVersion(name, &fn, 12000, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !fn) return fail(LBM_ECUDA, "driver entry point %s is unavailable", name);
  *out = reinterpret_cast<F>(fn);
  return LBM_OK;
}

// Descriptor exchanged between neighbours (lbm_cuboid_p2p_export / _connect).
struct P2PBlob {
  char magic[8];
  int32_t pid, device, rank, world, precision, nx, ny, nzl, ipc_ok, pad;
  int64_t buf_elems;
  uint64_t ptr[4];   // buffer 0, buffer 1, flag words, FULL_FD density field or 0 (exporter's addresses)
  uint64_t off[4];   // offset of ptr[i] from the base of its allocation
  cudaIpcMemHandle_t ipc[4];
};
static_assert(sizeof(P2PBlob) <= LBM_P2P_BLOB_BYTES, "P2P blob too large");
constexpr char kBlobMagic[8] = {'L', 'B', 'M', 'P', '2', 'P', '1', 0};

// the halo stream runs after everything already enqueued on the compute stream
int p2p_fork(lbm_cuboid* h) {
  CU(cudaEventRecord(h->ev_fork, h->stream));
  CU(cudaStreamWaitEvent(h->comm_stream, h->ev_fork, 0));
  return LBM_OK;
}

// the compute stream continues after the halo stream's work
int p2p_join(lbm_cuboid* h) {
  CU(cudaEventRecord(h->ev_bnd, h->comm_stream));
  CU(cudaStreamWaitEvent(h->stream, h->ev_bnd, 0));
  return LBM_OK;
}

// Before publish e + 1 (e = h->epoch): both neighbours have completed publish e,
// so (i) the ghost planes this slab reads next hold their data of the previous
// time level and (ii) they no longer read the ghost planes this publish writes
// (their last reader was their publish e or earlier).  Stream-ordered wait on
// the flag words in this GPU's memory; nothing spins.
int p2p_wait(lbm_cuboid* h) {
  const PfnWaitValue32 wait32 = reinterpret_cast<PfnWaitValue32>(h->wait32);
  const CUstream cs = (CUstream)h->comm_stream;
  if (h->peer_down >= 0) {
    CUresult r = wait32(cs, (CUdeviceptr)(h->d_sig + 0), h->epoch, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(LBM_ECUDA, "cuStreamWaitValue32 failed (%d)", int(r));
  }
  if (h->peer_up >= 0) {
    CUresult r = wait32(cs, (CUdeviceptr)(h->d_sig + 1), h->epoch, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(LBM_ECUDA, "cuStreamWaitValue32 failed (%d)", int(r));
  }
  return LBM_OK;
}

int p2p_ready(const lbm_cuboid* h) {
  if (!h->p2p_ready) return fail(LBM_EINVAL, "LBM_HALO_P2P: call lbm_cuboid_p2p_connect() on every rank first");
  return LBM_OK;
}

// Halo publish of buffer `which` without a collision (init / set_populations).
int p2p_push(lbm_cuboid* h, int which) {
  int rc;
  if ((rc = p2p_ready(h)) || (rc = p2p_fork(h)) || (rc = p2p_wait(h))) return rc;
  const dim3 g(unsigned((9 * h->nxy + lbm::kBlock - 1) / lbm::kBlock), 2, 1);
  const double* rsrc = h->fd_lag ? rho_field(h, which) : nullptr;
  if (h->p.precision == LBM_FP64)
    lbm::k_halo_push<double><<<g, lbm::kBlock, 0, h->comm_stream>>>((const double*)h->buf[which], rsrc, h->c,
                                                                     p2p_args<double>(h, which, h->epoch + 1));
  else
    lbm::k_halo_push<float><<<g, lbm::kBlock, 0, h->comm_stream>>>((const float*)h->buf[which], rsrc, h->c,
                                                                    p2p_args<float>(h, which, h->epoch + 1));
  CU(cudaGetLastError());
  h->launches++;
  h->epoch++;
  return p2p_join(h);
}

// One time step with the fused halo: boundary planes on the halo stream
// (storing into the neighbours' ghost planes of buffer cur ^ 1), interior
// planes concurrently on the compute stream, then join.
int p2p_step(lbm_cuboid* h) {
  NvtxRange nv("lbm step (P2P halo)");
  int rc;
  if ((rc = p2p_ready(h))) return rc;
  const int which = h->cur ^ 1;
  const void* src = h->buf[h->cur];
  void* dst = h->buf[which];
  const bool timed = h->timing && h->ev_t.size() < kMaxTimedLaunches;
  if (timed) {  // one event pair per step around both launches (they overlap)
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    h->ev_t.push_back({a, b});
    CU(cudaEventRecord(a, h->stream));
  }
  if ((rc = p2p_fork(h)) || (rc = p2p_wait(h))) return rc;
  const int nb = (h->nzl > 1) ? 2 : 1;
  if (h->fd && !h->fd_lag) {
    // FULL_FD: publish the same-time density of the boundary planes into the
    // neighbours' density ghost planes first, then wait for theirs
    // planes the boundary-plane collision needs: 0, 1, nz_l - 2, nz_l - 1 (distinct)
    lbm::PlaneList pl{};
    int np = 0;
    for (int z : {0, 1, h->nzl - 2, h->nzl - 1}) {
      bool seen = (z < 0 || z >= h->nzl);
      for (int i = 0; i < np; ++i) seen = seen || (pl.z[i] == z);
      if (!seen) pl.z[np++] = z;
    }
    const dim3 gd = grid_for(h, np);
    lbm::P2PArgs<double> ra{};
    ra.up = h->peer_rho_up;
    ra.dn = h->peer_rho_dn;
    ra.counter = h->d_sig + 2;
    ra.flag_up = h->peer_flag_up;
    ra.flag_dn = h->peer_flag_dn;
    ra.epoch = h->epoch + 1;
    if (h->p.precision == LBM_FP64)
      lbm::k_density_p2p<double><<<gd, lbm::kBlock, 0, h->comm_stream>>>((const double*)src, h->d_rho, h->c, pl,
                                                                          ra);
    else
      lbm::k_density_p2p<float><<<gd, lbm::kBlock, 0, h->comm_stream>>>((const float*)src, h->d_rho, h->c, pl,
                                                                         ra);
    CU(cudaGetLastError());
    h->launches++;
    h->epoch++;
    // the interior's fused FULL_FD kernel takes the density of planes 0 and
    // nz_l - 1 from d_rho (ring_rho: it never reads the ghost planes, which the
    // neighbours overwrite once this slab's boundary launch has published)
    CU(cudaEventRecord(h->ev_rho, h->comm_stream));
    CU(cudaStreamWaitEvent(h->stream, h->ev_rho, 0));
    if ((rc = p2p_wait(h))) return rc;
  }
  if ((rc = launch_cs(h, src, dst, 0, nb, std::max(1, h->nzl - 1), h->comm_stream, which, h->epoch + 1, false)))
    return rc;
  h->epoch++;
  if ((rc = launch_cs(h, src, dst, 1, h->nzl - 2, 1, h->stream, -1, 0, false))) return rc;
  if ((rc = p2p_join(h))) return rc;
  if (timed) {
    CU(cudaEventRecord(h->ev_t.back().second, h->stream));
    h->ev_t_nodes.push_back(int64_t(h->nzl) * h->nxy);
  }
  return LBM_OK;
}

int ensure_stage(lbm_cuboid* h, size_t bytes) {
  if (h->stage_bytes >= bytes) return LBM_OK;
  if (h->stage) {
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaFree(h->stage));
    h->stage = nullptr;
    h->stage_bytes = 0;
  }
  if (cudaMalloc(&h->stage, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(LBM_ENOMEM, "cudaMalloc(%zu) for the staging buffer failed", bytes);
  }
  h->stage_bytes = bytes;
  return LBM_OK;
}

// planes per staging chunk for `per_node` doubles per node
int chunk_planes(const lbm_cuboid* h, int per_node) {
  const size_t per_plane = size_t(per_node) * size_t(h->nxy) * sizeof(double);
  return int(std::max<size_t>(1, std::min<size_t>(h->nzl, kStageBytes / per_plane)));
}

template <typename T>
int init_kernel(lbm_cuboid* h, const double* rho, const double* u, long long ustride, int zbeg, int n) {
  lbm::k_init<T><<<grid_for(h, n), lbm::kBlock, 0, h->stream>>>(rho, u, ustride, (T*)h->buf[h->cur], h->c, zbeg,
                                                                 h->aa ? 1 : 0);
  CU(cudaGetLastError());
  h->launches++;
  return LBM_OK;
}

// AA with the moving lid: densities of the lid-row nodes of the stored layout-R
// state (after init_fields / set_populations) for the first odd step
// FULL_FD_LAG: density field of the stored state in buf[cur] (after init_fields /
// set_populations), before its ghost planes are exchanged
int stored_rho(lbm_cuboid* h) {
  if (!h->fd_lag) return LBM_OK;
  const dim3 g = grid_for(h, h->nzl);
  if (h->p.precision == LBM_FP64)
    lbm::k_stored_rho<double><<<g, lbm::kBlock, 0, h->stream>>>((const double*)h->buf[h->cur], rho_field(h, h->cur),
                                                                 h->c, 0);
  else
    lbm::k_stored_rho<float><<<g, lbm::kBlock, 0, h->stream>>>((const float*)h->buf[h->cur], rho_field(h, h->cur),
                                                                h->c, 0);
  CU(cudaGetLastError());
  h->launches++;
  return LBM_OK;
}

int aa_lid_prep(lbm_cuboid* h) {
  if (!h->d_aa_lid) return LBM_OK;
  const dim3 g(unsigned((h->p.nx + lbm::kBlock - 1) / lbm::kBlock), unsigned(h->nzl), 1);
  if (h->p.precision == LBM_FP64)
    lbm::k_aa_lid_rho<double><<<g, lbm::kBlock, 0, h->stream>>>((const double*)h->buf[0], h->c);
  else
    lbm::k_aa_lid_rho<float><<<g, lbm::kBlock, 0, h->stream>>>((const float*)h->buf[0], h->c);
  CU(cudaGetLastError());
  h->launches++;
  return LBM_OK;
}

int run_init(lbm_cuboid* h, const double* rho, const double* u, long long ustride, int zbeg, int n) {
  return (h->p.precision == LBM_FP64) ? init_kernel<double>(h, rho, u, ustride, zbeg, n)
                                       : init_kernel<float>(h, rho, u, ustride, zbeg, n);
}

int run_macro(lbm_cuboid* h, double* rho, double* u, long long ustride, int zbeg, int n) {
  if (h->p.precision == LBM_FP64)
    lbm::k_macro<double><<<grid_for(h, n), lbm::kBlock, 0, h->stream>>>((const double*)h->buf[h->cur], rho, u,
                                                                        ustride, h->c, zbeg, aa_mode(h));
  else
    lbm::k_macro<float><<<grid_for(h, n), lbm::kBlock, 0, h->stream>>>((const float*)h->buf[h->cur], rho, u,
                                                                       ustride, h->c, zbeg, aa_mode(h));
  CU(cudaGetLastError());
  h->launches++;
  return LBM_OK;
}

// Enqueue one time step from buf[cur] into buf[cur ^ 1] (does not flip cur).
int step_once(lbm_cuboid* h) {
  int rc;
  void* src = h->buf[h->cur];
  void* dst = h->buf[h->cur ^ 1];
  if (h->aa) return launch_aa(h, h->stream);
  if (h->p2p) return p2p_step(h);
  NvtxRange nv(h->ghost ? "lbm step (NCCL halo)" : "lbm step");
  if (!h->ghost) {
    if (h->fd && !h->fd_lag && !h->fd_fused && (rc = launch_density(h, src, 0, h->nzl, 1, h->stream))) return rc;
    return launch_cs(h, src, dst, 0, h->nzl, 1, h->stream);
  }
  if ((rc = wait_halo(h))) return rc;
  if (h->fd && !h->fd_lag) {
    // same-time density (fused: of the two boundary planes only; the fused
    // kernel forms the rest itself), then the boundary planes to the neighbours
    if (h->fd_fused) {
      if ((rc = launch_density(h, src, 0, (h->nzl > 1) ? 2 : 1, std::max(1, h->nzl - 1), h->stream))) return rc;
    } else if ((rc = launch_density(h, src, 0, h->nzl, 1, h->stream))) {
      return rc;
    }
    if ((rc = exchange_rho(h))) return rc;
  }
  // both boundary planes first, in one launch (critical path of the exchange) ...
  const int nb = (h->nzl > 1) ? 2 : 1;
  if ((rc = launch_cs(h, src, dst, 0, nb, std::max(1, h->nzl - 1), h->stream))) return rc;
  if ((rc = exchange(h, h->cur ^ 1))) return rc;
  // ... then the interior, overlapping the NCCL transfer
  return launch_cs(h, src, dst, 1, h->nzl - 2, 1, h->stream);
}

}  // namespace

extern "C" {

void lbm_cuboid_default_params(lbm_cuboid_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->nx = p->ny = p->nz = 32;
  p->r = p->s = 1.0;
  p->cs2 = 0.0;
  p->omega_nu = p->omega_xi = p->omega_1 = p->omega_high = 1.0;
  p->world = 1;
}

int lbm_cuboid_buffer_bytes(const lbm_cuboid_params* p, int64_t* bytes) {
  int rc = validate(p);
  if (rc) return rc;
  if (!bytes) return fail(LBM_EINVAL, "bytes is NULL");
  const int64_t nzl = p->nz / p->world;
  *bytes = int64_t(27) * p->nx * p->ny * (nzl + 2) * (p->precision == LBM_FP64 ? 8 : 4);
  return LBM_OK;
}

int lbm_cuboid_halo_plan(const lbm_cuboid_params* p, int64_t out[8]) {
  int rc = validate(p);
  if (rc) return rc;
  if (!out) return fail(LBM_EINVAL, "out is NULL");
  const HaloPlan hp = make_plan(p);
  out[0] = hp.ghost ? 1 : 0;
  out[1] = hp.peer_up;
  out[2] = hp.peer_down;
  out[3] = hp.count;
  out[4] = hp.send_up;
  out[5] = hp.recv_dn;
  out[6] = hp.send_dn;
  out[7] = hp.recv_up;
  return LBM_OK;
}

int lbm_cuboid_nccl_unique_id(void* out128) {
  if (!out128) return fail(LBM_EINVAL, "out is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return LBM_OK;
}

int lbm_cuboid_create(const lbm_cuboid_params* p, lbm_cuboid_t** out) {
  if (!out) return fail(LBM_EINVAL, "out is NULL");
  *out = nullptr;
  int rc = validate(p);
  if (rc) return rc;
  lbm_cuboid* h = new (std::nothrow) lbm_cuboid();
  if (!h) return fail(LBM_ENOMEM, "host allocation failed");
  h->p = *p;
  h->nzl = p->nz / p->world;
  h->z0 = p->rank * h->nzl;
  h->nxy = int64_t(p->nx) * p->ny;
  h->plane = 27 * h->nxy;
  h->elem = (p->precision == LBM_FP64) ? 8 : 4;
  h->buf_elems = h->plane * (h->nzl + 2);
  const HaloPlan hp = make_plan(p);
  h->ghost = hp.ghost;
  h->peer_up = hp.peer_up;
  h->peer_down = hp.peer_down;
  h->paper_rates = (p->omega_1 == 1.0 && p->omega_high == 1.0);
  h->fd = (p->corrections == LBM_CORR_FULL_FD || p->corrections == LBM_CORR_FULL_FD_LAG);
  h->fd_lag = (p->corrections == LBM_CORR_FULL_FD_LAG);
  // measured at 512^3: with the FD collide bounded to 80
  // registers (round 2) the two-pass path is the faster one in both precisions
  // (fp64 9.9 k vs 9.4 k MLUPS fused; fp32 13.7 k vs 12.0 k)
  h->fd_fused = false;
  if (const char* e = std::getenv("LBM_FD_FUSED")) h->fd_fused = (std::atoi(e) != 0);
  h->aa = (p->streaming == LBM_STREAM_AA);
  // plane shapes of the BASELINE configs 3-5 with a compiled-in specialisation
  h->shape_spec = (p->nx == 512 && p->ny == 512) || (p->nx == 256 && p->ny == 256) ||
                  (p->nx == 512 && p->ny == 256) || (p->nx == 1024 && p->ny == 1024);
  if (const char* e = std::getenv("LBM_SHAPE_SPEC")) h->shape_spec = h->shape_spec && (std::atoi(e) != 0);
  // fp32 storage with an even nx (8-byte aligned node pairs): the x-pair kernel,
  // opt-in (LBM_XPAIR=1): measured no faster than one node per thread
  const char* xp = std::getenv("LBM_XPAIR");
  h->xpair = (p->precision == LBM_FP32_STORAGE) && (p->nx % 2 == 0) && !h->aa && xp && std::atoi(xp) != 0;
  h->p2p = h->ghost && (p->halo == LBM_HALO_P2P);
  // the P2P step forms only the density planes the boundary collision needs
  // (k_density_p2p); its interior must be the fused kernel, which forms its own
  if (h->p2p && h->fd) h->fd_fused = true;
  if (h->fd_lag) h->fd_fused = false;  // one collide-stream launch reads the stored density field
  fill_consts(h);

  auto bail = [&](int code) {
    lbm_cuboid_destroy(h);
    return code;
  };
  if ((rc = set_device(h))) return bail(rc);
  if (p->stream) {
    h->stream = (cudaStream_t)p->stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(fail(LBM_ECUDA, "cudaStreamCreate failed"));
    h->own_stream = true;
  }
  const size_t bytes = size_t(h->buf_elems) * h->elem;
  const int nbuf = h->aa ? 1 : 2;  // AA streaming updates one buffer in place
  if (p->buf_a || p->buf_b) {
    if (!p->buf_a || (!h->aa && !p->buf_b))
      return bail(fail(LBM_EINVAL, "buf_a and buf_b must both be given (buf_a only with AA) or both NULL"));
    h->buf[0] = p->buf_a;
    h->buf[1] = h->aa ? p->buf_a : p->buf_b;
  } else {
    for (int i = 0; i < nbuf; ++i)
      if (cudaMalloc(&h->buf[i], bytes) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(LBM_ENOMEM, "cudaMalloc(%zu) for a population buffer failed", bytes));
      }
    if (h->aa) h->buf[1] = h->buf[0];
    h->own_buf = true;
  }
  // ghost planes must hold finite values even when unused (wall faces)
  for (int i = 0; i < nbuf; ++i)
    if (cudaMemsetAsync(h->buf[i], 0, bytes, h->stream) != cudaSuccess)
      return bail(fail(LBM_ECUDA, "cudaMemsetAsync failed"));
  {
    // TMA-staged kernel (opt-in, LBM_TMA=1: measured slower than the LDG kernel,
    // DESIGN §7): rows whose byte stride is a multiple of 16, 16-byte aligned
    // buffers, at least one full tile per row; AB streaming, not FULL_FD
    const size_t align = uintptr_t(h->buf[0]) | uintptr_t(h->buf[1]);
    const char* tma_env = std::getenv("LBM_TMA");
    h->tma = tma_env && std::atoi(tma_env) != 0 && !h->aa && !h->fd && (size_t(p->nx) * h->elem) % 16 == 0 &&
             p->nx >= lbm::kTmaTx && (align % 16) == 0;
    if (h->tma && (rc = tma_setup(h))) return bail(rc);
    // FULL_FD (same-time density): the TMA-staged fused kernel where it applies
    // -- z faces periodic or ghost planes (it has no z-wall rules; its interior
    // never reads a ghost plane, so the P2P halo may use it too), rows of a
    // 16-byte multiple -- by default when >= 3/4 of its tiles are staged (the
    // rest run the LDG body, slower than the two-pass path);
    // LBM_FD_TMA=0/1 forces it off / on
    const auto zok = [](int fk) { return fk == lbm::FK_WRAP || fk == lbm::FK_GHOST; };
    const bool fdt_ok = h->fd && !h->fd_lag && !h->aa && zok(h->c.face[4]) && zok(h->c.face[5]) &&
                        (size_t(p->nx) * h->elem) % 16 == 0 && (align % 16) == 0;
    bool fdt_on = fdt_ok && fd_tma_staged_fraction(p->nx, p->ny, h->c.face[0] == lbm::FK_WRAP) >= 0.75;
    // an explicit LBM_FD_FUSED selects the LDG fused / two-pass path unless LBM_FD_TMA=1 too
    if (std::getenv("LBM_FD_FUSED")) fdt_on = false;
    if (const char* e = std::getenv("LBM_FD_TMA")) fdt_on = fdt_ok && std::atoi(e) != 0;
    h->fd_tma = fdt_on;
    if (h->fd_tma) {
      h->fd_fused = true;
      if ((rc = fd_tma_setup(h))) return bail(rc);
    }
  }
  if (p->check_every > 0 &&
      (cudaHostAlloc(&h->h_watch, 8 * sizeof(double), cudaHostAllocDefault) != cudaSuccess ||
       cudaEventCreateWithFlags(&h->ev_watch, cudaEventDisableTiming) != cudaSuccess))
    return bail(fail(LBM_ENOMEM, "pinned host memory / event for check_every"));
  // check(): 8 result slots + 8 partials per reduction block
  if (cudaMalloc(&h->d_check, size_t(8) * (1 + lbm::kCheckMaxBlocks) * sizeof(double)) != cudaSuccess)
    return bail(fail(LBM_ENOMEM, "cudaMalloc failed"));
  if (cudaMalloc(&h->d_dbg, 2 * sizeof(unsigned int)) != cudaSuccess ||
      cudaMemsetAsync(h->d_dbg, 0, 2 * sizeof(unsigned int), h->stream) != cudaSuccess)
    return bail(fail(LBM_ENOMEM, "cudaMalloc failed"));
  h->c.dbg_flag = h->d_dbg;
  h->c.sing_flag = h->d_dbg + 1;
  if (h->aa && p->bc[3] == LBM_BC_MOVING_WALL) {
    const size_t lb = size_t(p->nx) * h->nzl * sizeof(double);
    if (cudaMalloc(&h->d_aa_lid, lb) != cudaSuccess || cudaMemsetAsync(h->d_aa_lid, 0, lb, h->stream) != cudaSuccess)
      return bail(fail(LBM_ENOMEM, "cudaMalloc(%zu) for the AA lid densities failed", lb));
    h->c.aa_lid_rho = h->d_aa_lid;
  }
  if (h->fd) {
    const size_t rb = size_t(h->nxy) * (h->nzl + 2) * sizeof(double) * (h->fd_lag ? 2 : 1);
    if (cudaMalloc(&h->d_rho, rb) != cudaSuccess || cudaMemsetAsync(h->d_rho, 0, rb, h->stream) != cudaSuccess)
      return bail(fail(LBM_ENOMEM, "cudaMalloc(%zu) for the density field failed", rb));
  }
  if (h->p2p) {
    // the halo stream at the highest priority: its boundary-plane CTAs are
    // scheduled ahead of the interior CTAs that fill every SM
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (cudaStreamCreateWithPriority(&h->comm_stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_bnd, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_rho, cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(LBM_ECUDA, "stream/event creation failed"));
    PfnWaitValue32 w32 = nullptr;
    if ((rc = driver_fn("cuStreamWaitValue32", &w32))) return bail(rc);
    h->wait32 = reinterpret_cast<void*>(w32);
    if (cudaMalloc(&h->d_sig, 4 * sizeof(unsigned int)) != cudaSuccess ||
        cudaMemsetAsync(h->d_sig, 0, 4 * sizeof(unsigned int), h->stream) != cudaSuccess)
      return bail(fail(LBM_ENOMEM, "cudaMalloc of the P2P flag words failed"));
    if (p->world == 1) {  // periodic z on one GPU: this slab is its own neighbour
      unsigned char blob[LBM_P2P_BLOB_BYTES];
      if ((rc = lbm_cuboid_p2p_export(h, blob)) || (rc = lbm_cuboid_p2p_connect(h, blob, blob))) return bail(rc);
    }
  } else if (h->ghost) {
    if (!p->nccl_uid) return bail(fail(LBM_EINVAL, "nccl_uid is required for the NCCL ghost exchange"));
    // highest priority: the NCCL blocks of the halo are scheduled ahead of the
    // interior collide-stream blocks that otherwise fill every SM's register file
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (cudaStreamCreateWithPriority(&h->comm_stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_bnd, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_rho, cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(LBM_ECUDA, "stream/event creation failed"));
    ncclUniqueId id;
    std::memcpy(&id, p->nccl_uid, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&h->comm, p->world, id, p->rank);
    if (r != ncclSuccess) {
      h->comm = nullptr;
      return bail(fail(LBM_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)));
    }
  }
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return bail(fail(LBM_ECUDA, "initial sync failed"));
  *out = h;
  return LBM_OK;
}

int lbm_cuboid_init_fields_device(lbm_cuboid_t* h, const double* rho, const double* u) {
  if (!h || !rho || !u) return fail(LBM_EINVAL, "NULL argument");
  int rc = set_device(h);
  if (rc) return rc;
  if ((rc = wait_halo(h))) return rc;
  if (h->aa) h->cur = 0;  // AA: the canonical state is written in layout R
  if ((rc = run_init(h, rho, u, (long long)h->nzl * h->nxy, 0, h->nzl))) return rc;
  if ((rc = aa_lid_prep(h)) || (rc = stored_rho(h))) return rc;
  return exchange(h, h->cur);
}

int lbm_cuboid_init_fields(lbm_cuboid_t* h, const double* rho, const double* u) {
  if (!h || !rho || !u) return fail(LBM_EINVAL, "NULL argument");
  int rc = set_device(h);
  if (rc) return rc;
  if ((rc = wait_halo(h))) return rc;
  if (h->aa) h->cur = 0;  // AA: the canonical state is written in layout R
  const int cp = chunk_planes(h, 4);
  if ((rc = ensure_stage(h, size_t(4) * cp * h->nxy * sizeof(double)))) return rc;
  for (int z = 0; z < h->nzl; z += cp) {
    const int n = std::min(cp, h->nzl - z);
    const size_t cnt = size_t(n) * h->nxy;
    double* srho = h->stage;
    double* su = h->stage + cnt;
    CU(cudaMemcpyAsync(srho, rho + size_t(z) * h->nxy, cnt * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpy2DAsync(su, cnt * 8, u + size_t(z) * h->nxy, size_t(h->nzl) * h->nxy * 8, cnt * 8, 3,
                         cudaMemcpyHostToDevice, h->stream));
    if ((rc = run_init(h, srho, su, (long long)cnt, z, n))) return rc;
  }
  if ((rc = aa_lid_prep(h)) || (rc = stored_rho(h))) return rc;
  CU(cudaStreamSynchronize(h->stream));
  return exchange(h, h->cur);
}

namespace {

// the stability reduction of lbm_cuboid_check into h->d_check[0..6] (enqueued)
int enqueue_check(lbm_cuboid* h) {
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->p.device));
  const int64_t nodes = h->nxy * h->nzl;
  const int nb = int(std::max<int64_t>(1, std::min<int64_t>({(nodes + lbm::kCheckThreads - 1) / lbm::kCheckThreads,
                                                            int64_t(8) * sms, int64_t(lbm::kCheckMaxBlocks)})));
  double* partial = h->d_check + 8;
  if (h->p.precision == LBM_FP64)
    lbm::k_check<double><<<nb, lbm::kCheckThreads, 0, h->stream>>>((const double*)h->buf[h->cur], partial, h->c,
                                                                   aa_mode(h));
  else
    lbm::k_check<float><<<nb, lbm::kCheckThreads, 0, h->stream>>>((const float*)h->buf[h->cur], partial, h->c,
                                                                  aa_mode(h));
  CU(cudaGetLastError());
  lbm::k_check_final<<<1, lbm::kCheckThreads, 0, h->stream>>>(partial, nb, h->d_check);
  CU(cudaGetLastError());
  h->launches += 2;
  return LBM_OK;
}

// check_every: result of the pending watch (wait: block until it has landed)
int poll_watch(lbm_cuboid* h, bool wait) {
  if (h->watch_step < 0) return LBM_OK;
  if (wait) {
    CU(cudaEventSynchronize(h->ev_watch));
  } else {
    const cudaError_t e = cudaEventQuery(h->ev_watch);
    if (e == cudaErrorNotReady) return LBM_OK;
    CU(e);
  }
  const int64_t at = h->watch_step;
  h->watch_step = -1;
  if (h->h_watch[6] > 0)
    return fail(LBM_EUNSTABLE, "check_every: %.0f nodes with NaN, rho <= 0 or |u| > 1 at step %lld", h->h_watch[6],
                (long long)at);
  return LBM_OK;
}

int enqueue_watch(lbm_cuboid* h) {
  int rc;
  if ((rc = poll_watch(h, true))) return rc;  // the previous one (check_every steps ago)
  if ((rc = enqueue_check(h))) return rc;
  CU(cudaMemcpyAsync(h->h_watch, h->d_check, 7 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaEventRecord(h->ev_watch, h->stream));
  h->watch_step = h->steps;
  return LBM_OK;
}

int advance(lbm_cuboid* h, int64_t nsteps);

// Device flag words after a synchronisation: the singular strain-rate predicate
// (reading R17; reported once, then cleared) and, in
// LBM_DEBUG_BOUNDS builds, the bounds check.
int poll_flags(lbm_cuboid* h) {
  unsigned int flag[2] = {0, 0};
  CU(cudaMemcpy(flag, h->d_dbg, sizeof(flag), cudaMemcpyDeviceToHost));
#ifdef LBM_DEBUG_BOUNDS
  if (flag[0]) return fail(LBM_ECUDA, "bounds check: a collide-stream kernel accessed outside its buffer");
#endif
  if (flag[1]) {
    CU(cudaMemset(h->d_dbg + 1, 0, sizeof(unsigned int)));
    return fail(LBM_ESINGULAR, "singular strain-rate system at a node (|det| or |C_sy|, |C_sz| < 1e-12 rho cs2, "
                "S:L207) in the steps before step %lld", (long long)h->steps);
  }
  return LBM_OK;
}

}  // namespace

int lbm_cuboid_step(lbm_cuboid_t* h, int64_t nsteps) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  NvtxRange nv("lbm_cuboid_step");
  if (nsteps < 0) return fail(LBM_EINVAL, "nsteps must be >= 0");
  int rc = set_device(h);
  if (rc) return rc;
  if ((rc = poll_watch(h, false))) return rc;
  const int64_t K = h->p.check_every;
  if (K <= 0) return advance(h, nsteps);
  while (nsteps > 0) {
    const int64_t n = std::min<int64_t>(nsteps, K - h->steps % K);
    if ((rc = advance(h, n))) return rc;
    nsteps -= n;
    if (h->steps % K == 0 && (rc = enqueue_watch(h))) return rc;
  }
  return LBM_OK;
}

namespace {

int advance(lbm_cuboid* h, int64_t nsteps) {
  int rc;
  if (use_persistent(h)) return launch_persistent(h, nsteps);
  if (use_graphs(h)) {
    while (nsteps >= kGraphSteps) {
      if (!h->gexec[h->cur] && (rc = capture_graph(h, h->cur))) return rc;
      CU(cudaGraphLaunch(h->gexec[h->cur], h->stream));
      h->launches += kGraphSteps;
      h->cs_launches += kGraphSteps;
      h->steps += kGraphSteps;
      nsteps -= kGraphSteps;  // kGraphSteps is even: h->cur is unchanged
    }
  }
  for (int64_t t = 0; t < nsteps; ++t) {
    if ((rc = step_once(h))) return rc;
    h->cur ^= 1;
    h->steps++;
  }
  return LBM_OK;
}

}  // namespace

int lbm_cuboid_sync(lbm_cuboid_t* h) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  int rc = set_device(h);
  if (rc) return rc;
  if ((rc = wait_halo(h))) return rc;
  CU(cudaStreamSynchronize(h->stream));
  if (h->comm_stream) CU(cudaStreamSynchronize(h->comm_stream));
  if ((rc = poll_flags(h))) return rc;
  return poll_watch(h, true);
}

int lbm_cuboid_get_macroscopic_device(lbm_cuboid_t* h, double* rho, double* u) {
  if (!h || !rho || !u) return fail(LBM_EINVAL, "NULL argument");
  int rc = set_device(h);
  if (rc) return rc;
  return run_macro(h, rho, u, (long long)h->nzl * h->nxy, 0, h->nzl);
}

int lbm_cuboid_get_macroscopic(lbm_cuboid_t* h, double* rho, double* u) {
  if (!h || !rho || !u) return fail(LBM_EINVAL, "NULL argument");
  int rc = set_device(h);
  if (rc) return rc;
  const int cp = chunk_planes(h, 4);
  if ((rc = ensure_stage(h, size_t(4) * cp * h->nxy * sizeof(double)))) return rc;
  for (int z = 0; z < h->nzl; z += cp) {
    const int n = std::min(cp, h->nzl - z);
    const size_t cnt = size_t(n) * h->nxy;
    double* srho = h->stage;
    double* su = h->stage + cnt;
    if ((rc = run_macro(h, srho, su, (long long)cnt, z, n))) return rc;
    CU(cudaMemcpyAsync(rho + size_t(z) * h->nxy, srho, cnt * 8, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaMemcpy2DAsync(u + size_t(z) * h->nxy, size_t(h->nzl) * h->nxy * 8, su, cnt * 8, cnt * 8, 3,
                         cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
  }
  return LBM_OK;
}

int lbm_cuboid_get_populations_planes(lbm_cuboid_t* h, int32_t z_begin, int32_t n_planes, double* f) {
  if (!h || !f) return fail(LBM_EINVAL, "NULL argument");
  if (z_begin < 0 || n_planes < 0 || z_begin + n_planes > h->nzl)
    return fail(LBM_EINVAL, "planes [%d, %d) outside the local slab [0, %d)", z_begin, z_begin + n_planes, h->nzl);
  int rc = set_device(h);
  if (rc) return rc;
  if (n_planes == 0) return LBM_OK;
  const int cp = std::min(chunk_planes(h, 27), int(n_planes));
  if ((rc = ensure_stage(h, size_t(27) * cp * h->nxy * sizeof(double)))) return rc;
  for (int z = 0; z < n_planes; z += cp) {
    const int n = std::min(cp, n_planes - z);
    const size_t cnt = size_t(n) * h->nxy;
    if (h->p.precision == LBM_FP64)
      lbm::k_pack<double><<<grid_for(h, n), lbm::kBlock, 0, h->stream>>>((const double*)h->buf[h->cur], h->stage, n,
                                                                         h->c, z_begin + z, aa_mode(h));
    else
      lbm::k_pack<float><<<grid_for(h, n), lbm::kBlock, 0, h->stream>>>((const float*)h->buf[h->cur], h->stage, n,
                                                                        h->c, z_begin + z, aa_mode(h));
    CU(cudaGetLastError());
    h->launches++;
    CU(cudaMemcpy2DAsync(f + size_t(z) * h->nxy, size_t(n_planes) * h->nxy * 8, h->stage, cnt * 8, cnt * 8, 27,
                         cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
  }
  return LBM_OK;
}

int lbm_cuboid_get_populations(lbm_cuboid_t* h, double* f) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  return lbm_cuboid_get_populations_planes(h, 0, h->nzl, f);
}

int lbm_cuboid_set_populations(lbm_cuboid_t* h, const double* f) {
  if (!h || !f) return fail(LBM_EINVAL, "NULL argument");
  int rc = set_device(h);
  if (rc) return rc;
  if ((rc = wait_halo(h))) return rc;
  if (h->aa) h->cur = 0;  // AA: the canonical state is written in layout R
  const int cp = chunk_planes(h, 27);
  if ((rc = ensure_stage(h, size_t(27) * cp * h->nxy * sizeof(double)))) return rc;
  for (int z = 0; z < h->nzl; z += cp) {
    const int n = std::min(cp, h->nzl - z);
    const size_t cnt = size_t(n) * h->nxy;
    CU(cudaMemcpy2DAsync(h->stage, cnt * 8, f + size_t(z) * h->nxy, size_t(h->nzl) * h->nxy * 8, cnt * 8, 27,
                         cudaMemcpyHostToDevice, h->stream));
    if (h->p.precision == LBM_FP64)
      lbm::k_unpack<double><<<grid_for(h, n), lbm::kBlock, 0, h->stream>>>(h->stage, (double*)h->buf[h->cur], n,
                                                                           h->c, z, h->aa ? 1 : 0);
    else
      lbm::k_unpack<float><<<grid_for(h, n), lbm::kBlock, 0, h->stream>>>(h->stage, (float*)h->buf[h->cur], n,
                                                                          h->c, z, h->aa ? 1 : 0);
    CU(cudaGetLastError());
    h->launches++;
    CU(cudaStreamSynchronize(h->stream));
  }
  if ((rc = aa_lid_prep(h)) || (rc = stored_rho(h))) return rc;
  return exchange(h, h->cur);
}

int lbm_cuboid_check(lbm_cuboid_t* h, double out[7]) {
  if (!h || !out) return fail(LBM_EINVAL, "NULL argument");
  int rc = set_device(h);
  if (rc) return rc;
  if ((rc = enqueue_check(h))) return rc;
  CU(cudaMemcpyAsync(out, h->d_check, 7 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  if (out[6] > 0) return fail(LBM_EUNSTABLE, "%.0f nodes with NaN, rho <= 0 or |u| > 1 after %lld steps", out[6],
                              (long long)h->steps);
  return poll_flags(h);
}

int lbm_cuboid_set_force(lbm_cuboid_t* h, const double force[3]) {
  if (!h || !force) return fail(LBM_EINVAL, "NULL argument");
  for (int d = 0; d < 3; ++d) {
    if (!std::isfinite(force[d])) return fail(LBM_EINVAL, "force must be finite");
    h->p.force[d] = force[d];
    h->c.F[d] = force[d];
  }
  drop_graphs(h);  // the parameter block is baked into captured launches
  return LBM_OK;
}

int lbm_cuboid_info(const lbm_cuboid_t* h, int64_t out[8]) {
  if (!h || !out) return fail(LBM_EINVAL, "NULL argument");
  out[0] = h->launches;
  out[1] = h->cs_launches;
  out[2] = h->steps;
  out[3] = int64_t(2 * 27) * int64_t(h->elem);
  out[4] = h->nxy * h->nzl;
  out[5] = h->buf_elems * int64_t(h->elem);
  out[6] = h->ghost ? (h->p2p ? 2 : 1) : 0;
  out[7] = (h->paper_rates && h->p.model == LBM_MODEL_CM) ? 1 : 0;
  return LBM_OK;
}

void* lbm_cuboid_stream(const lbm_cuboid_t* h) { return h ? (void*)h->stream : nullptr; }

const char* lbm_cuboid_kernel_name(const lbm_cuboid_t* h) {
  if (!h) return "";
  const char* t = (h->p.precision == LBM_FP64) ? "double" : "float";
  std::string k;
  if (h->aa) {
    k = (h->shape_spec && h->paper_rates && h->p.model == LBM_MODEL_CM)
            ? std::string("k_aa_shape<") + t + "," + std::to_string(h->p.nx) + "," + std::to_string(h->p.ny) + ">"
            : std::string("k_aa<") + t + ">";
  } else if (h->fd && h->fd_fused) {  // (the P2P interior launch too)
    k = std::string(h->fd_tma ? "k_collide_stream_fd_tma<" : "k_collide_stream_fd<") + t + ">";
  } else if (h->tma && !h->fd) {
    k = std::string("k_collide_stream_tma<") + t + ">";
  } else if (h->xpair && h->p.precision != LBM_FP64 && !h->fd) {
    k = "k_collide_stream_xpair<float>";
  } else if (h->shape_spec && h->paper_rates && h->p.model == LBM_MODEL_CM) {
    k = std::string("k_collide_stream_paper_shape<") + t + "," + std::to_string(h->p.nx) + "," +
        std::to_string(h->p.ny) + ">";
  } else {
    k = (h->p.model == LBM_MODEL_RM) ? "k_collide_stream_raw<" : (h->paper_rates ? "k_collide_stream_paper<"
                                                                                   : "k_collide_stream<");
    k = k + t + ">";
  }
  if (h->fd && !h->fd_lag && !h->fd_fused) k += " + k_density";
  const_cast<lbm_cuboid_t*>(h)->kname = k;
  return h->kname.c_str();
}

int lbm_cuboid_comm_ranks(const lbm_cuboid_t* h, int32_t out[2]) {
  if (!h || !out) return fail(LBM_EINVAL, "NULL argument");
  out[0] = out[1] = -1;
  if (!h->comm) return LBM_OK;
  int n = 0, r = 0;
  NC(ncclCommCount(h->comm, &n));
  NC(ncclCommUserRank(h->comm, &r));
  out[0] = n;
  out[1] = r;
  return LBM_OK;
}

static void clear_timing(lbm_cuboid_t* h) {
  for (auto& e : h->ev_t) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  h->ev_t.clear();
  h->ev_t_nodes.clear();
}

int lbm_cuboid_timing(lbm_cuboid_t* h, int enable) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  int rc = set_device(h);
  if (rc) return rc;
  CU(cudaStreamSynchronize(h->stream));
  clear_timing(h);
  h->timing = (enable != 0);
  return LBM_OK;
}

int lbm_cuboid_timing_read(lbm_cuboid_t* h, double out[3]) {
  if (!h || !out) return fail(LBM_EINVAL, "NULL argument");
  int rc = set_device(h);
  if (rc) return rc;
  CU(cudaStreamSynchronize(h->stream));
  double ms = 0.0;
  int64_t nodes = 0;
  for (size_t i = 0; i < h->ev_t.size(); ++i) {
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, h->ev_t[i].first, h->ev_t[i].second));
    ms += t;
    nodes += h->ev_t_nodes[i];
  }
  out[0] = double(h->ev_t.size());
  out[1] = ms;
  out[2] = double(nodes);
  return LBM_OK;
}

static void clear_trace(lbm_cuboid_t* h) {
  for (auto& r : h->trace) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  h->trace.clear();
  if (h->trace_base) {
    cudaEventDestroy(h->trace_base);
    h->trace_base = nullptr;
  }
}

int lbm_cuboid_trace(lbm_cuboid_t* h, int enable) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  int rc = set_device(h);
  if (rc) return rc;
  CU(cudaStreamSynchronize(h->stream));
  if (h->comm_stream) CU(cudaStreamSynchronize(h->comm_stream));
  clear_trace(h);
  h->tracing = (enable != 0);
  if (h->tracing) {
    drop_graphs(h);  // launches inside replayed graphs carry no events
    CU(cudaEventCreate(&h->trace_base));
    CU(cudaEventRecord(h->trace_base, h->stream));
  }
  return LBM_OK;
}

int lbm_cuboid_trace_read(lbm_cuboid_t* h, double* out, int32_t max_rows, int32_t* rows) {
  if (!h || !rows || (max_rows > 0 && !out)) return fail(LBM_EINVAL, "NULL argument");
  int rc = set_device(h);
  if (rc) return rc;
  CU(cudaStreamSynchronize(h->stream));
  if (h->comm_stream) CU(cudaStreamSynchronize(h->comm_stream));
  *rows = int32_t(h->trace.size());
  const int n = std::min<int>(max_rows, int(h->trace.size()));
  for (int i = 0; i < n; ++i) {
    const auto& r = h->trace[i];
    float ta = 0.f, tb = 0.f;
    CU(cudaEventElapsedTime(&ta, h->trace_base, r.a));
    CU(cudaEventElapsedTime(&tb, h->trace_base, r.b));
    double* o = out + 6 * i;
    o[0] = r.kind;
    o[1] = r.stream;
    o[2] = r.zbeg;
    o[3] = r.nplanes;
    o[4] = ta;
    o[5] = tb;
  }
  return LBM_OK;
}

int lbm_cuboid_p2p_export(const lbm_cuboid_t* h, void* blob) {
  if (!h || !blob) return fail(LBM_EINVAL, "NULL argument");
  if (!h->p2p) return fail(LBM_EINVAL, "the handle does not use the P2P halo (LBM_HALO_P2P with ghost planes)");
  int rc = set_device(h);
  if (rc) return rc;
  PfnAddressRange range = nullptr;
  if ((rc = driver_fn("cuMemGetAddressRange", &range))) return rc;
  P2PBlob b;
  std::memset(&b, 0, sizeof(b));
  std::memcpy(b.magic, kBlobMagic, sizeof(b.magic));
  b.pid = int32_t(getpid());
  b.device = h->p.device;
  b.rank = h->p.rank;
  b.world = h->p.world;
  b.precision = h->p.precision;
  b.nx = h->p.nx;
  b.ny = h->p.ny;
  b.nzl = h->nzl;
  b.buf_elems = h->buf_elems;
  b.ipc_ok = 1;
  void* const ptrs[4] = {h->buf[0], h->buf[1], h->d_sig, h->d_rho};
  for (int i = 0; i < 4; ++i) {
    if (!ptrs[i]) continue;  // no density field (not FULL_FD)
    b.ptr[i] = (uint64_t)(uintptr_t)ptrs[i];
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)(uintptr_t)ptrs[i]) != CUDA_SUCCESS)
      return fail(LBM_ECUDA, "cuMemGetAddressRange failed for a P2P buffer");
    b.off[i] = b.ptr[i] - (uint64_t)base;
    // IPC handles serve other processes only; a failure (e.g. memory from a
    // virtual-memory pool) still allows same-process peers
    if (cudaIpcGetMemHandle(&b.ipc[i], (void*)(uintptr_t)base) != cudaSuccess) {
      cudaGetLastError();
      b.ipc_ok = 0;
    }
  }
  std::memset(blob, 0, LBM_P2P_BLOB_BYTES);
  std::memcpy(blob, &b, sizeof(b));
  return LBM_OK;
}

int lbm_cuboid_p2p_connect(lbm_cuboid_t* h, const void* blob_down, const void* blob_up) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!h->p2p) return fail(LBM_EINVAL, "the handle does not use the P2P halo (LBM_HALO_P2P with ghost planes)");
  if (h->p2p_ready) return fail(LBM_EINVAL, "lbm_cuboid_p2p_connect: already connected");
  int rc = set_device(h);
  if (rc) return rc;
  const void* blobs[2] = {blob_down, blob_up};
  const int peers[2] = {h->peer_down, h->peer_up};
  P2PBlob b[2];
  for (int side = 0; side < 2; ++side) {
    if (peers[side] < 0) continue;  // no neighbour on this side: blob ignored
    if (!blobs[side]) return fail(LBM_EINVAL, "the %s neighbour (rank %d) needs a blob", side ? "up" : "down",
                                  peers[side]);
    std::memcpy(&b[side], blobs[side], sizeof(P2PBlob));
    const P2PBlob& x = b[side];
    if (std::memcmp(x.magic, kBlobMagic, sizeof(kBlobMagic)) != 0)
      return fail(LBM_EINVAL, "not a lbm_cuboid P2P blob");
    if (x.rank != peers[side] || x.world != h->p.world)
      return fail(LBM_EINVAL, "blob of rank %d/%d given for the %s neighbour, expected rank %d/%d", x.rank, x.world,
                  side ? "up" : "down", peers[side], h->p.world);
    if (x.nx != h->p.nx || x.ny != h->p.ny || x.nzl != h->nzl || x.precision != h->p.precision ||
        x.buf_elems != h->buf_elems)
      return fail(LBM_EINVAL, "neighbour blob has another geometry or precision");
    if ((x.ptr[3] != 0) != h->fd) return fail(LBM_EINVAL, "neighbour blob has another correction mode");
  }
  // map (a rank that is both neighbours is mapped once)
  void* m[2][4] = {{nullptr, nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr, nullptr}};
  const pid_t me = getpid();
  for (int side = 0; side < 2; ++side) {
    if (peers[side] < 0) continue;
    const P2PBlob& x = b[side];
    if (side == 1 && peers[0] >= 0 && b[0].pid == x.pid && b[0].ptr[0] == x.ptr[0] && b[0].ptr[2] == x.ptr[2]) {
      for (int i = 0; i < 4; ++i) m[1][i] = m[0][i];
      continue;
    }
    if (x.pid == int32_t(me)) {  // same process: direct pointers (peer access if another device)
      if (x.device != h->p.device) {
        int ok = 0;
        CU(cudaDeviceCanAccessPeer(&ok, h->p.device, x.device));
        if (!ok) return fail(LBM_ECUDA, "device %d cannot access peer device %d", h->p.device, x.device);
        cudaError_t e = cudaDeviceEnablePeerAccess(x.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CU(e);
        cudaGetLastError();
      }
      for (int i = 0; i < 4; ++i) m[side][i] = (void*)(uintptr_t)x.ptr[i];
    } else {
      if (!x.ipc_ok) return fail(LBM_EINVAL, "the neighbour's buffers cannot be shared between processes (no IPC)");
      for (int i = 0; i < 4; ++i) {
        if (!x.ptr[i]) continue;
        void* base = nullptr;
        CU(cudaIpcOpenMemHandle(&base, x.ipc[i], cudaIpcMemLazyEnablePeerAccess));
        h->ipc_open.push_back(base);
        m[side][i] = (char*)base + x.off[i];
      }
    }
  }
  for (int i = 0; i < 2; ++i) {
    h->peer_buf_dn[i] = m[0][i];
    h->peer_buf_up[i] = m[1][i];
  }
  // flag words: [0] is written by the slab below, [1] by the slab above
  h->peer_flag_dn = peers[0] >= 0 ? (unsigned int*)m[0][2] + 1 : nullptr;
  h->peer_rho_dn = (double*)m[0][3];
  h->peer_rho_up = (double*)m[1][3];
  h->peer_flag_up = peers[1] >= 0 ? (unsigned int*)m[1][2] + 0 : nullptr;
  h->p2p_ready = true;
  return LBM_OK;
}

int lbm_cuboid_destroy(lbm_cuboid_t* h) {
  if (!h) return LBM_OK;
  cudaSetDevice(h->p.device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->comm_stream) cudaStreamSynchronize(h->comm_stream);
  if (h->p2p_ready) {
    // no neighbour store into this slab may be in flight when it is freed: wait
    // (host side, bounded) until both neighbours have published this epoch
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      unsigned int sig[2] = {0, 0};
      if (cudaMemcpy(sig, h->d_sig, sizeof(sig), cudaMemcpyDeviceToHost) != cudaSuccess) break;
      const bool dn = h->peer_down < 0 || int32_t(sig[0] - h->epoch) >= 0;
      const bool up = h->peer_up < 0 || int32_t(sig[1] - h->epoch) >= 0;
      if (dn && up) break;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30)) break;
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    for (void* m : h->ipc_open) cudaIpcCloseMemHandle(m);
  }
  if (h->d_sig) cudaFree(h->d_sig);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->comm) ncclCommDestroy(h->comm);
  if (h->ev_bnd) cudaEventDestroy(h->ev_bnd);
  if (h->ev_halo) cudaEventDestroy(h->ev_halo);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  if (h->own_buf)
    for (int i = 0; i < (h->aa ? 1 : 2); ++i)
      if (h->buf[i]) cudaFree(h->buf[i]);
  if (h->stage) cudaFree(h->stage);
  if (h->d_check) cudaFree(h->d_check);
  if (h->h_watch) cudaFreeHost(h->h_watch);
  if (h->ev_watch) cudaEventDestroy(h->ev_watch);
  if (h->d_dbg) cudaFree(h->d_dbg);
  if (h->d_aa_lid) cudaFree(h->d_aa_lid);
  if (h->d_rho) cudaFree(h->d_rho);
  if (h->ev_rho) cudaEventDestroy(h->ev_rho);
  clear_timing(h);
  clear_trace(h);
  drop_graphs(h);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return LBM_OK;
}

const char* lbm_cuboid_last_error(void) { return g_err.c_str(); }

}  // extern "C"
