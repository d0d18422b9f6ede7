/*
 * lbm_cuboid.h -- C ABI of the B200 3D cuboid central-moment LBM (3DCCM-LBM)
 * hot path (arXiv 2107.14774, Yahia, Schupbach & Premnath).
 *
 * "P:Lnnn" cites /root/reference/PAPER.md line nnn.
 *
 * The library advances the D3Q27 cuboid-lattice central-moment scheme
 *   m^c = F S P f;  m~^c = m^c + B^-1 {Lambda (B m^{c,eq} - B m^c) + (I - Lambda/2) B Phi^c};
 *   f~  = P^-1 S^-1 F^-1 m~^c;  f(x, t+1) = f~(x - e, t)
 * (Eq. LBEcentralmomentcuboidlattice; step list P:L687-742; collision
 * App D) with halfway bounce-back and the momentum-augmented
 * moving wall of Eq. 69, on one GPU or on a z-slab decomposition
 * over several GPUs (one process per GPU; ghost-plane halo exchanged with NCCL,
 * or stored by the boundary-plane kernel itself into the neighbours' ghost planes
 * over NVLink peer memory, LBM_HALO_P2P).
 *
 * Conventions
 *  - Lattice units: dx = dt = 1, dy = r, dz = s.
 *  - Grid nodes (x, y, z), x fastest.  Host scalar fields are [nz_l][ny][nx],
 *    host vector fields [3][nz_l][ny][nx], host populations [27][nz_l][ny][nx]
 *    in the paper's direction order of Eqs. 1a-1c.  nz_l is the
 *    number of z-planes owned by this rank (nz / world).
 *  - Canonical state = post-collision populations f~(x, t_n) stored at their
 *    node (the pull scheme's natural state).  rho and u reported for that
 *    state are rho = sum f~, u = (sum f~ e - F/2)/rho (the collision adds F to
 *    the first raw moments).
 *  - Every function returns 0 (LBM_OK) or a negative lbm_status; the message
 *    of the last failure on the calling thread is lbm_cuboid_last_error().
 *  - A handle is thread-compatible, not thread-safe.
 *  - Host pointers are caller-owned and only read/written during the call.
 *    Device buffers passed in lbm_cuboid_params are caller-owned (e.g. torch
 *    tensors) and must outlive the handle.
 */
#ifndef LBM_CUBOID_H
#define LBM_CUBOID_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBM_CUBOID_ABI_VERSION 2

typedef enum {
  LBM_OK = 0,
  LBM_EINVAL = -1,    /* invalid argument / parameter combination */
  LBM_ENOMEM = -2,    /* device or host allocation failed */
  LBM_ECUDA = -3,     /* CUDA runtime error (message has the CUDA string) */
  LBM_ENCCL = -4,     /* NCCL error */
  LBM_EUNSTABLE = -5, /* NaN, rho <= 0 or |u| > 1 seen by lbm_cuboid_check() */
  LBM_ESINGULAR = -6, /* singular strain-rate system of the corrections (determinant of
                         the 3x3 system of P:L1199-1203, Eq. 65): at create for the fluid at rest, or
                         in flight at some node, where |D| or the back-substitution denominators
                         |C_sy|, |C_sz| fell below 1e-12 rho cs2 (the C's grow the -3u^2/2 terms of
                         P:L1194-1196); reported by lbm_cuboid_sync() and lbm_cuboid_check() after
                         the step that saw it (DESIGN reading R17) */
  LBM_ENOTSUP = -7    /* unsupported parameter combination (e.g. AA streaming on several GPUs) */
} lbm_status;

/* Face boundary types.  Faces are ordered -x, +x, -y, +y, -z, +z.  Opposite
 * faces are both periodic or both non-periodic. */
typedef enum {
  LBM_BC_PERIODIC = 0,
  LBM_BC_BOUNCE_BACK = 1,  /* halfway bounce-back f_q(x_f,t+1) = f~_qbar(x_f,t) (U = 0) */
  LBM_BC_MOVING_WALL = 2,  /* Eq. 69: +y face only, wall velocity (wall_u, 0, 0) */
  LBM_BC_FREE_SLIP = 3     /* halfway specular reflection; NOT in the paper (BASELINE config 4) */
} lbm_bc;

/* Second-order equilibrium corrections (Eqs. 38-40). */
typedef enum {
  LBM_CORR_FULL_LOCAL = 0, /* theta with the 3u^2 aliasing terms; local strain rates; lambda = e_rho = 0 */
  LBM_CORR_LOW_MACH = 1,   /* 3u^2 terms dropped (in theta and in the strain-rate solve) */
  LBM_CORR_OFF = 2,        /* no corrections (ablation) */
  LBM_CORR_FULL_FD = 3,    /* FULL_LOCAL plus the density-gradient terms lambda and e_rho,
                              with the isotropic lattice gradient of a same-time density field (P:L494,
                              DESIGN reading R16): the density of the pulled populations of every
                              neighbour (fused 2.5D kernel for fp64, density pass + collide for fp32) */
  LBM_CORR_FULL_FD_LAG = 4 /* the same terms with the gradient of the STORED state's density, one time
                              level earlier (reading R16b: the paper does not fix the time level of
                              P:L1181); the collision writes each node's density into a second field
                              that the next step's gradient reads: 2*27*sizeof(real) + 16 B/node;
                              pinned by the same moving-frame acoustic attenuation as FULL_FD */
} lbm_corr;

typedef enum {
  LBM_FP64 = 0,        /* fp64 populations, fp64 arithmetic */
  LBM_FP32_STORAGE = 1 /* fp32 populations in HBM, fp64 arithmetic in registers */
} lbm_prec;

/* Collision model. */
typedef enum {
  LBM_MODEL_CM = 0, /* 3DCCM-LBM: central moments (Eq. LBEcentralmomentcuboidlattice) */
  LBM_MODEL_RM = 1  /* 3DCRM-LBM: raw moments, same corrections (P:L642-648, L744(ii), L1011) */
} lbm_model;

/* Population storage / streaming pattern. */
typedef enum {
  LBM_STREAM_AB = 0, /* two buffers: pull from one, store into the other (default) */
  LBM_STREAM_AA = 1  /* one buffer updated in place, alternating an "odd" step (pull from reversed
                        slots, collide, push) and an "even" step (collide in place, store reversed):
                        half the memory, same 2*27*sizeof(real) bytes per node update; single GPU,
                        not with LBM_CORR_FULL_FD / LBM_CORR_FULL_FD_LAG */
} lbm_streaming;

typedef enum {
  LBM_HALO_AUTO = 0, /* 1 GPU + periodic z: wrap inside the kernel; else NCCL ghost planes */
  LBM_HALO_NCCL = 1, /* always exchange ghost planes with NCCL (also world == 1: send to self) */
  LBM_HALO_P2P = 2   /* fused halo: the boundary-plane collide-stream kernel stores the outgoing
                        directions straight into the neighbours' ghost planes (peer memory over
                        NVLink; CUDA IPC between processes, direct pointers within one process)
                        and publishes a per-step epoch flag; the neighbour's stream waits on the
                        flag (no NCCL, no spinning kernel).  The boundary planes run on a second,
                        high-priority stream concurrently with the interior.  Requires
                        lbm_cuboid_p2p_connect() when world > 1; not with AA streaming.  With
                        LBM_CORR_FULL_FD a density kernel first pushes the boundary planes'
                        density into the neighbours' density ghost planes (a second epoch). */
} lbm_halo;

/* Size of the opaque blob lbm_cuboid_p2p_export() writes. */
#define LBM_P2P_BLOB_BYTES 512

typedef struct {
  int32_t nx, ny, nz;          /* GLOBAL node counts (>= 1); nz % world == 0 */
  double r, s;                 /* aspect ratios r = dy/dx, s = dz/dx; > 0 */
  double cs2;                  /* speed of sound squared; <= 0 -> min(1, r^2, s^2)/3 (DESIGN R3);
                                  must satisfy 0 < cs2 < min(1, r^2, s^2) */
  double omega_nu, omega_xi;   /* shear / bulk rates in (0, 2): nu = cs2 (1/omega_nu - 1/2),
                                  xi = (2 cs2/3)(1/omega_xi - 1/2) (Eq. 53) */
  double omega_1, omega_high;  /* first-order and all higher-order rates in (0, 2]; paper: 1 */
  double force[3];             /* constant body force F, lattice units */
  int32_t bc[6];               /* lbm_bc per face -x,+x,-y,+y,-z,+z */
  double wall_u;               /* moving-wall speed U along +x (used when bc[3] == LBM_BC_MOVING_WALL) */
  int32_t corrections;         /* lbm_corr */
  int32_t precision;           /* lbm_prec */
  int32_t rank, world;         /* z-slab decomposition: rank owns global planes
                                  [rank*nz/world, (rank+1)*nz/world) */
  int32_t device;              /* CUDA device ordinal of this rank */
  int32_t halo;                /* lbm_halo */
  int32_t graphs;              /* launch mode of step(n): 0 auto (replay captured 32-step CUDA graphs when
                                  the slab has < 4M nodes and no ghost exchange), 1 one stream launch per
                                  step, 2 always graphs (when no ghost exchange), 3 persistent cooperative
                                  kernel running up to 1024 steps per launch with a grid-wide barrier
                                  between steps (single GPU, no ghost exchange, not AA) */
  int32_t model;               /* lbm_model */
  int32_t streaming;           /* lbm_streaming; with LBM_STREAM_AA only buf_a is used */
  const void *nccl_uid;        /* 128-byte ncclUniqueId from lbm_cuboid_nccl_unique_id() on rank 0,
                                  broadcast by the caller; required iff NCCL ghost exchange is used */
  void *stream;                /* cudaStream_t for all compute work; NULL -> library-owned stream */
  void *buf_a, *buf_b;         /* optional caller-owned device buffers of lbm_cuboid_buffer_bytes()
                                  bytes each (e.g. torch tensors); NULL -> library cudaMalloc */
  int32_t check_every;         /* > 0: every check_every steps step() enqueues the stability check of
                                  lbm_cuboid_check (NaN, rho <= 0, |u| > 1) without blocking; a
                                  failure is returned as LBM_EUNSTABLE, with the step, by a later
                                  step() or by lbm_cuboid_sync().  0: off (default) */
} lbm_cuboid_params;

typedef struct lbm_cuboid lbm_cuboid_t;

/* Fill *p with defaults: 32^3, r = s = 1, cs2 auto, omegas 1, periodic, fp64,
 * rank 0 of 1, device 0, AUTO halo, library-owned stream and buffers. */
void lbm_cuboid_default_params(lbm_cuboid_params *p);

/* Bytes of ONE population buffer for these parameters:
 * 27 * nx * ny * (nz/world + 2 ghost planes) * sizeof(real). */
int lbm_cuboid_buffer_bytes(const lbm_cuboid_params *p, int64_t *bytes);

/* Host-only halo plan of this rank (no GPU needed), element offsets into one
 * population buffer (layout: DESIGN.md "Data layout"):
 * out[0] = 1 if ghost planes are exchanged (world > 1, or periodic z with
 *          LBM_HALO_NCCL / LBM_HALO_P2P),
 * out[1] = peer above (-1 none), out[2] = peer below (-1 none),
 * out[3] = elements per message (9 * nx * ny),
 * out[4] = send-up offset (top plane, the 9 directions with e_z = +1),
 * out[5] = recv-down offset (lower ghost plane, e_z = +1 directions),
 * out[6] = send-down offset (bottom plane, e_z = -1 directions),
 * out[7] = recv-up offset (upper ghost plane, e_z = -1 directions).
 * NCCL: every rank issues, inside one NCCL group: send(up), recv(down),
 * send(down), recv(up), skipping absent peers.  P2P: the send regions are
 * stored by the boundary kernel at the neighbours' recv offsets. */
int lbm_cuboid_halo_plan(const lbm_cuboid_params *p, int64_t out[8]);

/* LBM_HALO_P2P wiring.  export: write this handle's LBM_P2P_BLOB_BYTES-byte
 * descriptor (IPC handles and addresses of both population buffers, of the
 * flag words and, with LBM_CORR_FULL_FD, of the density field; pid; geometry)
 * into blob.  connect: map the neighbours' buffers
 * (blob_down = the rank below, blob_up = the rank above, as given by
 * lbm_cuboid_halo_plan; NULL where there is no neighbour; the same blob twice
 * when both neighbours are one rank).  Every rank calls connect once, after
 * all ranks have created their handles and before init_fields / step; with
 * world == 1 create() connects the handle to itself.  Errors: LBM_EINVAL for
 * a blob of another geometry/precision or a missing neighbour, LBM_ECUDA if
 * the peer mapping fails.  Handles of one process (e.g. several ranks' slabs
 * driven from one thread) are connected with direct pointers.  The neighbours
 * must stay alive until this handle is destroyed (destroy waits, up to 30 s,
 * for the neighbours' last epoch so no peer store is in flight).  Ranks must
 * step concurrently (one process or thread per rank): a step waits for the
 * neighbours' previous step, and with LBM_CORR_FULL_FD also for their
 * boundary-plane density of the same step. */
int lbm_cuboid_p2p_export(const lbm_cuboid_t *h, void *blob);
int lbm_cuboid_p2p_connect(lbm_cuboid_t *h, const void *blob_down, const void *blob_up);

/* Write a fresh 128-byte ncclUniqueId into out (call on rank 0 only). */
int lbm_cuboid_nccl_unique_id(void *out128);

/* Validate p (errors: LBM_EINVAL with a message naming the field;
 * LBM_ESINGULAR for a strain-rate system of the corrections that is singular
 * at rest;
 * LBM_ENOTSUP for unsupported mode combinations), bind the
 * device, allocate/bind buffers, upload the parameter block and, if needed,
 * create the NCCL communicator (collective over all ranks). */
int lbm_cuboid_create(const lbm_cuboid_params *p, lbm_cuboid_t **out);

/* Initialise the stored state with f~ = f^eq(rho, u + F/(2 rho)) (DESIGN R8)
 * from HOST fields rho [nz_l][ny][nx] and u [3][nz_l][ny][nx] (fp64).  Fills
 * the halo ghost planes: with ghost-plane exchange (world > 1, or a non-AUTO
 * halo) this is collective -- every rank calls it, like step().  Returns after
 * the device work is enqueued and the host buffers have been consumed. */
int lbm_cuboid_init_fields(lbm_cuboid_t *h, const double *rho, const double *u);
/* Same from DEVICE pointers (fp64, same layouts, on this rank's device). */
int lbm_cuboid_init_fields_device(lbm_cuboid_t *h, const double *rho, const double *u);

/* Advance nsteps time steps (pull-stream with wall rules, then collide),
 * asynchronously on the compute stream.  nsteps >= 0.  Collective over the
 * ranks of a z-slab decomposition (all ranks take the same steps). */
int lbm_cuboid_step(lbm_cuboid_t *h, int64_t nsteps);

/* Block until all enqueued work of the handle is complete; reports
 * asynchronous CUDA/NCCL failures, LBM_ESINGULAR if a node's strain-rate
 * system was singular during the steps since the last report (the steps still
 * ran; the flag is cleared once reported), and a failed check_every watch. */
int lbm_cuboid_sync(lbm_cuboid_t *h);

/* rho [nz_l][ny][nx] and u [3][nz_l][ny][nx] (fp64) of the stored state into
 * HOST buffers (synchronises) or into DEVICE buffers (asynchronous). */
int lbm_cuboid_get_macroscopic(lbm_cuboid_t *h, double *rho, double *u);
int lbm_cuboid_get_macroscopic_device(lbm_cuboid_t *h, double *rho, double *u);

/* Stored populations, HOST fp64 [27][nz_l][ny][nx], paper direction order.
 * set_populations also refreshes the halo ghost planes (collective like
 * init_fields). */
int lbm_cuboid_get_populations(lbm_cuboid_t *h, double *f);
/* Planes [z_begin, z_begin + n_planes) of the local slab only: HOST fp64
 * [27][n_planes][ny][nx], paper direction order. */
int lbm_cuboid_get_populations_planes(lbm_cuboid_t *h, int32_t z_begin, int32_t n_planes, double *f);
int lbm_cuboid_set_populations(lbm_cuboid_t *h, const double *f);

/* Rank-local reductions of the stored state, fp64:
 * out[0] = sum rho, out[1..3] = sum rho u, out[4] = sum rho |u|^2 / 2,
 * out[5] = max |u|, out[6] = number of nodes with NaN/Inf, rho <= 0 or |u| > 1.
 * Synchronises.  Returns LBM_EUNSTABLE if out[6] > 0, else LBM_ESINGULAR if
 * the singular-system flag is set (see lbm_cuboid_sync). */
int lbm_cuboid_check(lbm_cuboid_t *h, double out[7]);

/* Replace the body force (e.g. time-periodic forcing); takes effect for the
 * steps enqueued after the call. */
int lbm_cuboid_set_force(lbm_cuboid_t *h, const double force[3]);

/* Introspection:
 * out[0] = kernel launches enqueued so far by this handle (all kernels),
 * out[1] = collide-stream launches, out[2] = steps taken,
 * out[3] = algorithmic bytes per node update (2 * 27 * sizeof(real)),
 * out[4] = local node count, out[5] = bytes of one buffer,
 * out[6] = ghost-plane exchange: 0 none (in-kernel wrap), 1 NCCL, 2 fused P2P,
 * out[7] = 1 if the paper-rate specialisation (omega_1 = omega_high = 1) is used. */
int lbm_cuboid_info(const lbm_cuboid_t *h, int64_t out[8]);

/* cudaStream_t of the compute stream (for event timing by the caller). */
void *lbm_cuboid_stream(const lbm_cuboid_t *h);

/* Name of the collide-stream kernel this handle's steps launch (e.g.
 * "k_collide_stream_paper_shape<double,512,512>"; "k_collide_stream_fd_tma<double>"
 * for FULL_FD through the TMA-staged fused kernel; "+ k_density" for the
 * two-pass FULL_FD), for profiles and the bench's roofline record.  Valid until
 * the next call on the handle; "" for NULL. */
const char *lbm_cuboid_kernel_name(const lbm_cuboid_t *h);

/* The handle's NCCL communicator (ghost-plane exchange with LBM_HALO_AUTO at
 * world > 1, or LBM_HALO_NCCL): out[0] = ncclCommCount, out[1] = this rank in
 * it (ncclCommUserRank); both -1 when the handle has no communicator (single
 * GPU with in-kernel wrap, or the fused P2P halo).  Host-only query. */
int lbm_cuboid_comm_ranks(const lbm_cuboid_t *h, int32_t out[2]);

/* Per-launch timing of the collide-stream kernel: while enabled, every launch
 * is bracketed by a CUDA event pair on the compute stream (at most 65536
 * launches are recorded).  lbm_cuboid_timing() synchronises and clears the
 * record; lbm_cuboid_timing_read() synchronises and returns
 * out[0] = launches recorded, out[1] = their summed duration in ms,
 * out[2] = node updates they performed. */
int lbm_cuboid_timing(lbm_cuboid_t *h, int enable);
int lbm_cuboid_timing_read(lbm_cuboid_t *h, double out[3]);

/* Trace of the step structure (SURVEY §5 tracing; nsys is not available on this
 * pool): while enabled, every collide-stream / density launch and every NCCL
 * halo exchange is bracketed by a CUDA event pair on the stream it is enqueued
 * on (compute stream 0, halo/comm stream 1), so the overlap of the boundary
 * planes, the halo and the interior can be read back (CUDA graphs are not used
 * while tracing).  lbm_cuboid_trace() synchronises, clears the record and
 * starts it (enable != 0) or stops it.  lbm_cuboid_trace_read() synchronises
 * and writes min(max_rows, recorded) rows of 6 doubles into out:
 * {kind (0 collide-stream launch, 1 boundary-plane launch, 2 NCCL halo
 * exchange, 3 density pass), stream (0 compute, 1 halo), first plane, planes,
 * start ms, end ms} (times from the enable call's event on the compute stream);
 * *rows = number recorded (at most 65536). */
int lbm_cuboid_trace(lbm_cuboid_t *h, int enable);
int lbm_cuboid_trace_read(lbm_cuboid_t *h, double *out, int32_t max_rows, int32_t *rows);

/* Release library state (streams, events, NCCL comm, library-owned buffers).
 * Caller-owned buffers are untouched.  NULL is accepted. */
int lbm_cuboid_destroy(lbm_cuboid_t *h);

/* Message of the last failure on this thread ("" if none). */
const char *lbm_cuboid_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* LBM_CUBOID_H */
