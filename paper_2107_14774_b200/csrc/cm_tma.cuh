// cm_tma.cuh -- TMA-staged collide-stream kernel of the 3D cuboid
// central-moment LBM (arXiv 2107.14774): the pull of the 27 populations
// done by the tensor memory accelerator instead of per-thread
// address arithmetic.  "P:Lnnn" cites /root/reference/PAPER.md line nnn.
//
// The population buffer buf[((p*27 + q)*ny + y)*nx + x] is a 3D tensor
// (x: nx, y: ny, pq: 27 (nz_l + 2)) for the TMA unit.  A tile is a row segment
// of kTmaTx nodes (x0 .. x0 + kTmaTx - 1, row y, plane z).  For direction q
// with velocity e the pulled values of the tile are the row segment
//     R_q[x0 - e_x .. x0 - e_x + kTmaTx - 1],  R_q = buf[., y - e_y, (z - e_z + 1) 27 + q]
// with y - e_y and z - e_z wrapped (periodic) or pointing at a ghost plane.
// The TMA unit only starts a box on a 16-byte boundary of the row (measured on
// the B200: a box at x0 +- 1 raises an illegal-instruction fault;
// scripts/tma_min.cu), so the 9 directions with e_x = 0 load the aligned box
// [x0, x0 + kTmaTx) and the 18 with e_x = +-1 load the aligned superset
// [x0 - V, x0 + kTmaTx + V), V = 16 bytes / sizeof(real), and each node reads
// its element at offset tx + V - e_x.  27 cp.async.bulk.tensor instructions,
// issued by one producer thread, stage a tile; every consumer thread reads its
// node's 27 values at compile-time shared-memory offsets (no per-thread
// address arithmetic).  Elements beyond the row (x0 - V < 0, x0 + kTmaTx + V
// > nx) are zero-filled by the TMA unit; across a periodic x face the node at
// x = 0 / nx - 1 needs the row's other end: with fp32 storage the producer
// stages it with 16-byte "wrap" boxes (9 per tile end); with fp64 the warp
// holding that node takes the global-memory gather path instead (shared
// memory is the occupancy limit there).  Warps with a wall-adjacent node gather
// through the wall rules from global memory (gather(), out of line).
//
// Pipeline: a persistent grid; each CTA walks tiles t = blockIdx.x + i gridDim.x.
// The stage buffers form a ring guarded by two mbarriers per stage: full (the
// producer arms it with the expected byte count, the TMA unit completes it)
// and empty (one arrival per consumer warp once it has copied its values into
// registers).  Warp kTmaWarps (the extra warp) is the producer; the kTmaWarps
// consumer warps collide and store (st.global.cs).  The per-node arithmetic is
// the one of collide_stream_ab.
#pragma once

#include <cuda.h>

#include "cm_common.cuh"
#include "cm_kernels.cuh"
#include "cm_moments.cuh"
#include "cm_stream.cuh"

namespace lbm {

#ifndef LBM_TMA_TX
#define LBM_TMA_TX 128  // nodes per tile (one consumer thread each)
#endif
#ifndef LBM_TMA_STAGES32
#define LBM_TMA_STAGES32 3  // stages of the ring with fp32 storage
#endif
#ifndef LBM_TMA_STAGES64
#define LBM_TMA_STAGES64 2  // stages with fp64
#endif
#ifndef LBM_TMA_MINB
#define LBM_TMA_MINB 3  // 3 x 160 threads: 136 registers (4: 96 with spills, measured slower)
#endif
#ifndef LBM_FD_TMA_STAGES
#define LBM_FD_TMA_STAGES 2  // FULL_FD TMA kernel: stages of the ring (one read, one in flight)
#endif
#ifndef LBM_FD_TMA_MINB64
#define LBM_FD_TMA_MINB64 2  // resident CTAs per SM (fp64: 2 x 103 KB of shared memory)
#endif
#ifndef LBM_FD_TMA_MINB32
#define LBM_FD_TMA_MINB32 3
#endif
#ifndef LBM_TMA_WRAPBOX32
#define LBM_TMA_WRAPBOX32 1  // fp32: stage the x-wrap column with wrap boxes
#endif
#ifndef LBM_TMA_WRAPBOX64
#define LBM_TMA_WRAPBOX64 0  // fp64: the x-wrap warps gather from global memory
#endif
constexpr int kTmaTx = LBM_TMA_TX;
constexpr int kTmaWarps = kTmaTx / 32;    // consumer warps
constexpr int kTmaThreads = kTmaTx + 32;  // + one producer warp

// shared-memory layout of one stage (bytes; every box starts on a 128-byte
// boundary, the TMA destination alignment: a 16-byte-aligned destination
// faulted with "misaligned address" on the B200)
template <typename T> struct TmaLayout {
  static constexpr int V = 16 / int(sizeof(T));                          // elements per 16 bytes
  static constexpr int kCenter = kTmaTx * int(sizeof(T));                // e_x = 0 box
  static constexpr int kShiftW = kTmaTx + 2 * V;                         // e_x = +-1 box width
  static constexpr int kShift = ((kShiftW * int(sizeof(T)) + 127) / 128) * 128;
  static constexpr bool kWrap = sizeof(T) == 8 ? LBM_TMA_WRAPBOX64 : LBM_TMA_WRAPBOX32;
  static constexpr int kWrapBox = 128;                                   // one 16-byte box, padded
  static constexpr int kStages = sizeof(T) == 8 ? LBM_TMA_STAGES64 : LBM_TMA_STAGES32;
  // 9 center boxes (m = j + 3k), 18 shifted boxes (2m: e_x = +1, 2m + 1: e_x = -1), 18 wrap boxes
  static constexpr int kOffShift = 9 * kCenter;
  static constexpr int kOffWrap = kOffShift + 18 * kShift;
  static constexpr int kStage = kOffWrap + (kWrap ? 18 * kWrapBox : 0);
  static constexpr int kTileBytes = (9 * kTmaTx + 18 * kShiftW) * int(sizeof(T));  // TMA bytes per tile
  static constexpr size_t kSmem = size_t(kStages) * kStage + size_t(2 * kStages) * 8;
};
static_assert((kTmaTx * 4) % 128 == 0, "center boxes must keep 128-byte alignment");

template <typename T>
constexpr size_t tma_smem_bytes() {
  return TmaLayout<T>::kSmem;
}

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, unsigned long long* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Tensor maps of one population buffer: box kTmaTx (e_x = 0), kTmaTx + 2V
// (e_x = +-1), V (the x-wrap column)
struct TmaMaps {
  CUtensorMap center, shift, wrap;
};

// Tiles of the launch: planes zbeg + i zstride (i < nplanes), ny rows each,
// ntx = ceil(nx / kTmaTx) segments per row.
struct TmaTiles {
  int zbeg, zstride, nplanes, ntx;
  long long count;  // nplanes * ny * ntx
};

// Warps with a wall-adjacent node (or, without wrap boxes, the x-wrap node):
// the full rules of gather() from global memory, collide, store.  Out of line
// (no array crosses the call), so the registers of the main path (shared
// memory -> collide -> store) stay low.
template <typename T, int KIND>
__device__ __noinline__ void tma_global_node(const T* __restrict__ src, T* __restrict__ dst, const Consts& c, int x,
                                             int y, int z) {
  double f[27];
  gather<T>(src, c, x, y, z, f);
  StoreOwn<T> st{dst, dst + (long long)(z + 1) * c.plane + (y * c.nx + x), c.nxy, &c};
  run_core<KIND, false>(c, f, 0.0, 0.0, 0.0, st);
}

template <typename T, int KIND>
__global__ void __launch_bounds__(kTmaThreads, LBM_TMA_MINB)
    k_collide_stream_tma(const __grid_constant__ TmaMaps maps, const T* __restrict__ src, T* __restrict__ dst,
                         const __grid_constant__ Consts c, const TmaTiles tl) {
  using L = TmaLayout<T>;
  constexpr int V = L::V;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw + size_t(L::kStages) * L::kStage);
  unsigned long long* empty = full + L::kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long per_plane = (long long)c.ny * tl.ntx;
  const bool xwrap = (c.face[0] == FK_WRAP);

  if (warp == kTmaWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.center) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.shift) : "memory");
      int i = 0;
      for (long long t = blockIdx.x; t < tl.count; t += gridDim.x, ++i) {
        const int s = i % L::kStages;
        const unsigned n = unsigned(i / L::kStages);
        if (n > 0) mbar_wait(&empty[s], (n - 1) & 1);  // consumers released the stage's previous use
        const int pl = int(t / per_plane);
        const int rem = int(t - (long long)pl * per_plane);
        const int y = rem / tl.ntx;
        const int x0 = (rem - y * tl.ntx) * kTmaTx;
        const int z = tl.zbeg + pl * tl.zstride;
        int ys[3], ps[3];  // source row (e_y = j - 1) and plane (e_z = k - 1)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          int v = y - (j - 1);
          if (v < 0) v += c.ny;  // periodic y (a wall face never uses this row: global path)
          if (v >= c.ny) v -= c.ny;
          ys[j] = v;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          int v = z - (k - 1);
          if (v < 0 && c.face[4] == FK_WRAP) v += c.nzl;       // else ghost plane -1 (or unused: wall)
          if (v >= c.nzl && c.face[5] == FK_WRAP) v -= c.nzl;  // else ghost plane nz_l
          ps[k] = (v + 1) * 27;
        }
        const bool lo = L::kWrap && xwrap && x0 == 0;              // x = 0 pulls e_x = +1 from nx - 1
        const bool hi = L::kWrap && xwrap && x0 + kTmaTx >= c.nx;  // x = nx - 1 pulls e_x = -1 from 0
        mbar_expect_tx(&full[s], unsigned(L::kTileBytes + ((lo ? 9 : 0) + (hi ? 9 : 0)) * 16));
        unsigned char* sb = smem_raw + size_t(s) * L::kStage;
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const int m = j + 3 * k;
            tma_load_3d(sb + m * L::kCenter, &maps.center, &full[s], x0, ys[j], ps[k] + LBM_Q(1, j, k));
            tma_load_3d(sb + L::kOffShift + (2 * m) * L::kShift, &maps.shift, &full[s], x0 - V, ys[j],
                        ps[k] + LBM_Q(2, j, k));
            tma_load_3d(sb + L::kOffShift + (2 * m + 1) * L::kShift, &maps.shift, &full[s], x0 - V, ys[j],
                        ps[k] + LBM_Q(0, j, k));
            // the row's last V elements (e_x = +1 at x = 0) / first V (e_x = -1 at x = nx - 1)
            if (lo) tma_load_3d(sb + L::kOffWrap + m * L::kWrapBox, &maps.wrap, &full[s], c.nx - V, ys[j],
                                ps[k] + LBM_Q(2, j, k));
            if (hi) tma_load_3d(sb + L::kOffWrap + (9 + m) * L::kWrapBox, &maps.wrap, &full[s], 0, ys[j],
                                ps[k] + LBM_Q(0, j, k));
          }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int tx = threadIdx.x;
  int i = 0;
  for (long long t = blockIdx.x; t < tl.count; t += gridDim.x, ++i) {
    const int s = i % L::kStages;
    const int pl = int(t / per_plane);
    const int rem = int(t - (long long)pl * per_plane);
    const int y = rem / tl.ntx;
    const int x = (rem - y * tl.ntx) * kTmaTx + tx;
    const int z = tl.zbeg + pl * tl.zstride;
    const bool active = x < c.nx;
    const bool global_path = __any_sync(
        0xffffffffu, active && (wall_adjacent(c, x, y, z) || (!L::kWrap && xwrap && (x == 0 || x == c.nx - 1))));
    mbar_wait(&full[s], unsigned(i / L::kStages) & 1);
    double f[27];
    if (!global_path) {
      const unsigned char* sb = smem_raw + size_t(s) * L::kStage;
      const T* cen = reinterpret_cast<const T*>(sb) + tx;
      const T* sh = reinterpret_cast<const T*>(sb + L::kOffShift) + tx + V;
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int m = j + 3 * k;
          f[LBM_Q(1, j, k)] = (double)cen[m * (L::kCenter / int(sizeof(T)))];
          f[LBM_Q(2, j, k)] = (double)sh[(2 * m) * (L::kShift / int(sizeof(T))) - 1];      // source x - 1
          f[LBM_Q(0, j, k)] = (double)sh[(2 * m + 1) * (L::kShift / int(sizeof(T))) + 1];  // source x + 1
        }
      if (L::kWrap && xwrap && (x == 0 || x == c.nx - 1)) {
        // a source across the periodic x face (the shifted box holds a zero fill there)
        const T* wb = reinterpret_cast<const T*>(sb + L::kOffWrap);
#pragma unroll
        for (int m = 0; m < 9; ++m) {
          if (x == 0) f[LBM_Q(2, m % 3, m / 3)] = (double)wb[m * (L::kWrapBox / int(sizeof(T))) + V - 1];
          if (x == c.nx - 1) f[LBM_Q(0, m % 3, m / 3)] = (double)wb[(9 + m) * (L::kWrapBox / int(sizeof(T)))];
        }
      }
    }
    // release the stage: every thread's shared-memory reads of it are ordered
    // before the TMA unit's next writes into it (async proxy) -- without the
    // fence a warp's outstanding loads could read the refilled stage
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (!active) continue;
    if (global_path) {
      tma_global_node<T, KIND>(src, dst, c, x, y, z);
      continue;
    }
    StoreOwn<T> st{dst, dst + (long long)(z + 1) * c.plane + (y * c.nx + x), c.nxy, &c};
    run_core<KIND, false>(c, f, 0.0, 0.0, 0.0, st);
  }
}

// ------------------------------------------------ TMA-staged fused FULL_FD kernel
// The 2.5D march of collide_stream_fd_fused (cm_kernels.cuh; FULL_FD's
// same-time density) with the pulled populations of each
// plane staged by the TMA unit instead of gathered per thread from L2.
//
// A CTA owns the kFdTx x kFdTy tile (x0, y0) of one z-chunk; iteration p of the
// march needs the pulled populations of plane p on the tile and its one-node
// ring, X in [x0 - 1, x0 + kFdTx], Y in [y0 - 1, y0 + kFdTy].  For direction
// q = (e_x, e_y, e_z) they are the elements (X - e_x, Y - e_y) of slot q of
// plane p - e_z: one box of kFdTy + 2 rows starting at row y0 - 1 - e_y and
// BW = kFdTx + 2V columns starting at x0 - V (16 bytes before the tile, the
// TMA start alignment; V = 16 / sizeof(T) >= 2 covers e_x = +-1 and the ring).
// 27 boxes = one stage; ring node (lx, ly) reads element (ly, lx - 1 + V - e_x)
// of box q, so the consumers form the ring densities and load their own node's
// populations at compile-time offsets from shared memory.
//
// Per iteration p (consumer warps, 128 threads):
//   wait full[stage p] -> rho(p) on tile + ring (sum in q order, as k_density)
//   -> barrier -> collide plane p - 1 with the populations held in registers
//   since the previous iteration and the gradient from the density ring ->
//   load the own node's 27 populations of plane p from the stage -> release it.
// The producer warp (one elected lane) refills a stage as soon as it is
// released, so the next plane's 27 boxes land while the current plane is
// collided.  Two stages: one being read, one in flight.
//
// Across a periodic x face (nx a multiple of kFdTx, >= 2 tiles) the two seam
// tiles are staged too: the box's V columns beyond the row (zero-filled by the
// TMA unit) are the other end of the row, which the producer loads as 27 extra
// V-column "wrap" boxes into a side area (a TMA destination must be 128-byte
// aligned, so they cannot land inside the box rows); the consumers copy them
// into place (then a proxy fence, as the stage is refilled by the TMA unit
// later) before forming the densities.  Tiles whose ring or pull sources leave
// the plane otherwise (y0 < 2 or y0 + kFdTy + 2 > ny: the periodic y seam or a
// wall; an x wall; a partial tile) run the LDG body of the fused kernel
// instead (CTA-uniform).  z faces must be periodic or ghost planes (the
// host selects this kernel only then); planes next to a ghost face take their
// density from the exchanged field, as ring_rho.  Identical arithmetic and
// source values as collide_stream_fd_fused, so the results are bitwise those of
// k_collide_stream_fd.
template <typename T> struct TmaFdLayout {
  static constexpr int V = 16 / int(sizeof(T));
  static constexpr int BW = kFdTx + 2 * V;  // box columns
  static constexpr int BH = kFdTy + 2;      // box rows
  static constexpr int kBox = ((BW * BH * int(sizeof(T)) + 127) / 128) * 128;
  static constexpr int kWrapBox = ((V * BH * int(sizeof(T)) + 127) / 128) * 128;  // V columns x BH rows
  static constexpr int kStages = LBM_FD_TMA_STAGES;
  static constexpr int kOffWrap = 27 * kBox;
  static constexpr int kStage = kOffWrap + 27 * kWrapBox;
  static constexpr unsigned kTx = 27u * BW * BH * unsigned(sizeof(T));         // TMA bytes per stage
  static constexpr unsigned kTxWrap = 27u * V * BH * unsigned(sizeof(T));      // + the wrap boxes (seam tile)
  static constexpr int kOffBar = kStages * kStage;
  static constexpr int kOffRho = kOffBar + 2 * kStages * 8;
  static constexpr size_t kSmem = size_t(kOffRho) + sizeof(double) * 4 * (kFdTy + 2) * kFdRw;
};
constexpr int kFdTmaThreads = kFdThreads + 32;  // + the producer warp
struct FdTmaMaps {
  CUtensorMap box;   // kFdTx + 2V columns x kFdTy + 2 rows x 1 slot
  CUtensorMap wrap;  // V columns x kFdTy + 2 rows x 1 slot (x seam)
};

template <typename T, int KIND>
__global__ void __launch_bounds__(kFdTmaThreads, sizeof(T) == 8 ? LBM_FD_TMA_MINB64 : LBM_FD_TMA_MINB32)
    k_collide_stream_fd_tma(const __grid_constant__ FdTmaMaps maps, const T* __restrict__ src, T* __restrict__ dst,
                            const double* __restrict__ rf, const __grid_constant__ Consts c, int zbeg, int zstride,
                            int zlen, int zend) {
  using L = TmaFdLayout<T>;
  constexpr int V = L::V;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw + L::kOffBar);
  unsigned long long* empty = full + L::kStages;
  FdRho* srho = reinterpret_cast<FdRho*>(smem_raw + L::kOffRho);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int x0 = blockIdx.x * kFdTx, y0 = blockIdx.y * kFdTy;
  auto consumer_sync = [] { asm volatile("bar.sync 1, %0;" ::"n"(kFdThreads) : "memory"); };
  // tile whose ring and pull sources stay inside the plane (no seam, no wall)
  const bool xseam_ok = c.face[0] == FK_WRAP && c.nx % kFdTx == 0 && c.nx >= 2 * kFdTx;
  const bool lo_seam = xseam_ok && x0 == 0;                // box columns [0, V): x = nx - V .. nx - 1
  const bool hi_seam = xseam_ok && x0 + kFdTx == c.nx;     // box columns [BW - V, BW): x = 0 .. V - 1
  const bool staged = (lo_seam || hi_seam || (x0 >= kFdTx && x0 + kFdTx + 2 <= c.nx)) && y0 >= 2 &&
                      y0 + kFdTy + 2 <= c.ny;
  const bool seam = lo_seam || hi_seam;
  if (!staged) {
    if (warp < kFdThreads / 32)
      collide_stream_fd_fused<T, KIND>(src, dst, rf, c, zbeg, zstride, zlen, zend, srho, consumer_sync,
                                       int(threadIdx.x));
    return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kFdThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int z0 = zbeg + blockIdx.z * zstride;
  const int z1 = min(z0 + zlen, zend);
  const int niter = z1 - z0 + 2;  // p = z0 - 1 .. z1
  // planes whose density comes from the exchanged field (next to / beyond a ghost face)
  // a plane is staged when its density is summed here or its populations are
  // collided in this launch (a plane next to a ghost face collided by a
  // contiguous boundary launch, nz_l = 2: density from the field, populations staged)
  auto staged_plane = [&](int p) {
    return !((p <= 0 && c.face[4] == FK_GHOST) || (p >= c.nzl - 1 && c.face[5] == FK_GHOST)) ||
           (p >= z0 && p < z1);
  };
  auto from_field = [&](int p) {
    return (p <= 0 && c.face[4] == FK_GHOST) || (p >= c.nzl - 1 && c.face[5] == FK_GHOST);
  };

  if (warp == kFdThreads / 32) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.box) : "memory");
      for (int it = 0; it < niter; ++it) {
        const int s = it % L::kStages;
        const unsigned n = unsigned(it / L::kStages);
        if (n > 0) mbar_wait(&empty[s], (n - 1) & 1);
        const int p = z0 - 1 + it;
        if (!staged_plane(p)) {
          mbar_arrive(&full[s]);  // nothing to stage: complete the phase
          continue;
        }
        // periodic z (a plane beyond a ghost face is never staged)
        const int pw = (p < 0) ? p + c.nzl : (p >= c.nzl ? p - c.nzl : p);
        mbar_expect_tx(&full[s], L::kTx + (seam ? L::kTxWrap : 0u));
        unsigned char* sb = smem_raw + size_t(s) * L::kStage;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          int ps = pw - (k - 1);  // source plane of e_z = k - 1: wrapped, or the ghost plane -1 / nz_l
          if (ps < 0 && c.face[4] == FK_WRAP) ps += c.nzl;
          if (ps >= c.nzl && c.face[5] == FK_WRAP) ps -= c.nzl;
#pragma unroll
          for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              const int q = LBM_Q(i, j, k);
              tma_load_3d(sb + q * L::kBox, &maps.box, &full[s], x0 - V, y0 - j, (ps + 1) * 27 + q);
              if (seam)
                tma_load_3d(sb + L::kOffWrap + q * L::kWrapBox, &maps.wrap, &full[s], lo_seam ? c.nx - V : 0,
                            y0 - j, (ps + 1) * 27 + q);
            }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int tid = threadIdx.x;
  const int tx = tid % kFdTx, ty = tid / kFdTx;
  const int x = x0 + tx, y = y0 + ty;
  double f[27];
  for (int it = 0; it < niter; ++it) {
    const int s = it % L::kStages;
    const int p = z0 - 1 + it;
    mbar_wait(&full[s], unsigned(it / L::kStages) & 1);
    const T* sb = reinterpret_cast<const T*>(smem_raw + size_t(s) * L::kStage);
    constexpr int kBoxE = L::kBox / int(sizeof(T));
    if (seam && staged_plane(p)) {  // the wrap columns into the box rows (CTA-uniform)
      T* sbw = const_cast<T*>(sb);
      const T* wb = reinterpret_cast<const T*>(smem_raw + size_t(s) * L::kStage + L::kOffWrap);
      for (int i = tid; i < 27 * L::BH * V; i += kFdThreads) {
        const int q = i / (L::BH * V), r = (i / V) % L::BH, cc = i % V;
        sbw[q * kBoxE + r * L::BW + (lo_seam ? cc : L::BW - V + cc)] = wb[q * (L::kWrapBox / int(sizeof(T))) + r * V + cc];
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes before the next TMA refill
      consumer_sync();
    }
    if (from_field(p)) {
      for (int pos = tid; pos < kFdRing; pos += kFdThreads) {
        const int ly = pos / kFdRw, lx = pos - ly * kFdRw;
        int gx = x0 + lx - 1;  // wrapped across the periodic x seam
        gx += (gx < 0) ? c.nx : (gx >= c.nx ? -c.nx : 0);
        srho[p & 3][ly][lx] = __ldg(rf + (long long)(p + 1) * c.nxy + (y0 + ly - 1) * c.nx + gx);
      }
    } else {
      for (int pos = tid; pos < kFdRing; pos += kFdThreads) {
        const int ly = pos / kFdRw, lx = pos - ly * kFdRw;
        const T* e = sb + ly * L::BW + lx - 1 + V;
        double r0 = 0.0;
#pragma unroll
        for (int q = 0; q < 27; ++q) r0 += (double)e[q * kBoxE - (q % 3 - 1)];
        srho[p & 3][ly][lx] = r0;
      }
    }
    consumer_sync();
    if (it >= 2) {  // collide plane p - 1 (its populations are in f since the last iteration)
      const int z = p - 1;
      double gxr, gyr, gzr;
      auto at = [&](int i, int j, int k) { return srho[(z + k - 1) & 3][ty + j][tx + i]; };
      density_gradient_g<decltype(at), true>(c, x, y, z, at, gxr, gyr, gzr);
      StoreOwn<T> st{dst, dst + (long long)(z + 1) * c.plane + (y * c.nx + x), c.nxy, &c};
      run_core<KIND, true>(c, f, gxr, gyr, gzr, st);
    }
    if (p >= z0 && p < z1) {  // own populations of plane p, collided next iteration
      const T* e = sb + (ty + 1) * L::BW + tx + V;
#pragma unroll
      for (int q = 0; q < 27; ++q) f[q] = (double)e[q * kBoxE - (q % 3 - 1)];
    }
    // release the stage: every thread's shared-memory reads of it are ordered
    // before the TMA unit's next writes into it (async proxy) -- without the
    // fence a warp's outstanding loads could read the refilled stage
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

}  // namespace lbm
