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

}  // namespace lbm
