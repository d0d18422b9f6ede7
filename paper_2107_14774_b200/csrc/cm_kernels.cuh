// cm_kernels.cuh -- sm_100a kernels of the 3D cuboid central-moment LBM
// (arXiv 2107.14774).  "P:Lnnn" cites /root/reference/PAPER.md line nnn.
//
// Layout in HBM: one buffer per time level,
//   buf[(p*27 + q)*nxy + y*nx + x],  p = z_local + 1 in [0, nz_l + 1]
// (p = 0 and p = nz_l + 1 are ghost planes filled by the halo exchange), and the
// internal direction index q = (ex+1) + 3(ey+1) + 9(ez+1) with e in {-1,0,1}^3,
// so the 9 directions with e_z = -1 / 0 / +1 are contiguous in a plane (one
// contiguous send/recv region per slab face).
//
// The per-node moment transforms are the tensor-product (per-axis) form of
// m^c = F S P f and f~ = P^-1 S^-1 F^-1 m~^c (Eq. LBEcentralmomentcuboidlattice,
// P:L676-681): central moments k_mnp = sum_a f_a (e_ax-u_x)^m (e_ay-u_y)^n (e_az-u_z)^p
// (Eq. 3a) factorise over the three axes, so each of the 27x27
// transforms is three passes of nine 3-point transforms, all in registers.
//
// This file holds the __global__ kernels; the per-node arithmetic is in
// cm_moments.cuh, the pull sources / wall rules / store policies in
// cm_stream.cuh, shared definitions in cm_common.cuh.
#pragma once

#include <cooperative_groups.h>

#include "cm_common.cuh"
#include "cm_moments.cuh"
#include "cm_stream.cuh"

namespace lbm {

// density pass for FULL_FD: rho(x, t+1) = sum_q f_q(x, t+1) of the pulled populations
template <typename T>
__global__ void __launch_bounds__(kBlock) k_density(const T* __restrict__ src, double* __restrict__ rho_out,
                                                    const __grid_constant__ Consts c, int zbeg, int zstride) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx >= c.nxy) return;
  const int y = row_of(c, idx);
  const int x = idx - y * c.nx;
  const int z = zbeg + blockIdx.y * zstride;
  double f[27];
  gather<T>(src, c, x, y, z, f);
  double r0 = 0.0;
#pragma unroll
  for (int q = 0; q < 27; ++q) r0 += f[q];
  rho_out[(long long)(z + 1) * c.nxy + idx] = r0;
}

// ------------------------------------- fused FULL_FD collide-stream (2.5D blocking)
// FULL_FD needs the same-time density of the 26 neighbours, i.e. their pulled
// populations.  Instead of a separate density pass (+216 B/node of HBM reads
// and a density field), a CTA owns a kFdTx x kFdTy tile of one z-chunk and
// marches up the chunk: at plane p it gathers the pulled populations of the
// tile and its one-node ring (periodic wrap; ghost planes from the exchanged
// density field), sums them to rho and keeps rho of the last four planes in a
// shared-memory ring; then it collides plane p - 1 with the gradient read from
// shared memory, re-gathering the node's own populations (an L2 hit: the same
// CTA read them one plane earlier).  Every population comes from HBM once
// (plus the 2/kFdZc chunk overlap), the neighbour reuse of rho lives in shared
// memory, and the arithmetic is density_gradient's and k_density's, so the
// result is bitwise that of the two-pass path.
#ifndef LBM_FD_ZC
#define LBM_FD_ZC 32  // planes per z-chunk
#endif
#ifndef LBM_FD_TY
#define LBM_FD_TY 4   // tile rows (tile = 32 x LBM_FD_TY nodes, one thread each)
#endif
#ifndef LBM_FD_MINB
#define LBM_FD_MINB 4 // resident CTAs per SM requested from ptxas
#endif
#ifndef LBM_FD_TX
#define LBM_FD_TX 32  // tile columns
#endif
constexpr int kFdTx = LBM_FD_TX, kFdTy = LBM_FD_TY, kFdThreads = kFdTx * kFdTy, kFdZc = LBM_FD_ZC;
constexpr int kFdRw = kFdTx + 2, kFdRing = (kFdTx + 2) * (kFdTy + 2);

// rho(t+1) at node (gx, gy, p) of the tile ring (coordinates may lie one node
// outside the slab/grid); 0 where no active node of the tile needs it (across
// a wall, or beyond a partial tile)
template <typename T>
__device__ __forceinline__ double ring_rho(const T* src, const double* rf, const Consts& c, int gx, int gy, int p) {
  if (gx < 0 || gx >= c.nx) {
    if (c.face[0] != FK_WRAP || gx < -1 || gx > c.nx) return 0.0;
    gx = (gx < 0) ? c.nx - 1 : 0;
  }
  if (gy < 0 || gy >= c.ny) {
    if (c.face[2] != FK_WRAP || gy < -1 || gy > c.ny) return 0.0;
    gy = (gy < 0) ? c.ny - 1 : 0;
  }
  if (p < 0 || p >= c.nzl) {
    const int fk = c.face[p < 0 ? 4 : 5];
    if (fk == FK_GHOST) return __ldg(rf + (long long)(p + 1) * c.nxy + gy * c.nx + gx);
    if (fk != FK_WRAP) return 0.0;
    p = (p < 0) ? c.nzl - 1 : 0;
  }
  // a slab plane next to a ghost face: its pulled populations come partly from
  // the ghost plane, which a neighbour overwrites concurrently with this launch
  // (fused P2P halo: the neighbour's next step may start once this slab's
  // boundary launch has published).  Its density is formed before this launch
  // by the boundary-plane density pass (k_density / k_density_p2p), so read it
  // from the density field and never touch the ghost planes here.
  if ((p == 0 && c.face[4] == FK_GHOST) || (p == c.nzl - 1 && c.face[5] == FK_GHOST))
    return __ldg(rf + (long long)(p + 1) * c.nxy + gy * c.nx + gx);
  double f[27];
  gather<T>(src, c, gx, gy, p, f);
  double r0 = 0.0;
#pragma unroll
  for (int q = 0; q < 27; ++q) r0 += f[q];
  return r0;
}

// ------------------------------------------------ the fused kernels (two buffers)
// One thread per node of planes zbeg + i*zstride, i < gridDim.y, of the local
// slab: pull (gather) from src, collide, store at the own node of dst.
// SNX > 0: the plane width is the compile-time SNX (k_collide_stream_paper_shape)
template <typename T, int KIND, bool FD, int SNX = 0>
__device__ __forceinline__ void collide_stream_ab(const T* __restrict__ src, T* __restrict__ dst,
                                                  const double* __restrict__ rf, const Consts& c, int zbeg,
                                                  int zstride) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx >= c.nxy) return;
  const int y = SNX ? idx / SNX : row_of(c, idx);
  const int x = idx - y * c.nx;
  const int z = zbeg + blockIdx.y * zstride;  // zstride > 1: the two boundary planes in one launch
  double f[27];
  // FULL_FD: gradient first, so its L2-resident loads overlap the population loads
  double gxr = 0.0, gyr = 0.0, gzr = 0.0;
  if (FD) density_gradient(rf, c, x, y, z, gxr, gyr, gzr);
  bool interior = false;
  if (SNX > 0 && SNX % 32 == 0) {
    // compile-time plane width, a multiple of the warp: a warp is 32 nodes of one
    // row, so the warp-uniform interior test of gather() reduces to the warp's
    // first x, its row and its plane -- decided before any per-lane source index
    // is formed (the general prologue costs ~100 instructions per node)
    const int x0 = x & ~31;
    interior = x0 > 0 && x0 + 32 < SNX && y > 0 && y < c.ny - 1 &&
               !(z == 0 && (c.face[4] == FK_WRAP || (c.face[4] >= FK_BOUNCE && c.face[4] <= FK_SLIP))) &&
               !(z == c.nzl - 1 && (c.face[5] == FK_WRAP || (c.face[5] >= FK_BOUNCE && c.face[5] <= FK_SLIP)));
  }
  if (interior) {
    const T* b = src + (long long)(z + 1) * c.plane + idx;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int q = LBM_Q(i, j, k);
          f[q] = ldg(LBM_CHECK_LD(src, b + ((long long)(1 - k) * c.plane + (q * c.nxy + (1 - j) * c.nx + (1 - i))), c));
        }
  } else {
    gather<T>(src, c, x, y, z, f);
  }
  StoreOwn<T, FD> st{dst, dst + (long long)(z + 1) * c.plane + idx, c.nxy, &c,
                     (FD && c.rf_out) ? c.rf_out + (long long)(z + 1) * c.nxy + idx : nullptr};
  run_core<KIND, FD>(c, f, gxr, gyr, gzr, st);
}

template <typename T, bool FD>
__global__ void LBM_CS_BOUNDS_FD(FD) k_collide_stream(const T* __restrict__ src, T* __restrict__ dst,
                                               const double* __restrict__ rf, const __grid_constant__ Consts c,
                                               int zbeg, int zstride) {
  collide_stream_ab<T, CORE_GENERIC, FD>(src, dst, rf, c, zbeg, zstride);
}

template <typename T, bool FD>
__global__ void LBM_CS_BOUNDS_FD(FD) k_collide_stream_paper(const T* __restrict__ src, T* __restrict__ dst,
                                                     const double* __restrict__ rf, const __grid_constant__ Consts c,
                                                     int zbeg, int zstride) {
  collide_stream_ab<T, CORE_PAPER, FD>(src, dst, rf, c, zbeg, zstride);
}

// Plane-shape specialisation of the paper-rate kernel (the default collision of
// every BASELINE configuration): with nx and ny compile-time constants every
// pull-source and store offset of the warp-uniform interior path is a constant,
// which the loads and stores carry as immediates (27 LDG + 8 integer
// instructions per node instead of 27 LDG + ~160; cuobjdump), the rest of the
// code is the same inlined collide_stream_ab, so results are bitwise those of
// k_collide_stream_paper (also with the density-gradient terms: FD, whose
// 26-neighbour density stencil gets immediate offsets too).  Instantiated for the
// plane shapes of the BASELINE configs 3-5 (lbm_cuboid.cu, launch_cs); other
// shapes use the general kernel.
// fp32 storage: 7 resident 128-thread CTAs per SM (78 -> 72 registers): 28.9-29.0 k
// vs 28.6 k MLUPS at 512^3, 30.1 k vs 29.1 k on the config-3 cavity, 27.5 k vs
// 27.2 k over 600 steps (profiles/r2/shape_minb32.jsonl; 8 CTAs: slower)
#ifndef LBM_SHAPE_MINB32
#define LBM_SHAPE_MINB32 7
#endif
template <typename T, int SNX, int SNY, bool FD>
__global__ void __launch_bounds__(kBlock, (FD) ? LBM_FD_CS_MINB : ((sizeof(T) == 4 && LBM_SHAPE_MINB32) ? LBM_SHAPE_MINB32 : LBM_MINB))
    k_collide_stream_paper_shape(const T* __restrict__ src, T* __restrict__ dst,
                                                                  const double* __restrict__ rf,
                                                                  const __grid_constant__ Consts c0, int zbeg,
                                                                  int zstride) {
  Consts c = c0;
  c.nx = SNX;
  c.ny = SNY;
  c.nxy = SNX * SNY;
  c.plane = 27LL * SNX * SNY;
  collide_stream_ab<T, CORE_PAPER, FD, SNX>(src, dst, rf, c, zbeg, zstride);
}

template <typename T, bool FD>
__global__ void LBM_CS_BOUNDS_FD(FD) k_collide_stream_raw(const T* __restrict__ src, T* __restrict__ dst,
                                                   const double* __restrict__ rf, const __grid_constant__ Consts c,
                                                   int zbeg, int zstride) {
  collide_stream_ab<T, CORE_RAW, FD>(src, dst, rf, c, zbeg, zstride);
}

// ------------------------------------- x-pair kernel (fp32 storage, nx even)
// One thread per pair of nodes (x, x + 1), x even, with 8-byte float2 loads and
// stores (north_star: vectorised HBM access).  For direction q the pair's
// sources in row R_q (plane z - e_z, row y - e_y, slot q) are
//   e_x =  0: (R[x],     R[x + 1])  = the aligned pair P = R[x .. x+1]
//   e_x = +1: (R[x - 1], R[x])      = (hi of lane-1's P, lo of P)
//   e_x = -1: (R[x + 1], R[x + 2])  = (hi of P, lo of lane+1's P)
// so a warp (32 pairs = 64 consecutive x of one row) issues ONE aligned 8-byte
// load and at most one shuffle per direction; lane 0 / lane 31 fetch the one
// value beyond the warp with a predicated scalar load (wrapped across a
// periodic x face).  Rows and planes wrap periodically or address the ghost
// planes as in gather().  A warp with any lane next to a wall, at the ragged
// end of the plane, or whose x-neighbour pair sits on another row, gathers
// each node with gather() instead.  Node x is
// collided first and its 27 results are kept as fp32; node x + 1's collision
// then stores each direction of both nodes as one float2.  The per-node
// arithmetic, the loaded values and the stored values are exactly those of the
// one-node-per-thread kernel, so the results are bitwise equal to it.
template <typename T>
struct StoreStash {  // node x: keep the rounded results until node x + 1's are known
  float (&a)[27];
  __device__ __forceinline__ void begin(double) {}
  __device__ __forceinline__ void operator()(int q, double v) const { a[q] = (float)v; }
};

template <typename T>
struct StorePair {  // node x + 1: store (node x, node x + 1) of direction q as one float2
  float2* out;      // own pair of slot 0 (plane z)
  int nxy2;         // nxy / 2 (float2 elements per slot)
  const float (&a)[27];
  const Consts* c;
  const T* base;
  __device__ __forceinline__ void begin(double) {}
  __device__ __forceinline__ void operator()(int q, double v) const {
    float2* p = out + q * nxy2;
#ifdef LBM_DEBUG_BOUNDS
    if ((unsigned long long)((const T*)p - base) + 1 >= (unsigned long long)c->buf_elems) {
      atomicOr(c->dbg_flag, 1u);
      return;
    }
#endif
    __stcs(p, make_float2(a[q], (float)v));
  }
};

#ifndef LBM_XP_MINB
#define LBM_XP_MINB 4  // paper-rate kernel: resident 128-thread CTAs per SM requested from ptxas (<= 128 registers)
#endif
template <int KIND>
__global__ void __launch_bounds__(kBlock, KIND == CORE_PAPER ? LBM_XP_MINB : 3) k_collide_stream_xpair(const float* __restrict__ src, float* __restrict__ dst,
                                                     const __grid_constant__ Consts c, int zbeg, int zstride) {
  const int npair = c.nxy >> 1;
  const int pi = blockIdx.x * kBlock + threadIdx.x;
  if (pi >= npair) return;
  const int idx = 2 * pi;
  const int y = row_of(c, idx);
  const int x = idx - y * c.nx;  // even
  const int z = zbeg + blockIdx.y * zstride;
  const unsigned mask = __activemask();
  const int lane = threadIdx.x & 31;
  // pull sources of node x (rows and planes with periodic wrap or ghost planes)
  const PullSrc<float> ps(src, c, x, y, z);
  const bool wall = ps.wall || (c.has_walls && x + 1 == c.nx - 1 && c.face[1] >= FK_BOUNCE && c.face[1] <= FK_SLIP);
  // a lane whose x-neighbour pair lies on another row (a warp spanning two
  // rows) or beyond a periodic x face can use the shuffle only if it is the
  // warp's first / last lane, which loads that value itself (wrapped in x)
  const bool lane_ok = !wall && (x > 0 || lane == 0) && (x + 2 < c.nx || lane == 31);
  const bool fast = (mask == 0xffffffffu) && __all_sync(mask, lane_ok);
  float a[27];
  double f[27];
  float2* own = reinterpret_cast<float2*>(dst + (long long)(z + 1) * c.plane + idx);
  const int nxy2 = c.nxy >> 1;
  if (fast) {
    // no lane next to a wall: every direction is one aligned float2 of row
    // R_q = plane ps.pz[k], row ps.sy[j], slot q, plus one shuffle (e_x != 0)
    const int xm = (x == 0) ? c.nx - 1 : x - 1;       // lane 0's extra source (e_x = +1)
    const int xp2 = (x + 2 == c.nx) ? 0 : x + 2;      // lane 31's extra source (e_x = -1)
    float v1[27];  // node x + 1
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const float* row = ps.pz[k] + ps.sy[j];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int q = LBM_Q(i, j, k);
          const float* r = row + q * c.nxy;  // R_q
          const float2 P = __ldg(reinterpret_cast<const float2*>(LBM_CHECK_LD(src, r + x, c)));
          if (i == 1) {
            a[q] = P.x;
            v1[q] = P.y;
          } else if (i == 2) {  // e_x = +1
            float lo = __shfl_up_sync(0xffffffffu, P.y, 1);
            if (lane == 0) lo = __ldg(LBM_CHECK_LD(src, r + xm, c));
            a[q] = lo;
            v1[q] = P.x;
          } else {  // e_x = -1
            float hi = __shfl_down_sync(0xffffffffu, P.x, 1);
            if (lane == 31) hi = __ldg(LBM_CHECK_LD(src, r + xp2, c));
            a[q] = P.y;
            v1[q] = hi;
          }
        }
      }
#pragma unroll
    for (int q = 0; q < 27; ++q) f[q] = (double)a[q];
    StoreStash<float> s0{a};
    run_core<KIND, false>(c, f, 0.0, 0.0, 0.0, s0);
#pragma unroll
    for (int q = 0; q < 27; ++q) f[q] = (double)v1[q];
    StorePair<float> s1{own, nxy2, a, &c, dst};
    run_core<KIND, false>(c, f, 0.0, 0.0, 0.0, s1);
    return;
  }
  gather<float>(src, c, x, y, z, f);
  StoreStash<float> s0{a};
  run_core<KIND, false>(c, f, 0.0, 0.0, 0.0, s0);
  gather<float>(src, c, x + 1, y, z, f);
  StorePair<float> s1{own, nxy2, a, &c, dst};
  run_core<KIND, false>(c, f, 0.0, 0.0, 0.0, s1);
}

// chunk blockIdx.z covers planes [z0, z1), z0 = zbeg + blockIdx.z * zstride,
// z1 = min(z0 + zlen, zend).  Iteration p forms rho(p) on the tile and its ring,
// then collides plane p - 1.
// srho: the CTA's four-plane density ring; sync: the barrier of the kFdThreads
// threads that run this (the whole CTA, or the consumer warps of the TMA kernel)
typedef double FdRho[kFdTy + 2][kFdRw];
template <typename T, int KIND, class Sync>
__device__ __forceinline__ void collide_stream_fd_fused(const T* __restrict__ src, T* __restrict__ dst,
                                                        const double* __restrict__ rf, const Consts& c, int zbeg,
                                                        int zstride, int zlen, int zend, FdRho* srho, Sync sync,
                                                        int tid) {
  const int tx = tid % kFdTx, ty = tid / kFdTx;
  const int x0 = blockIdx.x * kFdTx, y0 = blockIdx.y * kFdTy;
  const int z0 = zbeg + blockIdx.z * zstride;
  const int z1 = min(z0 + zlen, zend);
  const int x = x0 + tx, y = y0 + ty;
  const bool active = (x < c.nx) && (y < c.ny);
  for (int p = z0 - 1; p <= z1; ++p) {
    // four slots: the slot written here was last read two planes ago, and this
    // iteration's barrier separates the two (one barrier per plane)
    for (int pos = tid; pos < kFdRing; pos += kFdThreads) {
      const int ly = pos / kFdRw, lx = pos - ly * kFdRw;
      srho[p & 3][ly][lx] = ring_rho<T>(src, rf, c, x0 + lx - 1, y0 + ly - 1, p);
    }
    sync();
    if (p > z0 && active) {
      const int z = p - 1;
      double gxr, gyr, gzr;
      density_gradient_g(
          c, x, y, z, [&](int i, int j, int k) { return srho[(z + k - 1) & 3][ty + j][tx + i]; }, gxr, gyr, gzr);
      double f[27];
      gather<T>(src, c, x, y, z, f);
      const int idx = y * c.nx + x;
      StoreOwn<T> st{dst, dst + (long long)(z + 1) * c.plane + idx, c.nxy, &c};
      run_core<KIND, true>(c, f, gxr, gyr, gzr, st);
    }
  }
}

template <typename T, int KIND>
__global__ void __launch_bounds__(kFdThreads, LBM_FD_MINB)
    k_collide_stream_fd(const T* __restrict__ src, T* __restrict__ dst, const double* __restrict__ rf,
                        const __grid_constant__ Consts c, int zbeg, int zstride, int zlen, int zend) {
  __shared__ double srho[4][kFdTy + 2][kFdRw];
  collide_stream_fd_fused<T, KIND>(src, dst, rf, c, zbeg, zstride, zlen, zend, srho, [] { __syncthreads(); },
                                   int(threadIdx.x));
}

// ------------------------------------ fused collide-stream + peer-memory halo (P2P)
// LBM_HALO_P2P: the launch over the two boundary planes of the slab also stores
// the nine outgoing directions of each boundary plane straight into the
// neighbour's ghost plane of the same time level (NVLink peer memory, or this
// GPU's own ghost plane when the neighbour is this slab), then the last CTA
// publishes the step's epoch in the neighbours' flag words.  A neighbour's
// stream waits for that epoch (cuStreamWaitValue32) before its next boundary
// launch, so no kernel ever spins on another rank.
template <typename T>
struct P2PArgs {
  T* up;                 // up neighbour's buffer of this time level (nullptr: none)
  T* dn;                 // down neighbour's buffer of this time level (nullptr: none)
  unsigned int* counter; // CTA arrival counter (own device memory, 0 between launches)
  unsigned int* flag_up; // my slot in the up neighbour's flag words (nullptr: none)
  unsigned int* flag_dn; // my slot in the down neighbour's flag words
  unsigned int epoch;    // value published when every CTA has stored
  double* rho_up;        // FULL_FD_LAG: up / down neighbour's density field of this time level
  double* rho_dn;        // (nullptr: none)
};

// Own-node store plus the peer copy of the outgoing directions:
//   top plane (z = nz_l - 1), e_z = +1 (q 18..26) -> up neighbour's ghost p = 0
//   bottom plane (z = 0),     e_z = -1 (q 0..8)   -> down neighbour's ghost p = nz_l + 1
// (the pull of the neighbour's plane adjacent to the ghost reads exactly these).
template <typename T>
struct StoreHalo {
  T* base;
  T* out;
  int nxy;
  const Consts* c;
  T* rup;  // up neighbour's ghost plane at this node, or nullptr
  T* rdn;  // down neighbour's ghost plane at this node, or nullptr
  T* up_base;
  T* dn_base;
  double* rho_own = nullptr;  // FULL_FD_LAG: own density field at this node (sum of the stored
  double* rho_up = nullptr;   // values in q order, as StoreOwn) and the neighbours' density
  double* rho_dn = nullptr;   // ghost planes at this node
  double acc = 0.0;
  __device__ __forceinline__ void begin(double) {}
  __device__ __forceinline__ void operator()(int q, double v) {
    stcs<T>(LBM_CHECK_ST(base, out + q * nxy, *c), v);
    if (q >= 18 && rup) stcs<T>(LBM_CHECK_ST(up_base, rup + q * nxy, *c), v);
    if (q < 9 && rdn) stcs<T>(LBM_CHECK_ST(dn_base, rdn + q * nxy, *c), v);
    if (rho_own) {
      acc += (double)(T)v;
      if (q == 26) {
        *rho_own = acc;
        if (rho_up) *rho_up = acc;
        if (rho_dn) *rho_dn = acc;
      }
    }
  }
};

__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Every CTA: barrier, system fence (its peer stores are visible system-wide
// before it arrives), arrive.  The last CTA to arrive resets the counter and
// publishes the epoch (fence-cumulative: all CTAs' stores precede the flag).
template <typename T>
__device__ __forceinline__ void p2p_signal(const P2PArgs<T>& a) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned int total = gridDim.x * gridDim.y;
    if (atomicAdd(a.counter, 1u) == total - 1) {
      atomicExch(a.counter, 0u);
      __threadfence_system();
      if (a.flag_up) st_release_sys(a.flag_up, a.epoch);
      if (a.flag_dn) st_release_sys(a.flag_dn, a.epoch);
    }
  }
}

template <typename T, int KIND, bool FD>
__global__ void LBM_CS_BOUNDS k_collide_stream_p2p(const T* __restrict__ src, T* __restrict__ dst,
                                                   const double* __restrict__ rf, const __grid_constant__ Consts c,
                                                   int zbeg, int zstride, const P2PArgs<T> a) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx < c.nxy) {  // no early return: every thread reaches the barrier of p2p_signal
    const int y = row_of(c, idx);
    const int x = idx - y * c.nx;
    const int z = zbeg + blockIdx.y * zstride;
    double gxr = 0.0, gyr = 0.0, gzr = 0.0;
    if (FD) density_gradient(rf, c, x, y, z, gxr, gyr, gzr);  // ghost-plane rho pushed by the neighbours
    double f[27];
    gather<T>(src, c, x, y, z, f);
    StoreHalo<T> st{dst,
                    dst + (long long)(z + 1) * c.plane + idx,
                    c.nxy,
                    &c,
                    (z == c.nzl - 1 && a.up) ? a.up + idx : nullptr,
                    (z == 0 && a.dn) ? a.dn + (long long)(c.nzl + 1) * c.plane + idx : nullptr,
                    a.up,
                    a.dn,
                    c.rf_out ? c.rf_out + (long long)(z + 1) * c.nxy + idx : nullptr,
                    (c.rf_out && z == c.nzl - 1 && a.rho_up) ? a.rho_up + idx : nullptr,                         // ghost p = 0
                    (c.rf_out && z == 0 && a.rho_dn) ? a.rho_dn + (long long)(c.nzl + 1) * c.nxy + idx : nullptr};
    run_core<KIND, FD>(c, f, gxr, gyr, gzr, st);
  }
  p2p_signal(a);
}

// FULL_FD with the P2P halo: the same-time density (as k_density) of the
// planes the boundary-plane collision reads, planes = {0, 1, nz_l-2, nz_l-1}
// (blockIdx.y indexes the list), the two boundary planes' also stored into
// the neighbours' density ghost planes (a.up / a.dn are the neighbours'
// density fields), then signal.
struct PlaneList {
  int z[4];
};

template <typename T>
__global__ void __launch_bounds__(kBlock) k_density_p2p(const T* __restrict__ src, double* __restrict__ rho_out,
                                                        const __grid_constant__ Consts c, const PlaneList pl,
                                                        const P2PArgs<double> a) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx < c.nxy) {
    const int y = row_of(c, idx);
    const int z = pl.z[blockIdx.y];
    double f[27];
    gather<T>(src, c, idx - y * c.nx, y, z, f);
    double r0 = 0.0;
#pragma unroll
    for (int q = 0; q < 27; ++q) r0 += f[q];
    rho_out[(long long)(z + 1) * c.nxy + idx] = r0;
    if (z == c.nzl - 1 && a.up) a.up[idx] = r0;                                     // up's ghost p = 0
    if (z == 0 && a.dn) a.dn[(long long)(c.nzl + 1) * c.nxy + idx] = r0;           // down's ghost p = nz_l + 1
  }
  p2p_signal(a);
}

// Halo publish without a collision (after init_fields / set_populations): copy
// the outgoing directions of the two boundary planes of `src` into the
// neighbours' ghost planes (blockIdx.y = 0: down, 1: up), then signal.
template <typename T>
__global__ void __launch_bounds__(kBlock) k_halo_push(const T* __restrict__ src, const double* __restrict__ rsrc,
                                                      const __grid_constant__ Consts c, const P2PArgs<T> a) {
  const long long e = (long long)blockIdx.x * kBlock + threadIdx.x;
  if (e < 9LL * c.nxy) {
    if (blockIdx.y == 0 && a.dn)  // bottom plane p = 1, q 0..8 -> ghost p = nz_l + 1
      a.dn[(long long)(c.nzl + 1) * c.plane + e] = src[c.plane + e];
    if (blockIdx.y == 1 && a.up)  // top plane p = nz_l, q 18..26 -> ghost p = 0
      a.up[18LL * c.nxy + e] = src[(long long)c.nzl * c.plane + 18LL * c.nxy + e];
  }
  if (rsrc && e < c.nxy) {  // FULL_FD_LAG: the boundary planes' densities into the neighbours' ghost planes
    if (blockIdx.y == 0 && a.rho_dn) a.rho_dn[(long long)(c.nzl + 1) * c.nxy + e] = rsrc[c.nxy + e];
    if (blockIdx.y == 1 && a.rho_up) a.rho_up[e] = rsrc[(long long)c.nzl * c.nxy + e];
  }
  p2p_signal(a);
}

// FULL_FD_LAG after init_fields / set_populations: the density field of the
// stored state, rho = sum_q f~_q of each node of the planes zbeg + blockIdx.y
template <typename T>
__global__ void __launch_bounds__(kBlock) k_stored_rho(const T* __restrict__ src, double* __restrict__ rf,
                                                       const __grid_constant__ Consts c, int zbeg) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx >= c.nxy) return;
  const int z = zbeg + blockIdx.y;
  const T* p = src + (long long)(z + 1) * c.plane + idx;
  double r0 = 0.0;  // q order, as StoreOwn forms it
#pragma unroll
  for (int q = 0; q < 27; ++q) r0 += ldg(p + q * c.nxy);
  rf[(long long)(z + 1) * c.nxy + idx] = r0;
}

// ------------------------------------ persistent multi-step kernel (small lattices)
// The paper's own grids are small (27k-2M nodes): both population
// buffers then sit in the 126 MB L2 and a step is a few microseconds, so the
// per-launch cost dominates.  One cooperative launch of co-resident CTAs runs
// nsteps time steps; each CTA walks the nodes grid-stride (x fastest: coalesced)
// and a grid-wide barrier separates the steps (and, for FULL_FD, the density
// pass from the collision).  Per node the arithmetic is collide_stream_ab's
// (same gather, core and store), so results are bitwise those of one launch per
// step.  Single GPU, no ghost exchange.
template <typename T, int KIND, bool FD>
__global__ void LBM_CS_BOUNDS k_persistent(T* __restrict__ b0, T* __restrict__ b1, double* __restrict__ rf,
                                           const __grid_constant__ Consts c, int cur, int nsteps) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const long long nodes = (long long)c.nzl * c.nxy;
  const long long stride = (long long)gridDim.x * kBlock;
  const long long first = (long long)blockIdx.x * kBlock + threadIdx.x;
  for (int t = 0; t < nsteps; ++t) {
    const bool odd = ((cur + t) & 1) != 0;
    const T* src = odd ? b1 : b0;
    T* dst = odd ? b0 : b1;
    if (FD) {
      for (long long n = first; n < nodes; n += stride) {
        const int z = int(n / c.nxy);
        const int idx = int(n - (long long)z * c.nxy);
        const int y = row_of(c, idx);
        double f[27];
        gather<T>(src, c, idx - y * c.nx, y, z, f);
        double r0 = 0.0;
#pragma unroll
        for (int q = 0; q < 27; ++q) r0 += f[q];
        rf[(long long)(z + 1) * c.nxy + idx] = r0;
      }
      grid.sync();
    }
    for (long long n = first; n < nodes; n += stride) {
      const int z = int(n / c.nxy);
      const int idx = int(n - (long long)z * c.nxy);
      const int y = row_of(c, idx);
      const int x = idx - y * c.nx;
      double gxr = 0.0, gyr = 0.0, gzr = 0.0;
      if (FD) density_gradient(rf, c, x, y, z, gxr, gyr, gzr);
      double f[27];
      gather<T>(src, c, x, y, z, f);
      StoreOwn<T> st{dst, dst + (long long)(z + 1) * c.plane + idx, c.nxy, &c};
      run_core<KIND, FD>(c, f, gxr, gyr, gzr, st);
    }
    if (t + 1 < nsteps) grid.sync();
  }
}

// ------------------------------------------------ AA in-place streaming (one buffer)
// Layout R: slot 26 - q of node x holds f~_q(x) (post-collision, canonical);
// layout N: slot q of node x holds f_q(x) (pre-collision, already streamed).
//   odd step  (R -> N): gather through the wall rules from layout R (REV slots),
//                       collide, push through the wall rules into layout N;
//   even step (N -> R): load the own slots, collide, store reversed.
// Each memory location is read and written only by the thread of one node, which
// reads all its 27 values before writing any (the pull map is a bijection), so
// the update is race-free in place.  Single-GPU only (no ghost planes).
template <typename T, int KIND, bool ODD>
__global__ void LBM_CS_BOUNDS k_aa(T* buf, const __grid_constant__ Consts c, int zbeg, int zstride) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx >= c.nxy) return;
  const int y = row_of(c, idx);
  const int x = idx - y * c.nx;
  const int z = zbeg + blockIdx.y * zstride;
  double f[27];
  if (ODD) {
    gather<T, true>(buf, c, x, y, z, f);
    StorePush<T> st(buf, c, x, y, z);
    run_core<KIND, false>(c, f, 0.0, 0.0, 0.0, st);
  } else {
    T* p = buf + (long long)(z + 1) * c.plane + idx;
#pragma unroll
    for (int q = 0; q < 27; ++q) f[q] = ldg(LBM_CHECK_LD(buf, p + q * c.nxy, c));
    StoreRev<T> st{buf, p, c.nxy, &c};
    run_core<KIND, false>(c, f, 0.0, 0.0, 0.0, st);
    if (c.aa_lid_rho && y == c.ny - 1) {
      // lid-row node with the moving lid: rho_f = sum of its stored f~ in q order
      // (the sum the two-buffer gather and k_aa_lid_rho form) for the next odd
      // step, read back from this thread's own stores (plain, coherent loads)
      double r0 = 0.0;
#pragma unroll
      for (int q = 0; q < 27; ++q) r0 += (double)p[(26 - q) * c.nxy];
      c.aa_lid_rho[z * c.nx + x] = r0;
    }
  }
}

// Plane-shape specialisation of the AA kernels (paper rates; see
// k_collide_stream_paper_shape): with nx, ny compile-time, a warp of 32 nodes in
// the interior of its row and plane pulls from reversed slots and pushes to
// x + e_q at constant offsets (immediates); other warps take the general code.
template <typename T>
struct StorePushInterior {  // AA odd step, interior node: f~_q(x) -> slot q of node x + e_q
  T* own;                   // slot 0 of the node itself (plane z)
  const Consts* c;
  T* base;
  __device__ __forceinline__ void begin(double) {}
  __device__ __forceinline__ void operator()(int q, double v) const {
    const int i = q % 3, j = (q / 3) % 3, k = q / 9;
    stcs<T>(LBM_CHECK_ST(base, own + ((long long)(k - 1) * c->plane + (q * c->nxy + (j - 1) * c->nx + (i - 1))), *c),
            v);
  }
};

// fp32 storage: 7 resident 128-thread CTAs per SM (the odd kernel 96 -> 72
// registers): 27.1 k vs 25.9 k MLUPS at 512^3 (profiles/r2/aa_minb.jsonl); with
// fp64 the same bound measured 1.4 % slower, so it keeps LBM_MINB
#ifndef LBM_AA_MINB32
#define LBM_AA_MINB32 7
#endif
template <typename T, bool ODD, int SNX, int SNY>
__global__ void __launch_bounds__(kBlock, sizeof(T) == 4 ? LBM_AA_MINB32 : LBM_MINB) k_aa_shape(T* buf, const __grid_constant__ Consts c0, int zbeg, int zstride) {
  Consts c = c0;
  c.nx = SNX;
  c.ny = SNY;
  c.nxy = SNX * SNY;
  c.plane = 27LL * SNX * SNY;
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx >= c.nxy) return;
  const int y = idx / SNX;
  const int x = idx - y * SNX;
  const int z = zbeg + blockIdx.y * zstride;
  if (!ODD) {  // the even step has no neighbour addressing: the general code is already constant-offset
    T* p = buf + (long long)(z + 1) * c.plane + idx;
    double f[27];
#pragma unroll
    for (int q = 0; q < 27; ++q) f[q] = ldg(LBM_CHECK_LD(buf, p + q * c.nxy, c));
    StoreRev<T> st{buf, p, c.nxy, &c};
    run_core<CORE_PAPER, false>(c, f, 0.0, 0.0, 0.0, st);
    if (c.aa_lid_rho && y == c.ny - 1) {
      double r0 = 0.0;
#pragma unroll
      for (int q = 0; q < 27; ++q) r0 += (double)p[(26 - q) * c.nxy];
      c.aa_lid_rho[z * c.nx + x] = r0;
    }
    return;
  }
  const int x0 = x & ~31;
  const bool interior = (SNX % 32 == 0) && x0 > 0 && x0 + 32 < SNX && y > 0 && y < SNY - 1 && z > 0 &&
                        z < c.nzl - 1;
  double f[27];
  if (interior) {
    T* b = buf + (long long)(z + 1) * c.plane + idx;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int q = LBM_Q(i, j, k);
          f[q] = ldg(LBM_CHECK_LD(buf, b + ((long long)(1 - k) * c.plane + ((26 - q) * c.nxy + (1 - j) * SNX + (1 - i))), c));
        }
    StorePushInterior<T> st{b, &c, buf};
    run_core<CORE_PAPER, false>(c, f, 0.0, 0.0, 0.0, st);
  } else {
    gather<T, true>(buf, c, x, y, z, f);
    StorePush<T> st(buf, c, x, y, z);
    run_core<CORE_PAPER, false>(c, f, 0.0, 0.0, 0.0, st);
  }
}

// AA with the moving lid, after init_fields / set_populations (layout R): the
// density sum f~ of every lid-row node for the first odd step (see gather<REV>).
template <typename T>
__global__ void __launch_bounds__(kBlock) k_aa_lid_rho(const T* __restrict__ buf, const __grid_constant__ Consts c) {
  const int x = blockIdx.x * kBlock + threadIdx.x;
  if (x >= c.nx) return;
  const int z = blockIdx.y;
  const T* p = buf + (long long)(z + 1) * c.plane + (c.ny - 1) * c.nx + x;
  double r0 = 0.0;  // sum f~_q in q order (layout R: slot 26 - q), as StoreRev forms it
#pragma unroll
  for (int q = 0; q < 27; ++q) r0 += ldg(p + (26 - q) * c.nxy);
  c.aa_lid_rho[z * c.nx + x] = r0;
}

// Canonical post-collision populations f~_q(x) of node x from an AA buffer:
// phase R: slot 26 - q; phase N: the slot the push wrote (minus the Eq. 69 term
// on lid links; the nine lid terms sum to zero, so rho_f = sum of the values).
template <typename T>
__device__ __forceinline__ void aa_canonical(const T* buf, const Consts& c, int x, int y, int z, int phase,
                                             double (&f)[27]) {
  if (phase == 1) {
    const T* p = buf + (long long)(z + 1) * c.plane + y * c.nx + x;
#pragma unroll
    for (int q = 0; q < 27; ++q) f[q] = ldg(p + (26 - q) * c.nxy);
    return;
  }
  StorePush<T> d(const_cast<T*>(buf), c, x, y, z);
  double rho_f = 0.0;
  bool lid[27];
#pragma unroll
  for (int q = 0; q < 27; ++q) {
    const int i = q % 3, j = (q / 3) % 3, k = q / 9;
    const T* a;
    lid[q] = false;
    if (!d.wall) {
      a = d.pz[k] + q * c.nxy + d.dy[j] + d.dx[i];
    } else {
      const int kx = d.cx[i], ky = d.cy[j], kz = d.cz[k];
      const bool noslip = (kx == FK_BOUNCE || kx == FK_MOVING) || (ky == FK_BOUNCE || ky == FK_MOVING) ||
                          (kz == FK_BOUNCE || kz == FK_MOVING);
      if (noslip) {
        a = d.pz[1] + (26 - q) * c.nxy + d.own;
        lid[q] = (ky == FK_MOVING);
      } else {
        const bool mx = (kx == FK_SLIP), my = (ky == FK_SLIP), mz = (kz == FK_SLIP);
        const int qi = mx ? 2 - i : i, qj = my ? 2 - j : j, qk = mz ? 2 - k : k;
        a = (mz ? d.pz[1] : d.pz[k]) + LBM_Q(qi, qj, qk) * c.nxy + (my ? y * c.nx : d.dy[j]) + (mx ? x : d.dx[i]);
      }
    }
    f[q] = ldg(a);
    rho_f += f[q];
  }
#pragma unroll
  for (int q = 0; q < 27; ++q)
    if (lid[q]) f[q] -= rho_f * c.lid_u * (double)(1 - q % 3) * c.lid_c[2 - q / 9];
}

// -------------------------------------------------------------- init kernel
// f~ = f^eq(rho, u + F/(2 rho)) (reading R8).  The raw equilibria of Eq. 10
// factorise per axis into 1D Maxwellian moments (1, u, cs2 + u^2), so
// f^eq_a = rho phi_x(e_x) phi_y(e_y) phi_z(e_z) with
// phi(0) = 1 - (cs2 + u^2)/c^2, phi(+-1) = ((cs2 + u^2)/c^2 +- u/c)/2.
__device__ __forceinline__ void axis_phi(double u, double c, double cs2, double (&p)[3]) {
  const double a = (cs2 + u * u) / (c * c);
  const double b = u / c;
  p[0] = 0.5 * (a - b);
  p[1] = 1.0 - a;
  p[2] = 0.5 * (a + b);
}

template <typename T>
__global__ void __launch_bounds__(kBlock) k_init(const double* __restrict__ rho_in, const double* __restrict__ u_in,
                                                 long long ustride, T* __restrict__ dst,
                                                 const __grid_constant__ Consts c, int zbeg, int rev) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx >= c.nxy) return;
  const long long n = (long long)blockIdx.y * c.nxy + idx;
  const double rho = rho_in[n];
  const double ux = u_in[n] + 0.5 * c.F[0] / rho;
  const double uy = u_in[n + ustride] + 0.5 * c.F[1] / rho;
  const double uz = u_in[n + 2 * ustride] + 0.5 * c.F[2] / rho;
  double px[3], py[3], pz[3];
  axis_phi(ux, 1.0, c.cs2, px);
  axis_phi(uy, c.r, c.cs2, py);
  axis_phi(uz, c.s, c.cs2, pz);
  T* out = dst + (long long)(zbeg + blockIdx.y + 1) * c.plane + idx;
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int q = LBM_Q(i, j, k);
        stcs<T>(out + (rev ? 26 - q : q) * c.nxy, rho * px[i] * py[j] * pz[k]);
      }
}

// -------------------------------------------------------- macroscopic kernel
// rho = sum f~, u = (sum f~ e - F/2)/rho of the stored post-collision state.
// aa: 0 two-buffer layout, 1 AA phase R, 2 AA phase N (see aa_canonical)
template <typename T>
__device__ __forceinline__ void load_canonical(const T* src, const Consts& c, int idx, int z, int aa,
                                               double (&f)[27]) {
  if (aa == 0) {
    const T* p = src + (long long)(z + 1) * c.plane + idx;
#pragma unroll
    for (int q = 0; q < 27; ++q) f[q] = ldg(p + q * c.nxy);
  } else {
    const int y = row_of(c, idx);
    aa_canonical<T>(src, c, idx - y * c.nx, y, z, aa == 1 ? 1 : 2, f);
  }
}

template <typename T>
__global__ void __launch_bounds__(kBlock) k_macro(const T* __restrict__ src, double* __restrict__ rho_out,
                                                  double* __restrict__ u_out, long long ustride,
                                                  const __grid_constant__ Consts c, int zbeg, int aa) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx >= c.nxy) return;
  double f[27];
  load_canonical<T>(src, c, idx, zbeg + blockIdx.y, aa, f);
  double rho = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double v = f[LBM_Q(i, j, k)];
        rho += v;
        jx += (double)(i - 1) * v;
        jy += (double)(j - 1) * v;
        jz += (double)(k - 1) * v;
      }
  const long long n = (long long)blockIdx.y * c.nxy + idx;
  const double inv = 1.0 / rho;
  rho_out[n] = rho;
  u_out[n] = (jx - 0.5 * c.F[0]) * inv;
  u_out[n + ustride] = (c.r * jy - 0.5 * c.F[1]) * inv;
  u_out[n + 2 * ustride] = (c.s * jz - 0.5 * c.F[2]) * inv;
}

// ---------------------------------------------------------- pack / unpack
// Paper direction order (Eqs. 1a-1c) <-> internal order; staging layout
// [27][nplanes][nxy] in the paper order.
__constant__ int8_t kPaperToInternal[27] = {
    // paper a: (ex,ey,ez) -> (ex+1) + 3(ey+1) + 9(ez+1)
    13, 14, 12, 16, 10, 22, 4, 17, 15, 11, 9, 23, 21, 5, 3, 25, 19, 7, 1, 26, 24, 20, 18, 8, 6, 2, 0};

template <typename T>
__global__ void __launch_bounds__(kBlock) k_pack(const T* __restrict__ src, double* __restrict__ stage, int nplanes,
                                                 const __grid_constant__ Consts c, int zbeg, int aa) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx >= c.nxy) return;
  const int zz = blockIdx.y;
  double f[27];
  load_canonical<T>(src, c, idx, zbeg + zz, aa, f);
  for (int a = 0; a < 27; ++a) stage[((long long)a * nplanes + zz) * c.nxy + idx] = f[kPaperToInternal[a]];
}

template <typename T>
__global__ void __launch_bounds__(kBlock) k_unpack(const double* __restrict__ stage, T* __restrict__ dst, int nplanes,
                                                   const __grid_constant__ Consts c, int zbeg, int rev) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx >= c.nxy) return;
  const int zz = blockIdx.y;
  T* p = dst + (long long)(zbeg + zz + 1) * c.plane + idx;
  for (int a = 0; a < 27; ++a) {
    const int q = kPaperToInternal[a];
    p[(rev ? 26 - q : q) * c.nxy] = (T)stage[((long long)a * nplanes + zz) * c.nxy + idx];
  }
}

// -------------------------------------------------------------- check kernel
// out[0] sum rho, out[1..3] sum rho u, out[4] sum rho|u|^2/2, out[5] max|u| (as
// ordered bits of a non-negative double), out[6] count of bad nodes.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic two-kernel reduction: every CTA of a grid-stride pass writes its
// seven partials; one CTA then reduces them in a fixed order (no atomics: the
// sums do not depend on scheduling).
constexpr int kCheckThreads = 256;
constexpr int kCheckMaxBlocks = 2048;

template <typename T>
__global__ void __launch_bounds__(kCheckThreads) k_check(const T* __restrict__ src, double* __restrict__ partial,
                                                         const __grid_constant__ Consts c, int aa) {
  const long long nodes = (long long)c.nzl * c.nxy;
  double v[7] = {0, 0, 0, 0, 0, 0, 0};
  for (long long n = (long long)blockIdx.x * kCheckThreads + threadIdx.x; n < nodes;
       n += (long long)gridDim.x * kCheckThreads) {
    const int z = int(n / c.nxy);
    const int idx = int(n - (long long)z * c.nxy);
    double fq[27];
    load_canonical<T>(src, c, idx, z, aa, fq);
    double rho = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
#pragma unroll
    for (int q = 0; q < 27; ++q) {
      const double fv = fq[q];
      const int i = q % 3, j = (q / 3) % 3, k = q / 9;
      rho += fv;
      jx += (i - 1) * fv;
      jy += (j - 1) * fv;
      jz += (k - 1) * fv;
    }
    const double ux = (jx - 0.5 * c.F[0]) / rho, uy = (c.r * jy - 0.5 * c.F[1]) / rho,
                 uz = (c.s * jz - 0.5 * c.F[2]) / rho;
    const double u2 = ux * ux + uy * uy + uz * uz;
    const bool bad = !(rho > 0.0) || !(u2 <= 1.0) || !isfinite(rho) || !isfinite(u2);
    v[0] += rho;
    v[1] += rho * ux;
    v[2] += rho * uy;
    v[3] += rho * uz;
    v[4] += 0.5 * rho * u2;
    v[5] = bad ? v[5] : fmax(v[5], sqrt(u2));
    v[6] += bad ? 1.0 : 0.0;
  }
  __shared__ double sm[7][kCheckThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < 7; ++t) {
    const double r = (t == 5) ? warp_max(v[t]) : warp_sum(v[t]);
    if (lane == 0) sm[t][w] = r;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    const int t = threadIdx.x;
    double r = sm[t][0];
    for (int i = 1; i < kCheckThreads / 32; ++i) r = (t == 5) ? fmax(r, sm[t][i]) : r + sm[t][i];
    partial[(long long)blockIdx.x * 8 + t] = r;
  }
}

__global__ void __launch_bounds__(kCheckThreads) k_check_final(const double* __restrict__ partial, int nblocks,
                                                               double* __restrict__ out) {
  double v[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < nblocks; b += kCheckThreads)
#pragma unroll
    for (int t = 0; t < 7; ++t) v[t] = (t == 5) ? fmax(v[t], partial[b * 8 + t]) : v[t] + partial[b * 8 + t];
  __shared__ double sm[7][kCheckThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < 7; ++t) {
    const double r = (t == 5) ? warp_max(v[t]) : warp_sum(v[t]);
    if (lane == 0) sm[t][w] = r;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    const int t = threadIdx.x;
    double r = sm[t][0];
    for (int i = 1; i < kCheckThreads / 32; ++i) r = (t == 5) ? fmax(r, sm[t][i]) : r + sm[t][i];
    out[t] = r;
  }
}



}  // namespace lbm
