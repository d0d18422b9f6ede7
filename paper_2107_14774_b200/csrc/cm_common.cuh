// cm_common.cuh -- shared definitions of the sm_100a kernels of the 3D cuboid
// central-moment LBM (arXiv 2107.14774): build-time knobs, the per-launch
// parameter block, bounds-check macros and the memory-access helpers.
// "P:Lnnn" cites /root/reference/PAPER.md line nnn.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lbm {


#ifndef LBM_BLOCK
#define LBM_BLOCK 128
#endif
#ifndef LBM_MINB
#define LBM_MINB 0  // min resident blocks per SM for __launch_bounds__ (0: none)
#endif
#ifndef LBM_LDMODE
#define LBM_LDMODE 0  // 0: ld.global.nc; 1: ld.global.nc.L1::no_allocate
#endif
#ifndef LBM_STMODE
#define LBM_STMODE 0  // 0: st.global.cs (evict-first); 1: plain st.global
#endif
constexpr int kBlock = LBM_BLOCK;  // threads per block (one node per thread)

// local face treatment (per rank; z faces depend on the slab position)
enum FaceKind : int {
  FK_WRAP = 0,        // periodic, wrapped inside the kernel
  FK_BOUNCE = 1,      // halfway bounce-back (P:L748-749 with U = 0)
  FK_MOVING = 2,      // Eq. 69 moving wall (+y only)
  FK_SLIP = 3,        // free-slip (reading R7)
  FK_GHOST = 4        // neighbour data in a ghost plane (z faces only)
};

struct Consts {
  int nx, ny, nzl, nxy;
  long long plane;      // 27 * nxy elements
  int face[6];          // FaceKind per local face -x,+x,-y,+y,-z,+z
  int has_walls;        // any face is BOUNCE/MOVING/SLIP
  int has_slip;         // any face is SLIP
  int corr_on;          // corrections != OFF
  double r, s, cs2;
  double h1y, h2y, h1z, h2z;  // 1/(2r), 1/(2r^2), 1/(2s), 1/(2s^2)
  double r2, s2;
  double wn, wx, w1, wh;      // omega_nu, omega_xi, omega_1, omega_high
  double an, ab;              // 1/omega_nu - 1/2, 1/omega_xi - 1/2
  double gx, gy, gz;          // 3cs2 - 1, 3cs2 - r^2, 3cs2 - s^2
  double galias;              // 1 (FULL_LOCAL: 3u^2 aliasing terms) or 0 (LOW_MACH)
  double csn, csx;            // 2 cs2/omega_nu, 2 cs2/omega_xi
  double F[3];
  double c4, c6;              // cs2^2, cs2^3
  double lid_u;               // moving-wall speed U
  double lid_c[3];            // Eq. 69 coefficient per e_z in {-1,0,1}: cs2/(2 r^2) * phi_z(e_z)
  double phx[3], phy[3], phz[3];  // cuboid rest weights per axis: phi(0) = 1 - cs2/c^2, phi(+-1) = cs2/(2c^2)
  long long buf_elems;        // elements of one population buffer (bounds checks)
  unsigned int nx_mul;        // fast division by nx (row of a plane index): see row_of()
  int nx_shift;
  unsigned int* dbg_flag;     // LBM_DEBUG_BOUNDS builds: set to 1 on an out-of-range access
  unsigned int* sing_flag;    // set to 1 when a node's strain-rate system is singular (reading R17)
  double sing_thr;            // 1e-12 cs2: threshold of the singular predicate on C/rho
  double* aa_lid_rho;         // AA with the moving lid: rho of the lid-row nodes [z][x] (see k_aa)
  double* rf_out;             // FULL_FD_LAG: density field the collision writes (the next step's gradient)
};

// Singular strain-rate system (reading R17): the closed-form
// denominators of P:L1199-1203 -- D, the determinant in the printed d_x u_x, and
// C_sy, C_sz of the back-substitution -- below 1e-12 rho cs2 in magnitude.  The
// kernels hold C/rho, so D = rho^3 det and C = rho (C/rho).  Rare: one flag word.
__device__ __forceinline__ void note_singular(const Consts& c, double det, double Csy, double Csz, double rho) {
  if (fabs(det) * (rho * rho) < c.sing_thr || fabs(Csy) < c.sing_thr || fabs(Csz) < c.sing_thr)
    atomicOr(c.sing_flag, 1u);
}

// Row y = idx / nx of a plane index idx < 2^31 by multiply-high and shift
// (round-up reciprocal, exact for 31-bit dividends; host side: fill_consts).
__device__ __forceinline__ int row_of(const Consts& c, int idx) {
  return c.nx_mul ? int(__umulhi((unsigned)idx, c.nx_mul) >> c.nx_shift) : idx;
}

// Debug builds (-DLBM_DEBUG_BOUNDS): every population access of the collide-stream
// kernels is checked against the buffer; a violation sets *dbg_flag and is skipped.
#ifdef LBM_DEBUG_BOUNDS
#define LBM_CHECK_LD(base, p, c)                                                          \
  (((unsigned long long)((p) - (base)) < (unsigned long long)(c).buf_elems)              \
       ? (p)                                                                              \
       : (atomicOr((c).dbg_flag, 1u), (base)))
#define LBM_CHECK_ST(base, p, c) LBM_CHECK_LD(base, p, c)
#else
#define LBM_CHECK_LD(base, p, c) (p)
#define LBM_CHECK_ST(base, p, c) (p)
#endif

// ------------------------------------------------------------------ memory ops
template <typename T> __device__ __forceinline__ double ldg(const T* p);
#if LBM_LDMODE == 1
template <> __device__ __forceinline__ double ldg<double>(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ double ldg<float>(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return (double)v;
}
#else
template <> __device__ __forceinline__ double ldg<double>(const double* p) { return __ldg(p); }
template <> __device__ __forceinline__ double ldg<float>(const float* p) { return (double)__ldg(p); }
#endif

template <typename T> __device__ __forceinline__ void stcs(T* p, double v);
#if LBM_STMODE == 1
template <> __device__ __forceinline__ void stcs<double>(double* p, double v) { *p = v; }
template <> __device__ __forceinline__ void stcs<float>(float* p, double v) { *p = (float)v; }
#else
template <> __device__ __forceinline__ void stcs<double>(double* p, double v) { __stcs(p, v); }
template <> __device__ __forceinline__ void stcs<float>(float* p, double v) { __stcs(p, (float)v); }
#endif

#define LBM_Q(i, j, k) ((i) + 3 * (j) + 9 * (k))


}  // namespace lbm
