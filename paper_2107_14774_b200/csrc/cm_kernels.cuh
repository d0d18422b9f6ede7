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
#pragma once

#include <cooperative_groups.h>
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
};

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

// ------------------------------------------------------- per-axis transforms
// Axis strides in the 3x3x3 slot cube: x -> 1, y -> 3, z -> 9.  A "triple" is
// the three slots along one axis with the other two indices fixed.
template <int AX> struct Axis;
template <> struct Axis<0> { static constexpr int st = 1, o1 = 3, o2 = 9; };
template <> struct Axis<1> { static constexpr int st = 3, o1 = 1, o2 = 9; };
template <> struct Axis<2> { static constexpr int st = 9, o1 = 1, o2 = 3; };

// raw moments along one axis, cubic units: (f-, f0, f+) -> (m0, m1, m2)   [App A]
template <int AX>
__device__ __forceinline__ void raw_pass(double (&f)[27]) {
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int q = a * Axis<AX>::o1 + b * Axis<AX>::o2;
      const double fm = f[q], f0 = f[q + Axis<AX>::st], fp = f[q + 2 * Axis<AX>::st];
      const double sp = fp + fm;
      f[q] = sp + f0;
      f[q + Axis<AX>::st] = fp - fm;
      f[q + 2 * Axis<AX>::st] = sp;
    }
}

// scale by the axis speed c (App B, S) and shift to the central frame (App C, F):
// (m0, m1, m2) -> (m0, c m1 - u m0, c^2 m2 - 2 u c m1 + u^2 m0)
template <int AX, bool UNIT>
__device__ __forceinline__ void central_pass(double (&f)[27], double u, double c, double c2) {
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int q = a * Axis<AX>::o1 + b * Axis<AX>::o2;
      const double m0 = f[q];
      const double m1 = UNIT ? f[q + Axis<AX>::st] : c * f[q + Axis<AX>::st];
      const double m2 = UNIT ? f[q + 2 * Axis<AX>::st] : c2 * f[q + 2 * Axis<AX>::st];
      const double k1 = fma(-u, m0, m1);
      f[q + Axis<AX>::st] = k1;
      f[q + 2 * Axis<AX>::st] = fma(-u, m1 + k1, m2);
    }
}

// central -> raw (App E, F^-1 = F(-u)), unscale (App F, S^-1) and back to the
// three populations along the axis (App G, P^-1), with h1 = 1/(2c), h2 = 1/(2c^2):
// A = k1 + u k0, B = k2 + 2u k1 + u^2 k0;  f0 = k0 - B/c^2, f+- = (B/c^2 +- A/c)/2
template <int AX>
__device__ __forceinline__ void inverse_pass(double (&f)[27], double u, double h1, double h2) {
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int q = a * Axis<AX>::o1 + b * Axis<AX>::o2;
      const double k0 = f[q], k1 = f[q + Axis<AX>::st], k2 = f[q + 2 * Axis<AX>::st];
      const double A = fma(u, k0, k1);
      const double B = fma(u, k1 + A, k2);
      const double t1 = A * h1, t2 = B * h2;
      f[q] = t2 - t1;
      f[q + Axis<AX>::st] = fma(-2.0, t2, k0);
      f[q + 2 * Axis<AX>::st] = t2 + t1;
    }
}

// ---------------------------------------------------------------- collision
// App D on the central moments held in slots K(i,j,k) = f[i+3j+9k].
// Local strain rates are solved with Cramer's rule on the
// system divided by rho (one reciprocal); lambda = e_rho = 0 (reading R1).
template <bool FD = false>
__device__ __forceinline__ void second_order_diag(const Consts& c, double rho, double inv_rho,
                                                  double ux, double uy, double uz,
                                                  double k200, double k020, double k002,
                                                  double& o200, double& o020, double& o002,
                                                  double gxr = 0.0, double gyr = 0.0, double gzr = 0.0) {
  const double k2s = k200 + k020 + k002;  // B
  const double k2d1 = k200 - k020;
  const double k2d2 = k200 - k002;
  const double c3r = 3.0 * c.cs2 * rho;
  double e2s = c3r, e2d1 = 0.0, e2d2 = 0.0;
  if (c.corr_on) {
    const double ga = 1.5 * c.galias;
    const double qx = ga * ux * ux, qy = ga * uy * uy, qz = ga * uz * uz;
    // C coefficients / rho
    const double Csx = -c.csn + 0.5 * c.gx + qx;
    const double Cbx = -c.csx + 0.5 * c.gx + qx;
    const double Csy = c.csn - 0.5 * c.gy - qy;
    const double Cby = -c.csx + 0.5 * c.gy + qy;
    const double Csz = c.csn - 0.5 * c.gz - qz;
    const double Cbz = -c.csx + 0.5 * c.gz + qz;
    // R / rho; e_rho terms only with FD (reading R1)
    double Rb = (k2s - c3r) * inv_rho, Rs1 = k2d1 * inv_rho, Rs2 = k2d2 * inv_rho;
    double lsx = 0.0, lsy = 0.0, lsz = 0.0;  // A d_x rho, B d_y rho, C d_z rho
    if (FD) {
      lsx = 0.5 * c.gx * ux * gxr;
      lsy = 0.5 * c.gy * uy * gyr;
      lsz = 0.5 * c.gz * uz * gzr;
      Rb += (-lsx - lsy - lsz) * inv_rho;
      Rs1 += (-lsx + lsy) * inv_rho;
      Rs2 += (-lsx + lsz) * inv_rho;
    }
    const double t1 = Csx * Cbz - Csz * Cbx;
    const double det = -Csx * Csz * Cby - Csy * t1;
    const double inv_det = 1.0 / det;
    const double dxux = (-Csz * Cby * Rs1 - Csy * (Cbz * Rs2 - Csz * Rb)) * inv_det;
    const double dyuy = (Csx * (Rs2 * Cbz - Csz * Rb) - Rs1 * t1) * inv_det;
    const double dzuz = (Csx * Cby * (Rs1 - Rs2) - Csy * (Csx * Rb - Rs2 * Cbx)) * inv_det;
    // theta / (-rho (1/omega - 1/2)) times the strain rates
    const double tx = (2.0 * qx + c.gx) * dxux;
    const double ty = (2.0 * qy + c.gy) * dyuy;
    const double tz = (2.0 * qz + c.gz) * dzuz;
    const double rn = rho * c.an, rb = rho * c.ab;
    e2d1 = -rn * (tx - ty);          // Eq. 63
    e2d2 = -rn * (tx - tz);          // Eq. 63
    e2s = c3r - rb * (tx + ty + tz); // Eq. 63
    if (FD) {
      // lambda_s x = -2 a_n A, lambda_s y = +2 a_n B, ..., times the gradients
      e2d1 += 2.0 * c.an * (-lsx + lsy);
      e2d2 += 2.0 * c.an * (-lsx + lsz);
      e2s += 2.0 * c.ab * (-lsx - lsy - lsz);
    }
  }
  const double s2s = fma(c.wx, e2s - k2s, k2s);
  const double s2d1 = fma(c.wn, e2d1 - k2d1, k2d1);
  const double s2d2 = fma(c.wn, e2d2 - k2d2, k2d2);
  const double third = 1.0 / 3.0;  // B^-1
  o200 = (s2s + s2d1 + s2d2) * third;
  o020 = (s2s - 2.0 * s2d1 + s2d2) * third;
  o002 = (s2s + s2d1 - 2.0 * s2d2) * third;
}

// Generic relaxation (any omega_1, omega_high): all 27 central moments are in f.
template <bool FD>
__device__ __forceinline__ void collide_generic(const Consts& c, double (&f)[27], double rho,
                                                double inv_rho, double ux, double uy, double uz,
                                                double gxr, double gyr, double gzr) {
#define K(i, j, k) f[LBM_Q(i, j, k)]
  const double w1 = c.w1, wn = c.wn, wh = c.wh;
  // first order: k~ = k + w1 (0 - k) + (1 - w1/2) F
  K(1, 0, 0) = fma(1.0 - w1, K(1, 0, 0), (1.0 - 0.5 * w1) * c.F[0]);
  K(0, 1, 0) = fma(1.0 - w1, K(0, 1, 0), (1.0 - 0.5 * w1) * c.F[1]);
  K(0, 0, 1) = fma(1.0 - w1, K(0, 0, 1), (1.0 - 0.5 * w1) * c.F[2]);
  // off-diagonal second order
  K(1, 1, 0) *= (1.0 - wn);
  K(1, 0, 1) *= (1.0 - wn);
  K(0, 1, 1) *= (1.0 - wn);
  double o200, o020, o002;
  second_order_diag<FD>(c, rho, inv_rho, ux, uy, uz, K(2, 0, 0), K(0, 2, 0), K(0, 0, 2), o200, o020, o002, gxr,
                        gyr, gzr);
  K(2, 0, 0) = o200;
  K(0, 2, 0) = o020;
  K(0, 0, 2) = o002;
  // third and higher orders: every B group has one rate, so B^-1 Lambda B acts
  // as omega_high on each moment; equilibria of Eq. 64
  const double om = 1.0 - wh;
  K(1, 2, 0) *= om; K(1, 0, 2) *= om; K(2, 1, 0) *= om;
  K(0, 1, 2) *= om; K(2, 0, 1) *= om; K(0, 2, 1) *= om;
  K(1, 1, 1) *= om;
  K(2, 1, 1) *= om; K(1, 2, 1) *= om; K(1, 1, 2) *= om;
  K(1, 2, 2) *= om; K(2, 1, 2) *= om; K(2, 2, 1) *= om;
  const double e4 = wh * c.c4 * rho;
  K(2, 2, 0) = fma(om, K(2, 2, 0), e4);
  K(2, 0, 2) = fma(om, K(2, 0, 2), e4);
  K(0, 2, 2) = fma(om, K(0, 2, 2), e4);
  K(2, 2, 2) = fma(om, K(2, 2, 2), wh * c.c6 * rho);
#undef K
}

// -------------------------------------------------------------- streaming
// Gather the 27 incoming populations of node (x, y, z) (pull form).
// Fast path: no wall face adjacent -> periodic/ghost addressing only.
// Pull sources of node (x, y, z): x/y neighbour indices with periodic wrap,
// the three source planes (ghost planes at -1 / nz_l unless z wraps), and
// whether a wall face is adjacent (then gather() applies the wall rules).
template <typename T>
struct PullSrc {
  int sx[3], sy[3];  // source x, y*nx for displacement e + 1 (source = node - e)
  const T* pz[3];    // source plane for e_z + 1
  bool wall;
  __device__ __forceinline__ PullSrc(const T* src, const Consts& c, int x, int y, int z) {
    const int nx = c.nx;
    const int xm = (x == 0) ? nx - 1 : x - 1;        // source of e_x = +1
    const int xp = (x == nx - 1) ? 0 : x + 1;        // source of e_x = -1
    const int ym = (y == 0) ? c.ny - 1 : y - 1;
    const int yp = (y == c.ny - 1) ? 0 : y + 1;
    int zm = z - 1, zp = z + 1;                      // -1 / nz_l address ghost planes
    if (z == 0 && c.face[4] == FK_WRAP) zm = c.nzl - 1;
    if (z == c.nzl - 1 && c.face[5] == FK_WRAP) zp = 0;
    sx[0] = xp; sx[1] = x; sx[2] = xm;
    sy[0] = yp * nx; sy[1] = y * nx; sy[2] = ym * nx;
    pz[0] = src + (long long)(zp + 1) * c.plane;
    pz[1] = src + (long long)(z + 1) * c.plane;
    pz[2] = src + (long long)(zm + 1) * c.plane;
    wall = false;
    if (c.has_walls) {
      wall = (x == 0 && c.face[0] >= FK_BOUNCE && c.face[0] <= FK_SLIP) ||
             (x == nx - 1 && c.face[1] >= FK_BOUNCE && c.face[1] <= FK_SLIP) ||
             (y == 0 && c.face[2] >= FK_BOUNCE && c.face[2] <= FK_SLIP) ||
             (y == c.ny - 1 && c.face[3] >= FK_BOUNCE && c.face[3] <= FK_SLIP) ||
             (z == 0 && c.face[4] >= FK_BOUNCE && c.face[4] <= FK_SLIP) ||
             (z == c.nzl - 1 && c.face[5] >= FK_BOUNCE && c.face[5] <= FK_SLIP);
    }
  }
};

// REV (AA odd steps): the source buffer holds f~_s(z) at slot 26 - s of node z.
template <typename T, bool REV = false>
__device__ __forceinline__ void gather(const T* src, const Consts& c, int x, int y, int z, double (&f)[27]) {
  auto slot = [](int s) { return REV ? 26 - s : s; };
  const int nx = c.nx;
  const PullSrc<T> ps(src, c, x, y, z);
  const int* sx = ps.sx;
  const int* sy = ps.sy;
  const T* const* pz = ps.pz;
  // warp-uniform choice: a warp with any wall-adjacent lane takes the wall path
  // (which reduces to the plain pull for its other lanes) instead of running
  // both paths one after the other
  const unsigned mask = __activemask();
  const bool wall = __any_sync(mask, ps.wall);
  // no lane of the warp wraps around a periodic face: every source is the own
  // node's address plus an offset that is the same for the whole warp
  // ((-e_z) plane + slot nxy - e_y nx - e_x), so the 27 addresses need no
  // per-lane index arithmetic (ghost planes included)
  const bool lane_inner = (x > 0 && x < nx - 1 && y > 0 && y < c.ny - 1 &&
                           !(z == 0 && c.face[4] == FK_WRAP) && !(z == c.nzl - 1 && c.face[5] == FK_WRAP));
  if (!wall && __all_sync(mask, lane_inner)) {
    const T* b = src + (long long)(z + 1) * c.plane + (y * nx + x);
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int q = LBM_Q(i, j, k);
          const long long off = (long long)(1 - k) * c.plane + (long long)(slot(q) * c.nxy + (1 - j) * nx + (1 - i));
          f[q] = ldg(LBM_CHECK_LD(src, b + off, c));
        }
    return;
  }
  if (!wall) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int q = LBM_Q(i, j, k);
          f[q] = ldg(LBM_CHECK_LD(src, pz[k] + slot(q) * c.nxy + sy[j] + sx[i], c));
        }
    return;
  }
  // Wall-adjacent node.  Crossing kind of the source of displacement e per axis:
  // 0 none (inside, periodic or ghost), 1 no-slip, 2 moving wall, 3 free-slip.
  auto kind = [](int fk) { return (fk >= FK_BOUNCE && fk <= FK_SLIP) ? fk : 0; };
  const int cxp = (x == 0) ? kind(c.face[0]) : 0, cxm = (x == nx - 1) ? kind(c.face[1]) : 0;
  const int cyp = (y == 0) ? kind(c.face[2]) : 0, cym = (y == c.ny - 1) ? kind(c.face[3]) : 0;
  const int czp = (z == 0) ? kind(c.face[4]) : 0, czm = (z == c.nzl - 1) ? kind(c.face[5]) : 0;
  const int own = y * nx + x;
  const T* p0 = pz[1];
  double rho_f = 0.0;  // reading R4: rho_f = sum_b f~_b(x_f, t) at the wall-adjacent node
  if (cym == FK_MOVING) {
#pragma unroll
    for (int q = 0; q < 27; ++q) rho_f += ldg(LBM_CHECK_LD(src, p0 + q * c.nxy + own, c));
  }
  if (!c.has_slip) {
    // no free-slip face (uniform branch): per direction either the plain pull or
    // the halfway bounce-back source (+ the Eq. 69 term across the lid)
    const bool nx0 = cxm != 0, nx2 = cxp != 0, ny0 = cym != 0, ny2 = cyp != 0, nz0 = czm != 0, nz2 = czp != 0;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int q = LBM_Q(i, j, k);
          const bool noslip = (i == 0 ? nx0 : (i == 2 ? nx2 : false)) || (j == 0 ? ny0 : (j == 2 ? ny2 : false)) ||
                              (k == 0 ? nz0 : (k == 2 ? nz2 : false));
          const T* a_plain = pz[k] + slot(q) * c.nxy + sy[j] + sx[i];
          const T* a_bb = p0 + slot(LBM_Q(2 - i, 2 - j, 2 - k)) * c.nxy + own;
          double v = ldg(LBM_CHECK_LD(src, noslip ? a_bb : a_plain, c));
          if (j == 0 && cym == FK_MOVING)  // e_y = -1 crosses the +y lid: Eq. 69
            v = fma(rho_f * c.lid_u * (double)(i - 1), c.lid_c[k], v);
          f[q] = v;
        }
    return;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int q = LBM_Q(i, j, k);
        const int ex = i - 1, ey = j - 1, ez = k - 1;
        const int kx = ex > 0 ? cxp : (ex < 0 ? cxm : 0);
        const int ky = ey > 0 ? cyp : (ey < 0 ? cym : 0);
        const int kz = ez > 0 ? czp : (ez < 0 ? czm : 0);
        const bool noslip = (kx == FK_BOUNCE || kx == FK_MOVING) || (ky == FK_BOUNCE || ky == FK_MOVING) ||
                            (kz == FK_BOUNCE || kz == FK_MOVING);
        // one load per direction, its source chosen per lane:
        //  no-slip crossing: halfway bounce-back from the own node's opposite
        //    direction, plus the Eq. 69 term across the lid;
        //  free-slip crossing (reading R7): the crossed axes mirrored, source at
        //    the own coordinate along them;
        //  otherwise the periodic/ghost neighbour
        const bool mx = (kx == FK_SLIP), my = (ky == FK_SLIP), mz = (kz == FK_SLIP);
        const int qi = mx ? 2 - i : i, qj = my ? 2 - j : j, qk = mz ? 2 - k : k;
        const int xs = mx ? x : sx[i];
        const int ys = my ? y * nx : sy[j];
        const T* zs = mz ? p0 : pz[k];
        const T* a_slip = zs + slot(LBM_Q(qi, qj, qk)) * c.nxy + ys + xs;
        const T* a_bb = p0 + slot(LBM_Q(2 - i, 2 - j, 2 - k)) * c.nxy + own;
        double v = ldg(LBM_CHECK_LD(src, noslip ? a_bb : a_slip, c));
        if (ky == FK_MOVING)  // Eq. 69: + rho_f U e_x cs2/(2 r^2) phi_z(e_z)
          v = fma(rho_f * c.lid_u * (double)ex, c.lid_c[k], v);
        f[q] = v;
      }
}

// ----------------------------------------------- isotropic density gradient
// d_d rho = (1/cs2) sum_a w_a e_ad rho(x + e_a) (reading R16)
// with the cuboid rest weights w_a = phi_x phi_y phi_z; per axis this is a central
// difference 1/(2c) weighted by the rest weights of the two other axes.  A
// neighbour across a wall face takes the node's own density.  rf has the
// population-buffer plane structure: rf[(z_local + 1) * nxy + y * nx + x].
// rho_at(i, j, k) = density at offset (i-1, j-1, k-1) from the node (never
// called for a neighbour across a wall); identical arithmetic for every source.
template <class RhoAt>
__device__ __forceinline__ void density_gradient_g(const Consts& c, int x, int y, int z, RhoAt rho_at, double& gx,
                                                   double& gy, double& gz) {
  auto is_wall = [](int fk) { return fk >= FK_BOUNCE && fk <= FK_SLIP; };
  const bool cx[3] = {x == 0 && is_wall(c.face[0]), false, x == c.nx - 1 && is_wall(c.face[1])};
  const bool cy[3] = {y == 0 && is_wall(c.face[2]), false, y == c.ny - 1 && is_wall(c.face[3])};
  const bool cz[3] = {z == 0 && is_wall(c.face[4]), false, z == c.nzl - 1 && is_wall(c.face[5])};
  const double own = rho_at(1, 1, 1);
  double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        if (i == 1 && j == 1 && k == 1) continue;
        const bool wall = cx[i] || cy[j] || cz[k];
        const double v = wall ? own : rho_at(i, j, k);
        if (i != 1) sx += (i == 2 ? 1.0 : -1.0) * c.phy[j] * c.phz[k] * v;
        if (j != 1) sy += (j == 2 ? 1.0 : -1.0) * c.phx[i] * c.phz[k] * v;
        if (k != 1) sz += (k == 2 ? 1.0 : -1.0) * c.phx[i] * c.phy[j] * v;
      }
  gx = 0.5 * sx;
  gy = c.h1y * sy;
  gz = c.h1z * sz;
}

__device__ __forceinline__ void density_gradient(const double* __restrict__ rf, const Consts& c, int x, int y,
                                                 int z, double& gx, double& gy, double& gz) {
  const int nx = c.nx;
  const int xs[3] = {(x == 0) ? nx - 1 : x - 1, x, (x == nx - 1) ? 0 : x + 1};
  const int ys[3] = {((y == 0) ? c.ny - 1 : y - 1) * nx, y * nx, ((y == c.ny - 1) ? 0 : y + 1) * nx};
  int zm = z - 1, zp = z + 1;
  if (z == 0 && c.face[4] == FK_WRAP) zm = c.nzl - 1;
  if (z == c.nzl - 1 && c.face[5] == FK_WRAP) zp = 0;
  const long long zb[3] = {(long long)(zm + 1) * c.nxy, (long long)(z + 1) * c.nxy, (long long)(zp + 1) * c.nxy};
  density_gradient_g(
      c, x, y, z, [&](int i, int j, int k) { return __ldg(rf + zb[k] + ys[j] + xs[i]); }, gx, gy, gz);
}

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
  double f[27];
  gather<T>(src, c, gx, gy, p, f);
  double r0 = 0.0;
#pragma unroll
  for (int q = 0; q < 27; ++q) r0 += f[q];
  return r0;
}

// --------------------------------------------------------- store policies
// Where the post-collision populations f~_q(x) go:
//   StoreOwn  (two-buffer "AB" pull scheme): own node, slot q of the other buffer;
//   StoreRev  (AA even step): own node, slot 26 - q of the same buffer;
//   StorePush (AA odd step): the slot whose next pull reads it (push with the
//             wall rules; the exact inverse of gather()).
template <typename T>
struct StoreOwn {
  T* base;
  T* out;
  int nxy;
  const Consts* c;
  __device__ __forceinline__ void begin(double) {}
  __device__ __forceinline__ void operator()(int q, double v) const {
    stcs<T>(LBM_CHECK_ST(base, out + q * nxy, *c), v);
  }
};

template <typename T>
struct StoreRev {
  T* base;
  T* out;
  int nxy;
  const Consts* c;
  __device__ __forceinline__ void begin(double) {}
  __device__ __forceinline__ void operator()(int q, double v) const {
    stcs<T>(LBM_CHECK_ST(base, out + (26 - q) * nxy, *c), v);
  }
};

// Push: f~_q(x) goes to the population the next pull at x + e_q takes it from.
// Normal link: node x + e_q (periodic wrap), slot q.  A crossed no-slip face:
// own node, slot 26 - q, plus the Eq. 69 term if the face is the moving lid
// (rho_f = rho of the node = sum f~, reading R4).  A crossed free-slip face:
// node x + e'_q (crossed axes zeroed), slot q* (crossed axes mirrored).
template <typename T>
struct StorePush {
  T* base;
  const Consts* c;
  int x, y, own;
  int dx[3], dy[3];   // destination x, y*nx for displacement e + 1
  T* pz[3];           // destination plane for e_z + 1
  int cx[3], cy[3], cz[3];  // kind of the face crossed by displacement e + 1 (0: none)
  bool wall;
  double rho_f;
  __device__ __forceinline__ StorePush(T* buf, const Consts& cc, int x_, int y_, int z) : base(buf), c(&cc), x(x_), y(y_) {
    const int nx = cc.nx;
    own = y * nx + x;
    dx[0] = (x == 0) ? nx - 1 : x - 1;
    dx[1] = x;
    dx[2] = (x == nx - 1) ? 0 : x + 1;
    dy[0] = ((y == 0) ? cc.ny - 1 : y - 1) * nx;
    dy[1] = y * nx;
    dy[2] = ((y == cc.ny - 1) ? 0 : y + 1) * nx;
    const int zm = (z == 0) ? cc.nzl - 1 : z - 1, zp = (z == cc.nzl - 1) ? 0 : z + 1;
    pz[0] = buf + (long long)(zm + 1) * cc.plane;
    pz[1] = buf + (long long)(z + 1) * cc.plane;
    pz[2] = buf + (long long)(zp + 1) * cc.plane;
    auto kind = [](int fk) { return (fk >= FK_BOUNCE && fk <= FK_SLIP) ? fk : 0; };
    cx[0] = (x == 0) ? kind(cc.face[0]) : 0;
    cx[1] = 0;
    cx[2] = (x == nx - 1) ? kind(cc.face[1]) : 0;
    cy[0] = (y == 0) ? kind(cc.face[2]) : 0;
    cy[1] = 0;
    cy[2] = (y == cc.ny - 1) ? kind(cc.face[3]) : 0;
    cz[0] = (z == 0) ? kind(cc.face[4]) : 0;
    cz[1] = 0;
    cz[2] = (z == cc.nzl - 1) ? kind(cc.face[5]) : 0;
    // warp-uniform: a warp with any wall-adjacent lane stores through the wall
    // rules (which reduce to the plain push for its other lanes)
    wall = __any_sync(__activemask(), (cx[0] | cx[2] | cy[0] | cy[2] | cz[0] | cz[2]) != 0);
    rho_f = 0.0;
  }
  __device__ __forceinline__ void begin(double rho) { rho_f = rho; }
  __device__ __forceinline__ void operator()(int q, double v) const {
    const int i = q % 3, j = (q / 3) % 3, k = q / 9;
    const int nxy = c->nxy;
    if (!wall) {
      stcs<T>(LBM_CHECK_ST(base, pz[k] + q * nxy + dy[j] + dx[i], *c), v);
      return;
    }
    const int kx = cx[i], ky = cy[j], kz = cz[k];
    T* a_bb = pz[1] + (26 - q) * nxy + own;
    double w = v;
    if (ky == FK_MOVING) w = fma(rho_f * c->lid_u * (double)(1 - i), c->lid_c[2 - k], w);
    if (!c->has_slip) {  // no free-slip face (uniform): plain push or bounce-back slot
      const bool noslip = (kx | ky | kz) != 0;
      stcs<T>(LBM_CHECK_ST(base, noslip ? a_bb : pz[k] + q * nxy + dy[j] + dx[i], *c), w);
      return;
    }
    const bool noslip = (kx == FK_BOUNCE || kx == FK_MOVING) || (ky == FK_BOUNCE || ky == FK_MOVING) ||
                        (kz == FK_BOUNCE || kz == FK_MOVING);
    // one store per direction, its destination chosen per lane: a crossed no-slip
    // face -> own node slot 26 - q (+ the Eq. 69 term across the lid, arriving as
    // direction 26 - q: + rho_f U e_x(26-q) lid_c[e_z(26-q)]); a crossed
    // free-slip face -> mirrored slot at the own coordinate along the crossed
    // axes; otherwise the periodic neighbour
    const bool mx = (kx == FK_SLIP), my = (ky == FK_SLIP), mz = (kz == FK_SLIP);
    const int qi = mx ? 2 - i : i, qj = my ? 2 - j : j, qk = mz ? 2 - k : k;
    const int xs = mx ? x : dx[i];
    const int ys = my ? y * c->nx : dy[j];
    T* zs = mz ? pz[1] : pz[k];
    T* a_slip = zs + LBM_Q(qi, qj, qk) * nxy + ys + xs;
    stcs<T>(LBM_CHECK_ST(base, noslip ? a_bb : a_slip, *c), w);
  }
};

// ------------------------------------------------------------ collision cores
// Each core takes the 27 pre-collision populations f (internal order) of one
// node and hands the 27 post-collision populations to the store policy.
#if LBM_MINB > 0
#define LBM_CS_BOUNDS __launch_bounds__(kBlock, LBM_MINB)
#else
#define LBM_CS_BOUNDS __launch_bounds__(kBlock)
#endif

// Generic rates (any omega_1, omega_high): all 27 central moments.
template <bool FD, class St>
__device__ __forceinline__ void core_generic(const Consts& c, double (&f)[27], double gxr, double gyr, double gzr,
                                             St& st) {
  // m = P f (App A), per axis
  raw_pass<0>(f);
  raw_pass<1>(f);
  raw_pass<2>(f);
  // rho, u (Eq. 12); y/z first moments carry the S factors r, s
  const double rho = f[LBM_Q(0, 0, 0)];
  const double inv_rho = 1.0 / rho;
  const double ux = (f[LBM_Q(1, 0, 0)] + 0.5 * c.F[0]) * inv_rho;
  const double uy = fma(c.r, f[LBM_Q(0, 1, 0)], 0.5 * c.F[1]) * inv_rho;
  const double uz = fma(c.s, f[LBM_Q(0, 0, 1)], 0.5 * c.F[2]) * inv_rho;
  // m^c = F S m (App B + App C), per axis
  central_pass<0, true>(f, ux, 1.0, 1.0);
  central_pass<1, false>(f, uy, c.r, c.r2);
  central_pass<2, false>(f, uz, c.s, c.s2);

  collide_generic<FD>(c, f, rho, inv_rho, ux, uy, uz, gxr, gyr, gzr);

  // f~ = P^-1 S^-1 F^-1 m~^c (App E, F, G), per axis
  inverse_pass<2>(f, uz, c.h1z, c.h2z);
  inverse_pass<1>(f, uy, c.h1y, c.h2y);
  inverse_pass<0>(f, ux, 0.5, 0.5);
  st.begin(rho);
#pragma unroll
  for (int q = 0; q < 27; ++q) st(q, f[q]);
}

// ------------------------------------- paper-rate kernel (omega_1 = omega_high = 1)
// With every rate except omega_nu and omega_xi equal to 1 (the setting
// of all the paper's results), App D sends every first-order central moment to
// F/2 (k~ = k + 1 (0 - k) + (1 - 1/2) F) and every moment of order >= 3 to its
// equilibrium of Eq. 64 (0, cs^4 rho or cs^6 rho), whatever its pre-collision
// value.  So the forward transform only needs the raw moments up to second
// order, and the post-collision central moments are
//   K000 = rho, K100 = Fx/2, K010 = Fy/2, K001 = Fz/2,
//   K110, K101, K011 (relaxed with omega_nu), K200, K020, K002 (App D, B/B^-1),
//   K220 = K202 = K022 = cs^4 rho, K222 = cs^6 rho, all others 0,
// which the inverse per-axis transforms exploit (zero inputs skipped).

// 1D inverse transform (central -> raw -> unscale -> populations), with
// compile-time knowledge of zero inputs k1 / k2 (see inverse_pass).
template <bool H1, bool H2>
__device__ __forceinline__ void inv1d(double k0, double k1, double k2, double u, double h1, double h2,
                                      double& fm, double& f0, double& fp) {
  const double A = H1 ? fma(u, k0, k1) : u * k0;
  const double t = H1 ? k1 + A : A;
  const double B = H2 ? fma(u, t, k2) : u * t;
  const double t1 = A * h1, t2 = B * h2;
  fm = t2 - t1;
  f0 = fma(-2.0, t2, k0);
  fp = t2 + t1;
}

template <bool FD, class St>
__device__ __forceinline__ void core_paper(const Consts& c, double (&f)[27], double gxr, double gyr, double gzr,
                                           St& st) {
  // raw moments up to second order, cubic units (App A restricted to m+n+p <= 2).
  // x-pass on all nine (y,z) rows: slots (0,j,k), (1,j,k), (2,j,k) <- m0, m1, m2 along x
  raw_pass<0>(f);
  // y-pass: x-order 0 needs (m0, m1, m2); x-order 1 needs (m0, m1); x-order 2 needs m0
  double a0[3], a1[3], a2[3], b0[3], b1[3], c0[3];  // [z slot]
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    {
      const double fm = f[LBM_Q(0, 0, k)], f0 = f[LBM_Q(0, 1, k)], fp = f[LBM_Q(0, 2, k)];
      const double sp = fp + fm;
      a0[k] = sp + f0;
      a1[k] = fp - fm;
      a2[k] = sp;
    }
    {
      const double fm = f[LBM_Q(1, 0, k)], f0 = f[LBM_Q(1, 1, k)], fp = f[LBM_Q(1, 2, k)];
      b0[k] = (fp + fm) + f0;
      b1[k] = fp - fm;
    }
    c0[k] = (f[LBM_Q(2, 0, k)] + f[LBM_Q(2, 2, k)]) + f[LBM_Q(2, 1, k)];
  }
  // z-pass
  const double rho = (a0[2] + a0[0]) + a0[1];  // M000
  const double Mz = a0[2] - a0[0];             // M001
  const double Mzz = a0[2] + a0[0];            // M002
  const double My = (a1[2] + a1[0]) + a1[1];   // M010
  const double Myz = a1[2] - a1[0];            // M011
  const double Myy = (a2[2] + a2[0]) + a2[1];  // M020
  const double Mx = (b0[2] + b0[0]) + b0[1];   // M100
  const double Mxz = b0[2] - b0[0];            // M101
  const double Mxy = (b1[2] + b1[0]) + b1[1];  // M110
  const double Mxx = (c0[2] + c0[0]) + c0[1];  // M200

  // scale to the cuboid lattice (App B) and shift to central moments (App C)
  const double inv_rho = 1.0 / rho;
  const double jx = Mx, jy = c.r * My, jz = c.s * Mz;
  const double ux = (jx + 0.5 * c.F[0]) * inv_rho;
  const double uy = (jy + 0.5 * c.F[1]) * inv_rho;
  const double uz = (jz + 0.5 * c.F[2]) * inv_rho;
  // k_ab = Pi_ab - u_a j_b - u_b j_a + rho u_a u_b
  const double k200 = Mxx - ux * fma(-rho, ux, 2.0 * jx);
  const double k020 = fma(c.r2, Myy, -uy * fma(-rho, uy, 2.0 * jy));
  const double k002 = fma(c.s2, Mzz, -uz * fma(-rho, uz, 2.0 * jz));
  const double k110 = fma(c.r, Mxy, -fma(ux, jy, uy * fma(-rho, ux, jx)));
  const double k101 = fma(c.s, Mxz, -fma(ux, jz, uz * fma(-rho, ux, jx)));
  const double k011 = fma(c.r * c.s, Myz, -fma(uy, jz, uz * fma(-rho, uy, jy)));

  // collision (App D) for the second order; first order -> F/2, higher -> Eq. 64
  double K200, K020, K002;
  second_order_diag<FD>(c, rho, inv_rho, ux, uy, uz, k200, k020, k002, K200, K020, K002, gxr, gyr, gzr);
  const double om = 1.0 - c.wn;
  const double K110 = om * k110, K101 = om * k101, K011 = om * k011;
  const double K100 = 0.5 * c.F[0], K010 = 0.5 * c.F[1], K001 = 0.5 * c.F[2];
  const double c4r = c.c4 * rho, c6r = c.c6 * rho;

  // inverse transforms (App E, F, G per axis), z first.  G[i][j][kz]
  double G00[3], G10[3], G01[3], G11[3], G20[3], G02[3], G22[3];
  inv1d<true, true>(rho, K001, K002, uz, c.h1z, c.h2z, G00[0], G00[1], G00[2]);
  inv1d<true, false>(K100, K101, 0.0, uz, c.h1z, c.h2z, G10[0], G10[1], G10[2]);
  inv1d<true, false>(K010, K011, 0.0, uz, c.h1z, c.h2z, G01[0], G01[1], G01[2]);
  inv1d<false, false>(K110, 0.0, 0.0, uz, c.h1z, c.h2z, G11[0], G11[1], G11[2]);
  inv1d<false, true>(K200, 0.0, c4r, uz, c.h1z, c.h2z, G20[0], G20[1], G20[2]);
  inv1d<false, true>(K020, 0.0, c4r, uz, c.h1z, c.h2z, G02[0], G02[1], G02[2]);
  inv1d<false, true>(c4r, 0.0, c6r, uz, c.h1z, c.h2z, G22[0], G22[1], G22[2]);

  st.begin(rho);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    // y: (x-order 0): (G00, G01, G02); (x-order 1): (G10, G11, 0); (x-order 2): (G20, 0, G22)
    double H0[3], H1[3], H2[3];  // [jy] for x-orders 0, 1, 2
    inv1d<true, true>(G00[k], G01[k], G02[k], uy, c.h1y, c.h2y, H0[0], H0[1], H0[2]);
    inv1d<true, false>(G10[k], G11[k], 0.0, uy, c.h1y, c.h2y, H1[0], H1[1], H1[2]);
    inv1d<false, true>(G20[k], 0.0, G22[k], uy, c.h1y, c.h2y, H2[0], H2[1], H2[2]);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double fm, f0, fp;
      inv1d<true, true>(H0[j], H1[j], H2[j], ux, 0.5, 0.5, fm, f0, fp);
      st(LBM_Q(0, j, k), fm);
      st(LBM_Q(1, j, k), f0);
      st(LBM_Q(2, j, k), fp);
    }
  }
}

// ------------------------------------------------ 3DCRM raw-moment kernel
// The raw-moment variant of P:L642-648 (Eq. LBErawmomentcuboidlattice), named
// 3DCRM at P:L1011: the same pipeline without F / F^-1; raw moments relax to the
// Eq. 10 equilibria (which factorise per axis: rho E_x[i] E_y[j] E_z[k] with
// E = (1, u, cs2 + u^2)) with the Eq. 11 sources (zero from third order on), the
// same B grouping, rates and theta corrections; strain rates from the raw
// non-equilibrium moments.

// scale raw moments by the axis speed (App B): (m0, m1, m2) -> (m0, c m1, c^2 m2)
template <int AX>
__device__ __forceinline__ void scale_pass(double (&f)[27], double c, double c2) {
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int q = a * Axis<AX>::o1 + b * Axis<AX>::o2;
      f[q + Axis<AX>::st] *= c;
      f[q + 2 * Axis<AX>::st] *= c2;
    }
}

// per-axis inverse with u = 0 (App F + App G): f0 = k0 - k2/c^2, f+- = (k2/c^2 +- k1/c)/2
template <int AX>
__device__ __forceinline__ void unscale_inverse_pass(double (&f)[27], double h1, double h2) {
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int q = a * Axis<AX>::o1 + b * Axis<AX>::o2;
      const double k0 = f[q], t1 = f[q + Axis<AX>::st] * h1, t2 = f[q + 2 * Axis<AX>::st] * h2;
      f[q] = t2 - t1;
      f[q + Axis<AX>::st] = fma(-2.0, t2, k0);
      f[q + 2 * Axis<AX>::st] = t2 + t1;
    }
}

template <bool FD>
__device__ __forceinline__ void collide_raw(const Consts& c, double (&f)[27], double rho, double inv_rho,
                                            double ux, double uy, double uz, double gxr, double gyr, double gzr) {
#define M(i, j, k) f[LBM_Q(i, j, k)]
  const double w1 = c.w1, wn = c.wn, wh = c.wh;
  const double Ex[3] = {1.0, ux, c.cs2 + ux * ux}, Ey[3] = {1.0, uy, c.cs2 + uy * uy},
               Ez[3] = {1.0, uz, c.cs2 + uz * uz};
  const double Fx = c.F[0], Fy = c.F[1], Fz = c.F[2];
  // first order: m + w1 (rho u - m) + (1 - w1/2) F
  M(1, 0, 0) = fma(w1, rho * ux - M(1, 0, 0), M(1, 0, 0)) + (1.0 - 0.5 * w1) * Fx;
  M(0, 1, 0) = fma(w1, rho * uy - M(0, 1, 0), M(0, 1, 0)) + (1.0 - 0.5 * w1) * Fy;
  M(0, 0, 1) = fma(w1, rho * uz - M(0, 0, 1), M(0, 0, 1)) + (1.0 - 0.5 * w1) * Fz;
  // off-diagonal second order, sources F_a u_b + F_b u_a
  const double hn = 1.0 - 0.5 * wn;
  M(1, 1, 0) = fma(wn, rho * ux * uy - M(1, 1, 0), M(1, 1, 0)) + hn * (Fx * uy + Fy * ux);
  M(1, 0, 1) = fma(wn, rho * ux * uz - M(1, 0, 1), M(1, 0, 1)) + hn * (Fx * uz + Fz * ux);
  M(0, 1, 1) = fma(wn, rho * uy * uz - M(0, 1, 1), M(0, 1, 1)) + hn * (Fy * uz + Fz * uy);
  // diagonal second order (B, corrections, relax, B^-1)
  {
    const double k200 = M(2, 0, 0), k020 = M(0, 2, 0), k002 = M(0, 0, 2);
    const double k2s = k200 + k020 + k002, k2d1 = k200 - k020, k2d2 = k200 - k002;
    const double q200 = rho * Ex[2], q020 = rho * Ey[2], q002 = rho * Ez[2];
    double e2s = q200 + q020 + q002, e2d1 = q200 - q020, e2d2 = q200 - q002;
    if (c.corr_on) {
      const double ga = 1.5 * c.galias;
      const double qx = ga * ux * ux, qy = ga * uy * uy, qz = ga * uz * uz;
      const double Csx = -c.csn + 0.5 * c.gx + qx;
      const double Cbx = -c.csx + 0.5 * c.gx + qx;
      const double Csy = c.csn - 0.5 * c.gy - qy;
      const double Cby = -c.csx + 0.5 * c.gy + qy;
      const double Csz = c.csn - 0.5 * c.gz - qz;
      const double Cbz = -c.csx + 0.5 * c.gz + qz;
      double Rb = (k2s - e2s) * inv_rho, Rs1 = (k2d1 - e2d1) * inv_rho, Rs2 = (k2d2 - e2d2) * inv_rho;
      double lsx = 0.0, lsy = 0.0, lsz = 0.0;  // e_rho terms, FULL_FD only
      if (FD) {
        lsx = 0.5 * c.gx * ux * gxr;
        lsy = 0.5 * c.gy * uy * gyr;
        lsz = 0.5 * c.gz * uz * gzr;
        Rb += (-lsx - lsy - lsz) * inv_rho;
        Rs1 += (-lsx + lsy) * inv_rho;
        Rs2 += (-lsx + lsz) * inv_rho;
      }
      const double t1 = Csx * Cbz - Csz * Cbx;
      const double inv_det = 1.0 / (-Csx * Csz * Cby - Csy * t1);
      const double dxux = (-Csz * Cby * Rs1 - Csy * (Cbz * Rs2 - Csz * Rb)) * inv_det;
      const double dyuy = (Csx * (Rs2 * Cbz - Csz * Rb) - Rs1 * t1) * inv_det;
      const double dzuz = (Csx * Cby * (Rs1 - Rs2) - Csy * (Csx * Rb - Rs2 * Cbx)) * inv_det;
      const double tx = (2.0 * qx + c.gx) * dxux, ty = (2.0 * qy + c.gy) * dyuy, tz = (2.0 * qz + c.gz) * dzuz;
      const double rn = rho * c.an, rb = rho * c.ab;
      e2d1 -= rn * (tx - ty);
      e2d2 -= rn * (tx - tz);
      e2s -= rb * (tx + ty + tz);
      if (FD) {
        e2d1 += 2.0 * c.an * (-lsx + lsy);
        e2d2 += 2.0 * c.an * (-lsx + lsz);
        e2s += 2.0 * c.ab * (-lsx - lsy - lsz);
      }
    }
    const double p2s = 2.0 * (Fx * ux + Fy * uy + Fz * uz), p2d1 = 2.0 * (Fx * ux - Fy * uy),
                 p2d2 = 2.0 * (Fx * ux - Fz * uz);
    const double s2s = fma(c.wx, e2s - k2s, k2s) + (1.0 - 0.5 * c.wx) * p2s;
    const double s2d1 = fma(wn, e2d1 - k2d1, k2d1) + hn * p2d1;
    const double s2d2 = fma(wn, e2d2 - k2d2, k2d2) + hn * p2d2;
    const double third = 1.0 / 3.0;
    M(2, 0, 0) = (s2s + s2d1 + s2d2) * third;
    M(0, 2, 0) = (s2s - 2.0 * s2d1 + s2d2) * third;
    M(0, 0, 2) = (s2s + s2d1 - 2.0 * s2d2) * third;
  }
  // third and higher orders: one rate per B group -> per moment, toward Eq. 10
  const double om = 1.0 - wh, wr = wh * rho;
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 3; ++i)
        if (i + j + k >= 3) M(i, j, k) = fma(om, M(i, j, k), wr * Ex[i] * Ey[j] * Ez[k]);
#undef M
}

template <bool FD, class St>
__device__ __forceinline__ void core_raw(const Consts& c, double (&f)[27], double gxr, double gyr, double gzr,
                                         St& st) {
  raw_pass<0>(f);
  raw_pass<1>(f);
  raw_pass<2>(f);
  const double rho = f[LBM_Q(0, 0, 0)];
  const double inv_rho = 1.0 / rho;
  const double ux = (f[LBM_Q(1, 0, 0)] + 0.5 * c.F[0]) * inv_rho;
  const double uy = fma(c.r, f[LBM_Q(0, 1, 0)], 0.5 * c.F[1]) * inv_rho;
  const double uz = fma(c.s, f[LBM_Q(0, 0, 1)], 0.5 * c.F[2]) * inv_rho;
  scale_pass<1>(f, c.r, c.r2);
  scale_pass<2>(f, c.s, c.s2);
  collide_raw<FD>(c, f, rho, inv_rho, ux, uy, uz, gxr, gyr, gzr);
  unscale_inverse_pass<2>(f, c.h1z, c.h2z);
  unscale_inverse_pass<1>(f, c.h1y, c.h2y);
  unscale_inverse_pass<0>(f, 0.5, 0.5);
  st.begin(rho);
#pragma unroll
  for (int q = 0; q < 27; ++q) st(q, f[q]);
}

enum CoreKind : int { CORE_GENERIC = 0, CORE_PAPER = 1, CORE_RAW = 2 };

template <int KIND, bool FD, class St>
__device__ __forceinline__ void run_core(const Consts& c, double (&f)[27], double gxr, double gyr, double gzr,
                                         St& st) {
  if (KIND == CORE_PAPER)
    core_paper<FD>(c, f, gxr, gyr, gzr, st);
  else if (KIND == CORE_RAW)
    core_raw<FD>(c, f, gxr, gyr, gzr, st);
  else
    core_generic<FD>(c, f, gxr, gyr, gzr, st);
}

// ------------------------------------------------ the fused kernels (two buffers)
// One thread per node of planes zbeg + i*zstride, i < gridDim.y, of the local
// slab: pull (gather) from src, collide, store at the own node of dst.
template <typename T, int KIND, bool FD>
__device__ __forceinline__ void collide_stream_ab(const T* __restrict__ src, T* __restrict__ dst,
                                                  const double* __restrict__ rf, const Consts& c, int zbeg,
                                                  int zstride) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  if (idx >= c.nxy) return;
  const int y = row_of(c, idx);
  const int x = idx - y * c.nx;
  const int z = zbeg + blockIdx.y * zstride;  // zstride > 1: the two boundary planes in one launch
  double f[27];
  // FULL_FD: gradient first, so its L2-resident loads overlap the population loads
  double gxr = 0.0, gyr = 0.0, gzr = 0.0;
  if (FD) density_gradient(rf, c, x, y, z, gxr, gyr, gzr);
  gather<T>(src, c, x, y, z, f);
  StoreOwn<T> st{dst, dst + (long long)(z + 1) * c.plane + idx, c.nxy, &c};
  run_core<KIND, FD>(c, f, gxr, gyr, gzr, st);
}

template <typename T, bool FD>
__global__ void LBM_CS_BOUNDS k_collide_stream(const T* __restrict__ src, T* __restrict__ dst,
                                               const double* __restrict__ rf, const __grid_constant__ Consts c,
                                               int zbeg, int zstride) {
  collide_stream_ab<T, CORE_GENERIC, FD>(src, dst, rf, c, zbeg, zstride);
}

template <typename T, bool FD>
__global__ void LBM_CS_BOUNDS k_collide_stream_paper(const T* __restrict__ src, T* __restrict__ dst,
                                                     const double* __restrict__ rf, const __grid_constant__ Consts c,
                                                     int zbeg, int zstride) {
  collide_stream_ab<T, CORE_PAPER, FD>(src, dst, rf, c, zbeg, zstride);
}

template <typename T, bool FD>
__global__ void LBM_CS_BOUNDS k_collide_stream_raw(const T* __restrict__ src, T* __restrict__ dst,
                                                   const double* __restrict__ rf, const __grid_constant__ Consts c,
                                                   int zbeg, int zstride) {
  collide_stream_ab<T, CORE_RAW, FD>(src, dst, rf, c, zbeg, zstride);
}

// chunk blockIdx.z covers planes [z0, z1), z0 = zbeg + blockIdx.z * zstride,
// z1 = min(z0 + zlen, zend).  Iteration p forms rho(p) on the tile and its ring,
// then collides plane p - 1.
template <typename T, int KIND>
__device__ __forceinline__ void collide_stream_fd_fused(const T* __restrict__ src, T* __restrict__ dst,
                                                        const double* __restrict__ rf, const Consts& c, int zbeg,
                                                        int zstride, int zlen, int zend) {
  __shared__ double srho[4][kFdTy + 2][kFdRw];
  const int tx = threadIdx.x % kFdTx, ty = threadIdx.x / kFdTx;
  const int x0 = blockIdx.x * kFdTx, y0 = blockIdx.y * kFdTy;
  const int z0 = zbeg + blockIdx.z * zstride;
  const int z1 = min(z0 + zlen, zend);
  const int x = x0 + tx, y = y0 + ty;
  const bool active = (x < c.nx) && (y < c.ny);
  for (int p = z0 - 1; p <= z1; ++p) {
    // four slots: the slot written here was last read two planes ago, and this
    // iteration's barrier separates the two (one barrier per plane)
    for (int pos = threadIdx.x; pos < kFdRing; pos += kFdThreads) {
      const int ly = pos / kFdRw, lx = pos - ly * kFdRw;
      srho[p & 3][ly][lx] = ring_rho<T>(src, rf, c, x0 + lx - 1, y0 + ly - 1, p);
    }
    __syncthreads();
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
  collide_stream_fd_fused<T, KIND>(src, dst, rf, c, zbeg, zstride, zlen, zend);
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
  __device__ __forceinline__ void begin(double) {}
  __device__ __forceinline__ void operator()(int q, double v) const {
    stcs<T>(LBM_CHECK_ST(base, out + q * nxy, *c), v);
    if (q >= 18 && rup) stcs<T>(LBM_CHECK_ST(up_base, rup + q * nxy, *c), v);
    if (q < 9 && rdn) stcs<T>(LBM_CHECK_ST(dn_base, rdn + q * nxy, *c), v);
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
                    a.dn};
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
__global__ void __launch_bounds__(kBlock) k_halo_push(const T* __restrict__ src, const __grid_constant__ Consts c,
                                                      const P2PArgs<T> a) {
  const long long e = (long long)blockIdx.x * kBlock + threadIdx.x;
  if (e < 9LL * c.nxy) {
    if (blockIdx.y == 0 && a.dn)  // bottom plane p = 1, q 0..8 -> ghost p = nz_l + 1
      a.dn[(long long)(c.nzl + 1) * c.plane + e] = src[c.plane + e];
    if (blockIdx.y == 1 && a.up)  // top plane p = nz_l, q 18..26 -> ghost p = 0
      a.up[18LL * c.nxy + e] = src[(long long)c.nzl * c.plane + 18LL * c.nxy + e];
  }
  p2p_signal(a);
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
  }
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

template <typename T>
__global__ void __launch_bounds__(kBlock) k_check(const T* __restrict__ src, double* __restrict__ out,
                                                  const __grid_constant__ Consts c, int aa) {
  const int idx = blockIdx.x * kBlock + threadIdx.x;
  const int z = blockIdx.y;
  double v[7] = {0, 0, 0, 0, 0, 0, 0};
  if (idx < c.nxy) {
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
    v[0] = rho;
    v[1] = rho * ux;
    v[2] = rho * uy;
    v[3] = rho * uz;
    v[4] = 0.5 * rho * u2;
    v[5] = sqrt(u2);
    const bool bad = !(rho > 0.0) || !(u2 <= 1.0) || !isfinite(rho) || !isfinite(u2);
    v[6] = bad ? 1.0 : 0.0;
    if (bad) v[5] = 0.0;
  }
  __shared__ double sm[7][kBlock / 32];
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
    for (int i = 1; i < kBlock / 32; ++i) r = (t == 5) ? fmax(r, sm[t][i]) : r + sm[t][i];
    if (t == 5)
      atomicMax(reinterpret_cast<unsigned long long*>(out + 5), (unsigned long long)__double_as_longlong(r));
    else
      atomicAdd(out + t, r);
  }
}

}  // namespace lbm
