// cm_moments.cuh -- per-node arithmetic of the 3D cuboid central-moment LBM:
// the per-axis moment transforms, the App D collision and the
// collision cores that take 27 pulled populations to 27 post-collision ones
// (generic rates, paper rates, 3DCRM raw moments).  "P:Lnnn" cites
// /root/reference/PAPER.md line nnn.
#pragma once

#include "cm_common.cuh"

namespace lbm {

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
    note_singular(c, det, Csy, Csz, rho);
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

// ------------------------------------------------------------ collision cores
// Each core takes the 27 pre-collision populations f (internal order) of one
// node and hands the 27 post-collision populations to the store policy.
#if LBM_MINB > 0
#define LBM_CS_BOUNDS __launch_bounds__(kBlock, LBM_MINB)
#else
#define LBM_CS_BOUNDS __launch_bounds__(kBlock)
#endif
// collide-stream kernels with the density-gradient terms (FULL_FD two-pass and
// FULL_FD_LAG): ask for 6 resident 128-thread CTAs (<= 80 registers; 112 without
// the bound cost ~7 % at 512^3)
#ifndef LBM_FD_CS_MINB
#define LBM_FD_CS_MINB 6
#endif
#define LBM_CS_BOUNDS_FD(FD) __launch_bounds__(kBlock, (FD) ? LBM_FD_CS_MINB : LBM_MINB)

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
      const double det = -Csx * Csz * Cby - Csy * t1;
      note_singular(c, det, Csy, Csz, rho);
      const double inv_det = 1.0 / det;
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


}  // namespace lbm
