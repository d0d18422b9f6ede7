/*
 * cm_oracle.c -- CPU ORACLE for the 3D cuboid central-moment LBM (3DCCM-LBM)
 * of Yahia, Schupbach & Premnath, arXiv 2107.14774.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_2107_14774_b200/) never links, imports or calls it.
 *
 * Plain, slow, single-threaded, IEEE fp64, built with -O2 -ffp-contract=off.
 * It shares no code, header, table or constant generator with the CUDA path.
 * Every function follows a definition or an algorithm step of the paper
 * ("P:Lnnn" = /root/reference/PAPER.md line nnn):
 *
 *   velocities          Eqs. 1a-1c
 *   Q moment basis      Eq. 57 (Q = S P, Eq. 58)
 *   Q^-1                numeric Gauss-Jordan inverse of Q        (Eq. 60)
 *   rho, u              Eq. 12
 *   central moments     Eq. 3a, literally
 *   raw equilibria      Eq. 10, literally
 *   collision           App D: B, effective equilibria, local
 *                       strain rates, relax, B^-1
 *   3DCRM variant       raw-moment collision, Eq. 10/11          P:L642-648, L744(ii), L1011
 *   central -> raw      binomial transform F^-1 = F(-u)
 *   post-coll. f        f~ = Q^-1 m~  (= P^-1 S^-1 m~)
 *   streaming           pull form f(x,t+1) = f~(x - e, t)
 *   halfway bounce-back + momentum-augmented moving wall,
 *                       f^eq at the wall from Q^-1 m^eq          P:L746-769 (Eq. 69)
 *
 * Readings where the paper is silent: R1 (lambda = 0,
 * e_rho = 0 in FULL_LOCAL; LOW_MACH drops the 3u^2 terms of theta and C), R4
 * (rho_f of Eq. 69 at the wall-adjacent node, same time level as the reflected
 * f~), R5 (lid augmentation on every link whose source crosses the +y face),
 * R6 (a wall wins over periodicity), R7 (free-slip = halfway specular
 * reflection), R8 (init f~ = f^eq(rho0, u0 + F/(2 rho0))), R16 (FULL_FD: the
 * isotropic lattice gradient of the same-time density, mirror-image neighbours
 * across walls), R16b (FULL_FD_LAG: the same gradient of the stored state's
 * density, one time level earlier), R17 (singular strain-rate system).
 *
 * Parity pins: tests/test_oracle_*.py (closed forms, paper-printed appendices
 * and Eq. 69, conservation, SRT limit, order of the corrections (slope 3 on the
 * cubic lattice, 1 on the cuboid one), analytic TGV/shear-wave/duct decay,
 * plane Couette flow under the moving lid, viscous and acoustic isotropy,
 * Galilean invariance, moving-frame sound attenuation for the density-gradient
 * terms, Womersley, long-wave eigenvalues of the linearised update).
 * The free-slip rule (reading R7) is not in the paper (BASELINE config 4 asks
 * for it); it is pinned by invariants (mass, tangential momentum) and by the
 * analytic decay nu k^2 of the cosine shear mode between stress-free walls
 * (tests/test_oracle_physics.py; bounce-back walls give 8x that rate).
 *
 * Population layout of every array argument: [q][z][y][x], q in the paper's
 * order of Eqs. 1a-1c, x fastest.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NQ 27

/* Eqs. 1a-1c: components in units of (1, r, s). */
static const int EX[NQ] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1};
static const int EY[NQ] = {0, 0, 0, 1, -1, 0, 0, 1, 1, -1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, 1, -1, -1, 1, 1, -1, -1};
static const int EZ[NQ] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, 1, -1, -1, 1, 1, -1, -1, 1, 1, 1, 1, -1, -1, -1, -1};

/* Moment ordering of m / m^c: exponents (m, n, p). */
static const int MNP[NQ][3] = {
    {0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1},
    {2, 0, 0}, {0, 2, 0}, {0, 0, 2}, {1, 2, 0}, {1, 0, 2}, {2, 1, 0}, {0, 1, 2},
    {2, 0, 1}, {0, 2, 1}, {1, 1, 1}, {2, 2, 0}, {2, 0, 2}, {0, 2, 2}, {2, 1, 1},
    {1, 2, 1}, {1, 1, 2}, {1, 2, 2}, {2, 1, 2}, {2, 2, 1}, {2, 2, 2}};

/* index of moment (m,n,p) in the list above (inverse of MNP) */
static const int MIDX[3][3][3] = {
    /* m=0 */ {{0, 3, 9}, {2, 6, 13}, {8, 15, 19}},
    /* m=1 */ {{1, 5, 11}, {4, 16, 22}, {10, 21, 23}},
    /* m=2 */ {{7, 14, 18}, {12, 20, 24}, {17, 25, 26}}};
#define midx(m, n, p) MIDX[m][n][p]

enum { BC_PERIODIC = 0, BC_BOUNCE_BACK = 1, BC_MOVING_WALL = 2, BC_FREE_SLIP = 3 };
enum { CORR_FULL_LOCAL = 0, CORR_LOW_MACH = 1, CORR_OFF = 2, CORR_FULL_FD = 3, CORR_FULL_FD_LAG = 4 };
/* the density-gradient (lambda, e_rho) modes: same-time density (R16) or the stored state's (R16b) */
#define FD_MODE(c) ((c) == CORR_FULL_FD || (c) == CORR_FULL_FD_LAG)

typedef struct {
  int32_t nx, ny, nz;
  double r, s, cs2;
  double omega_nu, omega_xi, omega_1, omega_high;
  double force[3];
  int32_t bc[6]; /* faces -x,+x,-y,+y,-z,+z */
  double wall_u; /* +y face moves with velocity (U,0,0) */
  int32_t corrections;
  int32_t model; /* 0: 3DCCM (central moments); 1: 3DCRM (raw moments) */
} oracle_params;

typedef struct {
  oracle_params p;
  double e[NQ][3];  /* particle velocities, Eqs. 1a-1c */
  double Q[NQ * NQ];
  double Qinv[NQ * NQ];
  int opp[NQ];
} oracle_ctx;

static double ipow(double x, int n) {
  double y = 1.0;
  for (int i = 0; i < n; ++i) y *= x;
  return y;
}

static double binom(int n, int k) {
  /* n <= 2 */
  if (k < 0 || k > n) return 0.0;
  if (k == 0 || k == n) return 1.0;
  return (double)n; /* C(2,1) = 2 */
}

/* ---------------------------------------------------------------- lattice */

void oracle_velocities(double r, double s, double *e /* [27][3] */) {
  for (int a = 0; a < NQ; ++a) {
    e[3 * a + 0] = (double)EX[a];
    e[3 * a + 1] = r * (double)EY[a];
    e[3 * a + 2] = s * (double)EZ[a];
  }
}

void oracle_opposite(int *opp) {
  for (int a = 0; a < NQ; ++a)
    for (int b = 0; b < NQ; ++b)
      if (EX[b] == -EX[a] && EY[b] == -EY[a] && EZ[b] == -EZ[a]) opp[a] = b;
}

/* Eq. 57: row j of Q is the monomial e_x^m e_y^n e_z^p evaluated on the 27
 * cuboid velocities, so that m = Q f (Eq. 56). */
void oracle_Q(double r, double s, double *Q) {
  double e[NQ * 3];
  oracle_velocities(r, s, e);
  for (int j = 0; j < NQ; ++j)
    for (int a = 0; a < NQ; ++a)
      Q[j * NQ + a] = ipow(e[3 * a], MNP[j][0]) * ipow(e[3 * a + 1], MNP[j][1]) * ipow(e[3 * a + 2], MNP[j][2]);
}

/* Gauss-Jordan elimination with partial pivoting.  Returns 0, or -1 if singular. */
int oracle_invert27(const double *A_in, double *Ainv) {
  double A[NQ][2 * NQ];
  for (int i = 0; i < NQ; ++i)
    for (int j = 0; j < NQ; ++j) {
      A[i][j] = A_in[i * NQ + j];
      A[i][NQ + j] = (i == j) ? 1.0 : 0.0;
    }
  for (int c = 0; c < NQ; ++c) {
    int piv = c;
    for (int i = c + 1; i < NQ; ++i)
      if (fabs(A[i][c]) > fabs(A[piv][c])) piv = i;
    if (fabs(A[piv][c]) < 1e-300) return -1;
    if (piv != c)
      for (int j = 0; j < 2 * NQ; ++j) {
        double t = A[c][j];
        A[c][j] = A[piv][j];
        A[piv][j] = t;
      }
    double d = A[c][c];
    for (int j = 0; j < 2 * NQ; ++j) A[c][j] /= d;
    for (int i = 0; i < NQ; ++i) {
      if (i == c) continue;
      double m = A[i][c];
      if (m == 0.0) continue;
      for (int j = 0; j < 2 * NQ; ++j) A[i][j] -= m * A[c][j];
    }
  }
  for (int i = 0; i < NQ; ++i)
    for (int j = 0; j < NQ; ++j) Ainv[i * NQ + j] = A[i][NQ + j];
  return 0;
}

/* ---------------------------------------------------------------- moments */

/* Eq. 12: rho = sum f, rho u = sum f e + F/2 (Delta t = 1). */
void oracle_hydro(const double *e, const double *f, const double *F, double *rho_out, double *u) {
  double rho = 0.0, j[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < NQ; ++a) {
    rho += f[a];
    for (int d = 0; d < 3; ++d) j[d] += f[a] * e[3 * a + d];
  }
  for (int d = 0; d < 3; ++d) u[d] = (j[d] + 0.5 * F[d]) / rho;
  *rho_out = rho;
}

/* Eq. 3a, literally: k_mnp = sum_a f_a (e_ax - u_x)^m (e_ay - u_y)^n (e_az - u_z)^p. */
void oracle_central_moments(const double *e, const double *f, const double *u, double *k) {
  double pw[NQ][3][3]; /* pw[a][d][n] = (e_ad - u_d)^n */
  for (int a = 0; a < NQ; ++a)
    for (int d = 0; d < 3; ++d)
      for (int n = 0; n < 3; ++n) pw[a][d][n] = ipow(e[3 * a + d] - u[d], n);
  for (int j = 0; j < NQ; ++j) {
    double acc = 0.0;
    for (int a = 0; a < NQ; ++a) acc += f[a] * pw[a][0][MNP[j][0]] * pw[a][1][MNP[j][1]] * pw[a][2][MNP[j][2]];
    k[j] = acc;
  }
}

/* Binomial frame transform:
 *   out_mnp = sum_{i<=m, j<=n, k<=p} C(m,i) C(n,j) C(p,k) a_x^(m-i) a_y^(n-j) a_z^(p-k) in_ijk.
 * With a = -u it maps raw -> central (F(u), App C); with a = +u it maps
 * central -> raw (F^-1 = F(-u), App E). */
void oracle_frame(const double *in, const double *a, double *out) {
  double cf[3][3][3]; /* cf[d][m][i] = C(m,i) a_d^(m-i) */
  for (int d = 0; d < 3; ++d)
    for (int m = 0; m < 3; ++m)
      for (int i = 0; i < 3; ++i) cf[d][m][i] = (i <= m) ? binom(m, i) * ipow(a[d], m - i) : 0.0;
  for (int t = 0; t < NQ; ++t) {
    int m = MNP[t][0], n = MNP[t][1], p = MNP[t][2];
    double acc = 0.0;
    for (int i = 0; i <= m; ++i)
      for (int j = 0; j <= n; ++j)
        for (int k = 0; k <= p; ++k) acc += cf[0][m][i] * cf[1][n][j] * cf[2][p][k] * in[midx(i, j, k)];
    out[t] = acc;
  }
}

/* Eq. 10, written out literally, in the order of P:L612-613. */
void oracle_raw_equilibria(double rho, const double *u, double cs2, double *m) {
  double ux = u[0], uy = u[1], uz = u[2];
  double c2 = cs2, c4 = cs2 * cs2, c6 = cs2 * cs2 * cs2;
  double ux2 = ux * ux, uy2 = uy * uy, uz2 = uz * uz;
  m[midx(0, 0, 0)] = rho;
  m[midx(1, 0, 0)] = rho * ux;
  m[midx(0, 1, 0)] = rho * uy;
  m[midx(0, 0, 1)] = rho * uz;
  m[midx(1, 1, 0)] = rho * ux * uy;
  m[midx(1, 0, 1)] = rho * ux * uz;
  m[midx(0, 1, 1)] = rho * uy * uz;
  m[midx(2, 0, 0)] = c2 * rho + rho * ux2;
  m[midx(0, 2, 0)] = c2 * rho + rho * uy2;
  m[midx(0, 0, 2)] = c2 * rho + rho * uz2;
  m[midx(1, 2, 0)] = c2 * rho * ux + rho * ux * uy2;
  m[midx(1, 0, 2)] = c2 * rho * ux + rho * ux * uz2;
  m[midx(2, 1, 0)] = c2 * rho * uy + rho * ux2 * uy;
  m[midx(0, 1, 2)] = c2 * rho * uy + rho * uy * uz2;
  m[midx(2, 0, 1)] = c2 * rho * uz + rho * ux2 * uz;
  m[midx(0, 2, 1)] = c2 * rho * uz + rho * uy2 * uz;
  m[midx(1, 1, 1)] = rho * ux * uy * uz;
  m[midx(2, 2, 0)] = c4 * rho + rho * c2 * (ux2 + uy2) + rho * ux2 * uy2;
  m[midx(2, 0, 2)] = c4 * rho + rho * c2 * (ux2 + uz2) + rho * ux2 * uz2;
  m[midx(0, 2, 2)] = c4 * rho + rho * c2 * (uy2 + uz2) + rho * uy2 * uz2;
  m[midx(2, 1, 1)] = rho * (c2 + ux2) * uy * uz;
  m[midx(1, 2, 1)] = rho * (c2 + uy2) * ux * uz;
  m[midx(1, 1, 2)] = rho * (c2 + uz2) * ux * uy;
  m[midx(1, 2, 2)] = c4 * rho * ux + rho * c2 * ux * (uy2 + uz2) + rho * ux * uy2 * uz2;
  m[midx(2, 1, 2)] = c4 * rho * uy + rho * c2 * uy * (ux2 + uz2) + rho * ux2 * uy * uz2;
  m[midx(2, 2, 1)] = c4 * rho * uz + rho * c2 * uz * (ux2 + uy2) + rho * ux2 * uy2 * uz;
  m[midx(2, 2, 2)] = c6 * rho + rho * c4 * (ux2 + uy2 + uz2) + rho * c2 * (ux2 * uy2 + uy2 * uz2 + ux2 * uz2) +
                     rho * ux2 * uy2 * uz2;
}

static void matvec(const double *M, const double *x, double *y) {
  for (int i = 0; i < NQ; ++i) {
    double acc = 0.0;
    for (int j = 0; j < NQ; ++j) acc += M[i * NQ + j] * x[j];
    y[i] = acc;
  }
}

/* ---------------------------------------------------------------- context */

oracle_ctx *oracle_create(const oracle_params *p) {
  oracle_ctx *c = (oracle_ctx *)calloc(1, sizeof(oracle_ctx));
  if (!c) return NULL;
  c->p = *p;
  oracle_velocities(p->r, p->s, &c->e[0][0]);
  oracle_Q(p->r, p->s, c->Q);
  if (oracle_invert27(c->Q, c->Qinv) != 0) {
    free(c);
    return NULL;
  }
  oracle_opposite(c->opp);
  return c;
}

void oracle_destroy(oracle_ctx *c) { free(c); }

/* Replace the body force (time-periodic forcing F = F_m cos(omega t)). */
void oracle_set_force(oracle_ctx *c, const double *F) {
  for (int d = 0; d < 3; ++d) c->p.force[d] = F[d];
}

const double *oracle_ctx_Qinv(const oracle_ctx *c) { return c->Qinv; }

/* f^eq = Q^-1 m^eq with m^eq from Eq. 10 (the procedure stated at P:L759). */
void oracle_feq(const oracle_ctx *c, double rho, const double *u, double *feq) {
  double meq[NQ];
  oracle_raw_equilibria(rho, u, c->p.cs2, meq);
  matvec(c->Qinv, meq, feq);
}

/* ------------------------------------------------------------- collision */

/* One node: f (pre-collision, time t) -> f~ (post-collision), following the
 * step list of P:L687-729 with App D for the relaxation. */
void oracle_collide_g(const oracle_ctx *c, const double *f, const double *grad_rho, double *ft);
void oracle_collide_raw_g(const oracle_ctx *c, const double *f, const double *grad_rho, double *ft);

void oracle_collide(const oracle_ctx *c, const double *f, double *ft) { oracle_collide_g(c, f, NULL, ft); }

/* Singular strain-rate system (reading R17): a node whose
 * closed-form denominators of P:L1199-1203 -- the determinant of the 3x3
 * system in the printed d_x u_x, and C_sy, C_sz of the back-substitution --
 * fall below 1e-12 rho cs2 in magnitude is counted here (the step still
 * completes, as in the GPU path, which reports LBM_ESINGULAR). */
static int64_t g_singular = 0;
int64_t oracle_singular_count(void) { return g_singular; }
void oracle_singular_reset(void) { g_singular = 0; }
static void note_singular(double D, double Csy, double Csz, double rho, double cs2) {
  const double thr = 1e-12 * rho * cs2;
  if (fabs(D) < thr || fabs(Csy) < thr || fabs(Csz) < thr) g_singular++;
}

/* grad_rho: density gradient at the node for CORR_FULL_FD (NULL: zero). */
void oracle_collide_g(const oracle_ctx *c, const double *f, const double *grad_rho, double *ft) {
  const oracle_params *p = &c->p;
  const double cs2 = p->cs2, r2 = p->r * p->r, s2 = p->s * p->s;
  const double wn = p->omega_nu, wx = p->omega_xi, w1 = p->omega_1, wh = p->omega_high;
  double rho, u[3];
  oracle_hydro(&c->e[0][0], f, p->force, &rho, u);
  const double ux = u[0], uy = u[1], uz = u[2];

  /* m^c = F S P f: central moments by their definition, Eq. 3a */
  double k[NQ];
  oracle_central_moments(&c->e[0][0], f, u, k);
#define K(m, n, p_) k[midx(m, n, p_)]

  /* App D, combine with B */
  double k2s = K(2, 0, 0) + K(0, 2, 0) + K(0, 0, 2);
  double k2d1 = K(2, 0, 0) - K(0, 2, 0);
  double k2d2 = K(2, 0, 0) - K(0, 0, 2);
  double k3s1 = K(1, 2, 0) + K(1, 0, 2), k3m1 = K(1, 2, 0) - K(1, 0, 2);
  double k3s2 = K(2, 1, 0) + K(0, 1, 2), k3m2 = K(2, 1, 0) - K(0, 1, 2);
  double k3s3 = K(2, 0, 1) + K(0, 2, 1), k3m3 = K(2, 0, 1) - K(0, 2, 1);
  double k4s = K(2, 2, 0) + K(2, 0, 2) + K(0, 2, 2);
  double k4d1 = K(2, 2, 0) + K(2, 0, 2) - K(0, 2, 2);
  double k4d2 = K(2, 2, 0) - K(2, 0, 2);

  /* effective equilibria of the second-order diagonal group, Eq. 63
   * with the coefficients of P:L1171-1180 and local strain rates of P:L1183-1203. */
  double k2s_eq = 3.0 * cs2 * rho, k2d1_eq = 0.0, k2d2_eq = 0.0;
  if (p->corrections != CORR_OFF) {
    const double g = (p->corrections == CORR_FULL_LOCAL || FD_MODE(p->corrections)) ? 1.0 : 0.0; /* aliasing (3u^2) terms */
    const double an = 1.0 / wn - 0.5, ab = 1.0 / wx - 0.5;
    double th_sx = -rho * (g * 3.0 * ux * ux + 3.0 * cs2 - 1.0) * an;
    double th_bx = -rho * (g * 3.0 * ux * ux + 3.0 * cs2 - 1.0) * ab;
    double th_sy = -rho * (g * 3.0 * uy * uy + 3.0 * cs2 - r2) * an;
    double th_by = -rho * (g * 3.0 * uy * uy + 3.0 * cs2 - r2) * ab;
    double th_sz = -rho * (g * 3.0 * uz * uz + 3.0 * cs2 - s2) * an;
    double th_bz = -rho * (g * 3.0 * uz * uz + 3.0 * cs2 - s2) * ab;
    /* density-gradient terms: only in CORR_FULL_FD
     * (reading R1: FULL_LOCAL and LOW_MACH set lambda = e_rho = 0) */
    double gx = 0.0, gy = 0.0, gz = 0.0;
    if (FD_MODE(p->corrections) && grad_rho) {
      gx = grad_rho[0];
      gy = grad_rho[1];
      gz = grad_rho[2];
    }
    double lam_sx = -(3.0 * cs2 - 1.0) * an * ux, lam_bx = -(3.0 * cs2 - 1.0) * ab * ux;
    double lam_sy = +(3.0 * cs2 - r2) * an * uy, lam_by = -(3.0 * cs2 - r2) * ab * uy;
    double lam_sz = +(3.0 * cs2 - s2) * an * uz, lam_bz = -(3.0 * cs2 - s2) * ab * uz;
    double A = 0.5 * (3.0 * cs2 - 1.0) * ux, B = 0.5 * (3.0 * cs2 - r2) * uy, C = 0.5 * (3.0 * cs2 - s2) * uz;
    double e_sr1 = -A * gx + B * gy, e_sr2 = -A * gx + C * gz, e_br = -A * gx - B * gy - C * gz;
    double Rb = k2s - 3.0 * cs2 * rho + e_br, Rs1 = k2d1 + e_sr1, Rs2 = k2d2 + e_sr2;
    double Csx = (-2.0 * cs2 / wn + (3.0 * cs2 - 1.0) / 2.0 + g * 3.0 * ux * ux / 2.0) * rho;
    double Cbx = (-2.0 * cs2 / wx + (3.0 * cs2 - 1.0) / 2.0 + g * 3.0 * ux * ux / 2.0) * rho;
    double Csy = (2.0 * cs2 / wn - (3.0 * cs2 - r2) / 2.0 - g * 3.0 * uy * uy / 2.0) * rho;
    double Cby = (-2.0 * cs2 / wx + (3.0 * cs2 - r2) / 2.0 + g * 3.0 * uy * uy / 2.0) * rho;
    double Csz = (2.0 * cs2 / wn - (3.0 * cs2 - s2) / 2.0 - g * 3.0 * uz * uz / 2.0) * rho;
    double Cbz = (-2.0 * cs2 / wx + (3.0 * cs2 - s2) / 2.0 + g * 3.0 * uz * uz / 2.0) * rho;
    note_singular(-Csx * Csz * Cby - Csy * (Csx * Cbz - Csz * Cbx), Csy, Csz, rho, cs2);
    double dxux = (-Csz * Cby * Rs1 - Csy * (Cbz * Rs2 - Csz * Rb)) /
                  (-Csx * Csz * Cby - Csy * (Csx * Cbz - Csz * Cbx));
    double dyuy = (Rs1 - Csx * dxux) / Csy;
    double dzuz = (Rs2 - Csx * dxux) / Csz;
    k2s_eq = 3.0 * cs2 * rho + (th_bx * dxux + th_by * dyuy + th_bz * dzuz + lam_bx * gx + lam_by * gy + lam_bz * gz);
    k2d1_eq = th_sx * dxux - th_sy * dyuy + lam_sx * gx + lam_sy * gy;
    k2d2_eq = th_sx * dxux - th_sz * dzuz + lam_sx * gx + lam_sz * gz;
  }
  /* higher-order equilibria, Eq. 64 */
  const double c4r = cs2 * cs2 * rho, c6r = cs2 * cs2 * cs2 * rho;

  /* relaxation; all higher-order rates = omega_high */
  double kt[NQ];
#define KT(m, n, p_) kt[midx(m, n, p_)]
  KT(0, 0, 0) = K(0, 0, 0);
  KT(1, 0, 0) = K(1, 0, 0) + w1 * (0.0 - K(1, 0, 0)) + (1.0 - w1 / 2.0) * p->force[0];
  KT(0, 1, 0) = K(0, 1, 0) + w1 * (0.0 - K(0, 1, 0)) + (1.0 - w1 / 2.0) * p->force[1];
  KT(0, 0, 1) = K(0, 0, 1) + w1 * (0.0 - K(0, 0, 1)) + (1.0 - w1 / 2.0) * p->force[2];
  KT(1, 1, 0) = K(1, 1, 0) + wn * (0.0 - K(1, 1, 0));
  KT(1, 0, 1) = K(1, 0, 1) + wn * (0.0 - K(1, 0, 1));
  KT(0, 1, 1) = K(0, 1, 1) + wn * (0.0 - K(0, 1, 1));
  double k2d1t = k2d1 + wn * (k2d1_eq - k2d1);
  double k2d2t = k2d2 + wn * (k2d2_eq - k2d2);
  double k2st = k2s + wx * (k2s_eq - k2s);
  double k3s1t = k3s1 + wh * (0.0 - k3s1), k3m1t = k3m1 + wh * (0.0 - k3m1);
  double k3s2t = k3s2 + wh * (0.0 - k3s2), k3m2t = k3m2 + wh * (0.0 - k3m2);
  double k3s3t = k3s3 + wh * (0.0 - k3s3), k3m3t = k3m3 + wh * (0.0 - k3m3);
  KT(1, 1, 1) = K(1, 1, 1) + wh * (0.0 - K(1, 1, 1));
  KT(2, 1, 1) = K(2, 1, 1) + wh * (0.0 - K(2, 1, 1));
  KT(1, 2, 1) = K(1, 2, 1) + wh * (0.0 - K(1, 2, 1));
  KT(1, 1, 2) = K(1, 1, 2) + wh * (0.0 - K(1, 1, 2));
  double k4st = k4s + wh * (3.0 * c4r - k4s);
  double k4d1t = k4d1 + wh * (c4r - k4d1);
  double k4d2t = k4d2 + wh * (0.0 - k4d2);
  KT(1, 2, 2) = K(1, 2, 2) + wh * (0.0 - K(1, 2, 2));
  KT(2, 1, 2) = K(2, 1, 2) + wh * (0.0 - K(2, 1, 2));
  KT(2, 2, 1) = K(2, 2, 1) + wh * (0.0 - K(2, 2, 1));
  KT(2, 2, 2) = K(2, 2, 2) + wh * (c6r - K(2, 2, 2));

  /* segregate with B^-1 */
  KT(2, 0, 0) = (k2st + k2d1t + k2d2t) / 3.0;
  KT(0, 2, 0) = (k2st - 2.0 * k2d1t + k2d2t) / 3.0;
  KT(0, 0, 2) = (k2st + k2d1t - 2.0 * k2d2t) / 3.0;
  KT(1, 2, 0) = (k3s1t + k3m1t) / 2.0;
  KT(1, 0, 2) = (k3s1t - k3m1t) / 2.0;
  KT(2, 1, 0) = (k3s2t + k3m2t) / 2.0;
  KT(0, 1, 2) = (k3s2t - k3m2t) / 2.0;
  KT(2, 0, 1) = (k3s3t + k3m3t) / 2.0;
  KT(0, 2, 1) = (k3s3t - k3m3t) / 2.0;
  KT(2, 2, 0) = (k4st + k4d1t + 2.0 * k4d2t) / 4.0;
  KT(2, 0, 2) = (k4st + k4d1t - 2.0 * k4d2t) / 4.0;
  KT(0, 2, 2) = (k4st - k4d1t) / 2.0;
#undef K
#undef KT

  /* m~ = F^-1 m~^c (binomial), then f~ = Q^-1 m~ (= P^-1 S^-1 m~) */
  double mt[NQ];
  oracle_frame(kt, u, mt);
  matvec(c->Qinv, mt, ft);
}

/* Eq. 11: raw moments of the source term, zero from third order on. */
void oracle_raw_source(const double *u, const double *F, double *phi) {
  for (int j = 0; j < NQ; ++j) phi[j] = 0.0;
  phi[midx(1, 0, 0)] = F[0];
  phi[midx(0, 1, 0)] = F[1];
  phi[midx(0, 0, 1)] = F[2];
  phi[midx(1, 1, 0)] = F[0] * u[1] + F[1] * u[0];
  phi[midx(1, 0, 1)] = F[0] * u[2] + F[2] * u[0];
  phi[midx(0, 1, 1)] = F[1] * u[2] + F[2] * u[1];
  phi[midx(2, 0, 0)] = 2.0 * F[0] * u[0];
  phi[midx(0, 2, 0)] = 2.0 * F[1] * u[1];
  phi[midx(0, 0, 2)] = 2.0 * F[2] * u[2];
}

/* 3DCRM-LBM (P:L1011 and remark (ii) of P:L744): the raw-moment scheme of
 * Eq. LBErawmomentcuboidlattice,
 *   m = S P f,  m~ = m + B^-1 {Lambda (B m^eq - B m) + (I - Lambda/2) B Phi},  f~ = P^-1 S^-1 m~,
 * with m^eq from Eq. 10, Phi from Eq. 11, the same B grouping and relaxation
 * rates as App D and "the same corrections via the extended moment equilibria"
 * (P:L744): the second-order diagonal equilibria carry the theta terms of
 * P:L1171-1178, and the strain rates come from the raw non-equilibrium moments
 * n^(1) through the same C/R system. */
void oracle_collide_raw(const oracle_ctx *c, const double *f, double *ft) { oracle_collide_raw_g(c, f, NULL, ft); }

void oracle_collide_raw_g(const oracle_ctx *c, const double *f, const double *grad_rho, double *ft) {
  const oracle_params *p = &c->p;
  const double cs2 = p->cs2, r2 = p->r * p->r, s2 = p->s * p->s;
  const double wn = p->omega_nu, wx = p->omega_xi, w1 = p->omega_1, wh = p->omega_high;
  double rho, u[3];
  oracle_hydro(&c->e[0][0], f, p->force, &rho, u);
  const double ux = u[0], uy = u[1], uz = u[2];
  double m[NQ], meq[NQ], phi[NQ], mt[NQ];
  matvec(c->Q, f, m); /* m = Q f = S P f (Eq. 56, 58) */
  oracle_raw_equilibria(rho, u, cs2, meq);
  oracle_raw_source(u, p->force, phi);
#define M(a, b, c_) m[midx(a, b, c_)]
#define E(a, b, c_) meq[midx(a, b, c_)]
#define PH(a, b, c_) phi[midx(a, b, c_)]
#define MT(a, b, c_) mt[midx(a, b, c_)]
  /* B: combine, for m, m^eq and Phi alike */
  double k2s = M(2, 0, 0) + M(0, 2, 0) + M(0, 0, 2), e2s = E(2, 0, 0) + E(0, 2, 0) + E(0, 0, 2);
  double k2d1 = M(2, 0, 0) - M(0, 2, 0), e2d1 = E(2, 0, 0) - E(0, 2, 0);
  double k2d2 = M(2, 0, 0) - M(0, 0, 2), e2d2 = E(2, 0, 0) - E(0, 0, 2);
  double p2s = PH(2, 0, 0) + PH(0, 2, 0) + PH(0, 0, 2), p2d1 = PH(2, 0, 0) - PH(0, 2, 0),
         p2d2 = PH(2, 0, 0) - PH(0, 0, 2);
  if (p->corrections != CORR_OFF) {
    const double g = (p->corrections == CORR_FULL_LOCAL || FD_MODE(p->corrections)) ? 1.0 : 0.0;
    const double an = 1.0 / wn - 0.5, ab = 1.0 / wx - 0.5;
    double th_sx = -rho * (g * 3.0 * ux * ux + 3.0 * cs2 - 1.0) * an;
    double th_bx = -rho * (g * 3.0 * ux * ux + 3.0 * cs2 - 1.0) * ab;
    double th_sy = -rho * (g * 3.0 * uy * uy + 3.0 * cs2 - r2) * an;
    double th_by = -rho * (g * 3.0 * uy * uy + 3.0 * cs2 - r2) * ab;
    double th_sz = -rho * (g * 3.0 * uz * uz + 3.0 * cs2 - s2) * an;
    double th_bz = -rho * (g * 3.0 * uz * uz + 3.0 * cs2 - s2) * ab;
    double gx = 0.0, gy = 0.0, gz = 0.0;
    if (FD_MODE(p->corrections) && grad_rho) {
      gx = grad_rho[0];
      gy = grad_rho[1];
      gz = grad_rho[2];
    }
    double lam_sx = -(3.0 * cs2 - 1.0) * an * ux, lam_bx = -(3.0 * cs2 - 1.0) * ab * ux;
    double lam_sy = +(3.0 * cs2 - r2) * an * uy, lam_by = -(3.0 * cs2 - r2) * ab * uy;
    double lam_sz = +(3.0 * cs2 - s2) * an * uz, lam_bz = -(3.0 * cs2 - s2) * ab * uz;
    double A = 0.5 * (3.0 * cs2 - 1.0) * ux, B = 0.5 * (3.0 * cs2 - r2) * uy, C = 0.5 * (3.0 * cs2 - s2) * uz;
    /* raw non-equilibrium moments n^(1) plus e_rho */
    double Rb = k2s - e2s + (-A * gx - B * gy - C * gz), Rs1 = k2d1 - e2d1 + (-A * gx + B * gy),
           Rs2 = k2d2 - e2d2 + (-A * gx + C * gz);
    double Csx = (-2.0 * cs2 / wn + (3.0 * cs2 - 1.0) / 2.0 + g * 3.0 * ux * ux / 2.0) * rho;
    double Cbx = (-2.0 * cs2 / wx + (3.0 * cs2 - 1.0) / 2.0 + g * 3.0 * ux * ux / 2.0) * rho;
    double Csy = (2.0 * cs2 / wn - (3.0 * cs2 - r2) / 2.0 - g * 3.0 * uy * uy / 2.0) * rho;
    double Cby = (-2.0 * cs2 / wx + (3.0 * cs2 - r2) / 2.0 + g * 3.0 * uy * uy / 2.0) * rho;
    double Csz = (2.0 * cs2 / wn - (3.0 * cs2 - s2) / 2.0 - g * 3.0 * uz * uz / 2.0) * rho;
    double Cbz = (-2.0 * cs2 / wx + (3.0 * cs2 - s2) / 2.0 + g * 3.0 * uz * uz / 2.0) * rho;
    note_singular(-Csx * Csz * Cby - Csy * (Csx * Cbz - Csz * Cbx), Csy, Csz, rho, cs2);
    double dxux = (-Csz * Cby * Rs1 - Csy * (Cbz * Rs2 - Csz * Rb)) /
                  (-Csx * Csz * Cby - Csy * (Csx * Cbz - Csz * Cbx));
    double dyuy = (Rs1 - Csx * dxux) / Csy;
    double dzuz = (Rs2 - Csx * dxux) / Csz;
    e2s += th_bx * dxux + th_by * dyuy + th_bz * dzuz + lam_bx * gx + lam_by * gy + lam_bz * gz;
    e2d1 += th_sx * dxux - th_sy * dyuy + lam_sx * gx + lam_sy * gy;
    e2d2 += th_sx * dxux - th_sz * dzuz + lam_sx * gx + lam_sz * gz;
  }
  double k3s1 = M(1, 2, 0) + M(1, 0, 2), k3m1 = M(1, 2, 0) - M(1, 0, 2);
  double k3s2 = M(2, 1, 0) + M(0, 1, 2), k3m2 = M(2, 1, 0) - M(0, 1, 2);
  double k3s3 = M(2, 0, 1) + M(0, 2, 1), k3m3 = M(2, 0, 1) - M(0, 2, 1);
  double e3s1 = E(1, 2, 0) + E(1, 0, 2), e3m1 = E(1, 2, 0) - E(1, 0, 2);
  double e3s2 = E(2, 1, 0) + E(0, 1, 2), e3m2 = E(2, 1, 0) - E(0, 1, 2);
  double e3s3 = E(2, 0, 1) + E(0, 2, 1), e3m3 = E(2, 0, 1) - E(0, 2, 1);
  double k4s = M(2, 2, 0) + M(2, 0, 2) + M(0, 2, 2), e4s = E(2, 2, 0) + E(2, 0, 2) + E(0, 2, 2);
  double k4d1 = M(2, 2, 0) + M(2, 0, 2) - M(0, 2, 2), e4d1 = E(2, 2, 0) + E(2, 0, 2) - E(0, 2, 2);
  double k4d2 = M(2, 2, 0) - M(2, 0, 2), e4d2 = E(2, 2, 0) - E(2, 0, 2);
  /* relaxation with sources (Phi is zero from third order on) */
  MT(0, 0, 0) = M(0, 0, 0);
  MT(1, 0, 0) = M(1, 0, 0) + w1 * (E(1, 0, 0) - M(1, 0, 0)) + (1.0 - w1 / 2.0) * PH(1, 0, 0);
  MT(0, 1, 0) = M(0, 1, 0) + w1 * (E(0, 1, 0) - M(0, 1, 0)) + (1.0 - w1 / 2.0) * PH(0, 1, 0);
  MT(0, 0, 1) = M(0, 0, 1) + w1 * (E(0, 0, 1) - M(0, 0, 1)) + (1.0 - w1 / 2.0) * PH(0, 0, 1);
  MT(1, 1, 0) = M(1, 1, 0) + wn * (E(1, 1, 0) - M(1, 1, 0)) + (1.0 - wn / 2.0) * PH(1, 1, 0);
  MT(1, 0, 1) = M(1, 0, 1) + wn * (E(1, 0, 1) - M(1, 0, 1)) + (1.0 - wn / 2.0) * PH(1, 0, 1);
  MT(0, 1, 1) = M(0, 1, 1) + wn * (E(0, 1, 1) - M(0, 1, 1)) + (1.0 - wn / 2.0) * PH(0, 1, 1);
  double k2st = k2s + wx * (e2s - k2s) + (1.0 - wx / 2.0) * p2s;
  double k2d1t = k2d1 + wn * (e2d1 - k2d1) + (1.0 - wn / 2.0) * p2d1;
  double k2d2t = k2d2 + wn * (e2d2 - k2d2) + (1.0 - wn / 2.0) * p2d2;
  double k3s1t = k3s1 + wh * (e3s1 - k3s1), k3m1t = k3m1 + wh * (e3m1 - k3m1);
  double k3s2t = k3s2 + wh * (e3s2 - k3s2), k3m2t = k3m2 + wh * (e3m2 - k3m2);
  double k3s3t = k3s3 + wh * (e3s3 - k3s3), k3m3t = k3m3 + wh * (e3m3 - k3m3);
  MT(1, 1, 1) = M(1, 1, 1) + wh * (E(1, 1, 1) - M(1, 1, 1));
  MT(2, 1, 1) = M(2, 1, 1) + wh * (E(2, 1, 1) - M(2, 1, 1));
  MT(1, 2, 1) = M(1, 2, 1) + wh * (E(1, 2, 1) - M(1, 2, 1));
  MT(1, 1, 2) = M(1, 1, 2) + wh * (E(1, 1, 2) - M(1, 1, 2));
  double k4st = k4s + wh * (e4s - k4s), k4d1t = k4d1 + wh * (e4d1 - k4d1), k4d2t = k4d2 + wh * (e4d2 - k4d2);
  MT(1, 2, 2) = M(1, 2, 2) + wh * (E(1, 2, 2) - M(1, 2, 2));
  MT(2, 1, 2) = M(2, 1, 2) + wh * (E(2, 1, 2) - M(2, 1, 2));
  MT(2, 2, 1) = M(2, 2, 1) + wh * (E(2, 2, 1) - M(2, 2, 1));
  MT(2, 2, 2) = M(2, 2, 2) + wh * (E(2, 2, 2) - M(2, 2, 2));
  /* B^-1 */
  MT(2, 0, 0) = (k2st + k2d1t + k2d2t) / 3.0;
  MT(0, 2, 0) = (k2st - 2.0 * k2d1t + k2d2t) / 3.0;
  MT(0, 0, 2) = (k2st + k2d1t - 2.0 * k2d2t) / 3.0;
  MT(1, 2, 0) = (k3s1t + k3m1t) / 2.0;
  MT(1, 0, 2) = (k3s1t - k3m1t) / 2.0;
  MT(2, 1, 0) = (k3s2t + k3m2t) / 2.0;
  MT(0, 1, 2) = (k3s2t - k3m2t) / 2.0;
  MT(2, 0, 1) = (k3s3t + k3m3t) / 2.0;
  MT(0, 2, 1) = (k3s3t - k3m3t) / 2.0;
  MT(2, 2, 0) = (k4st + k4d1t + 2.0 * k4d2t) / 4.0;
  MT(2, 0, 2) = (k4st + k4d1t - 2.0 * k4d2t) / 4.0;
  MT(0, 2, 2) = (k4st - k4d1t) / 2.0;
#undef M
#undef E
#undef PH
#undef MT
  matvec(c->Qinv, mt, ft); /* f~ = Q^-1 m~ = P^-1 S^-1 m~ */
}

/* ------------------------------------------------------------- boundaries */

/* Momentum-augmented halfway bounce-back term for the incoming direction q at
 * a node next to the moving +y wall:
 *   f_q(x_f, t+1) = f~_{qbar}(x_f, t) - [f^eq_{qbar}(x_w) - f^eq_q(x_w)],
 * with f^eq = Q^-1 m^eq, m^eq from Eq. 10 at rho_w = rho_f, u_w = (U, 0, 0).
 * Returns the bracketed correction with its sign, i.e. the value to ADD. */
double oracle_lid_term(const oracle_ctx *c, int q, double rho_f) {
  double uw[3] = {c->p.wall_u, 0.0, 0.0}, feq[NQ];
  oracle_feq(c, rho_f, uw, feq);
  int qb = c->opp[q];
  return -(feq[qb] - feq[q]);
}

static int64_t nid(const oracle_params *p, int x, int y, int z) {
  return ((int64_t)z * p->ny + y) * p->nx + x;
}

static int wrap(int v, int n) { return ((v % n) + n) % n; }

/* Pull the incoming population q of node (x,y,z) for time t+1 from the
 * post-collision field fs at time t, applying the wall rules. */
static double pull(const oracle_ctx *c, const double *fs, int x, int y, int z, int q) {
  const oracle_params *p = &c->p;
  const int64_t nn = (int64_t)p->nx * p->ny * p->nz;
  int e[3] = {EX[q], EY[q], EZ[q]};
  int n[3] = {p->nx, p->ny, p->nz};
  int xyz[3] = {x, y, z};
  int src[3];
  int noslip = 0, lid = 0, slip[3] = {0, 0, 0}, anyslip = 0;
  for (int d = 0; d < 3; ++d) {
    src[d] = xyz[d] - e[d];
    int face = -1;
    if (src[d] < 0) face = 2 * d;
    if (src[d] >= n[d]) face = 2 * d + 1;
    if (face < 0) continue;
    int t = p->bc[face];
    if (t == BC_BOUNCE_BACK || t == BC_MOVING_WALL) noslip = 1;
    if (t == BC_MOVING_WALL && face == 3) lid = 1;
    if (t == BC_FREE_SLIP) {
      slip[d] = 1;
      anyslip = 1;
    }
  }
  int64_t own = nid(p, x, y, z);
  if (noslip) {
    /* halfway bounce-back: f_q(x_f, t+1) = f~_{qbar}(x_f, t) (+ Eq. 69 term) */
    double v = fs[(int64_t)c->opp[q] * nn + own];
    if (lid) {
      double rho_f = 0.0; /* reading R4: rho_f = sum_b f~_b(x_f, t) */
      for (int b = 0; b < NQ; ++b) rho_f += fs[(int64_t)b * nn + own];
      v += oracle_lid_term(c, q, rho_f);
    }
    return v;
  }
  int qs = q;
  if (anyslip) {
    /* reading R7: specular reflection on the crossed free-slip axes */
    int em[3];
    for (int d = 0; d < 3; ++d) {
      em[d] = slip[d] ? -e[d] : e[d];
      src[d] = slip[d] ? xyz[d] : xyz[d] - e[d];
    }
    for (int b = 0; b < NQ; ++b)
      if (EX[b] == em[0] && EY[b] == em[1] && EZ[b] == em[2]) qs = b;
  }
  for (int d = 0; d < 3; ++d) src[d] = wrap(src[d], n[d]);
  return fs[(int64_t)qs * nn + nid(p, src[0], src[1], src[2])];
}

/* Isotropic second-order density gradient (reading R16):
 *   d_d rho(x) = (1/cs2) sum_a w_a e_ad rho(x + e_a),
 * w_a the cuboid rest weights (f^eq at rho = 1, u = 0), which satisfy
 * sum_a w_a e_a e_a = cs2 I.  A neighbour across a wall face is the mirror
 * image of that neighbour in the halfway wall, i.e. the node x + e_a with the
 * crossed components of e_a set to zero (a zero-normal-gradient ghost: the
 * wall-parallel gradient of a field linear along the wall stays exact);
 * periodic faces wrap. */
void oracle_density_gradient(const oracle_ctx *c, const double *rho, int x, int y, int z, double *g) {
  const oracle_params *p = &c->p;
  double w[NQ], u0[3] = {0.0, 0.0, 0.0};
  oracle_feq(c, 1.0, u0, w);
  int n[3] = {p->nx, p->ny, p->nz}, xyz[3] = {x, y, z};
  g[0] = g[1] = g[2] = 0.0;
  for (int a = 0; a < NQ; ++a) {
    int e[3] = {EX[a], EY[a], EZ[a]}, nb[3];
    for (int d = 0; d < 3; ++d) {
      nb[d] = xyz[d] + e[d];
      if (nb[d] < 0 || nb[d] >= n[d]) {
        int face = (nb[d] < 0) ? 2 * d : 2 * d + 1;
        nb[d] = (p->bc[face] != BC_PERIODIC) ? xyz[d] : wrap(nb[d], n[d]);
      }
    }
    double rn = rho[nid(p, nb[0], nb[1], nb[2])];
    for (int d = 0; d < 3; ++d) g[d] += w[a] * c->e[a][d] * rn;
  }
  for (int d = 0; d < 3; ++d) g[d] /= p->cs2;
}

/* One time step on the whole grid: fdst = collide(pull(fsrc)).  With
 * CORR_FULL_FD the step is done in two passes: pull every node and form the
 * same-time density field (reading R16), then collide with its isotropic
 * gradient.  With CORR_FULL_FD_LAG (reading R16b) the density field is that of
 * the stored state, rho(x, t) = sum_q f~_q(x, t) at every node (the density of
 * the previous collision: the collision conserves mass), one time level behind
 * the populations it corrects. */
void oracle_step(const oracle_ctx *c, const double *fsrc, double *fdst) {
  const oracle_params *p = &c->p;
  const int64_t nn = (int64_t)p->nx * p->ny * p->nz;
  double f[NQ], ft[NQ], g[3];
  const int fd = FD_MODE(p->corrections);
  const int lag = (p->corrections == CORR_FULL_FD_LAG);
  double *rho = NULL;
  if (fd) {
    rho = (double *)malloc(sizeof(double) * nn);
    for (int z = 0; z < p->nz; ++z)
      for (int y = 0; y < p->ny; ++y)
        for (int x = 0; x < p->nx; ++x) {
          double r0 = 0.0;
          for (int q = 0; q < NQ; ++q)
            r0 += lag ? fsrc[(int64_t)q * nn + nid(p, x, y, z)] : pull(c, fsrc, x, y, z, q);
          rho[nid(p, x, y, z)] = r0;
        }
  }
  for (int z = 0; z < p->nz; ++z)
    for (int y = 0; y < p->ny; ++y)
      for (int x = 0; x < p->nx; ++x) {
        for (int q = 0; q < NQ; ++q) f[q] = pull(c, fsrc, x, y, z, q);
        if (fd) oracle_density_gradient(c, rho, x, y, z, g);
        if (p->model == 1)
          oracle_collide_raw_g(c, f, fd ? g : NULL, ft);
        else
          oracle_collide_g(c, f, fd ? g : NULL, ft);
        int64_t i = nid(p, x, y, z);
        for (int q = 0; q < NQ; ++q) fdst[(int64_t)q * nn + i] = ft[q];
      }
  free(rho);
}

/* n steps, ping-ponging between f and tmp; result ends in f. */
void oracle_run(const oracle_ctx *c, double *f, double *tmp, int64_t nsteps) {
  const int64_t nn = (int64_t)c->p.nx * c->p.ny * c->p.nz;
  double *a = f, *b = tmp;
  for (int64_t t = 0; t < nsteps; ++t) {
    oracle_step(c, a, b);
    double *s = a;
    a = b;
    b = s;
  }
  if (a != f) memcpy(f, a, sizeof(double) * NQ * nn);
}

/* Reading R8: stored state f~(t0) = f^eq(rho0, u0 + F/(2 rho0)). */
void oracle_init(const oracle_ctx *c, const double *rho, const double *u, double *f) {
  const oracle_params *p = &c->p;
  const int64_t nn = (int64_t)p->nx * p->ny * p->nz;
  double feq[NQ];
  for (int64_t i = 0; i < nn; ++i) {
    double uu[3];
    for (int d = 0; d < 3; ++d) uu[d] = u[d * nn + i] + 0.5 * p->force[d] / rho[i];
    oracle_feq(c, rho[i], uu, feq);
    for (int q = 0; q < NQ; ++q) f[(int64_t)q * nn + i] = feq[q];
  }
}

/* rho and u at the stored (post-collision) time level: the collision conserves
 * k'_000 and adds F to the first raw moments, hence
 * u = (sum f~ e - F/2)/rho. */
void oracle_macroscopic(const oracle_ctx *c, const double *f, double *rho, double *u) {
  const oracle_params *p = &c->p;
  const int64_t nn = (int64_t)p->nx * p->ny * p->nz;
  for (int64_t i = 0; i < nn; ++i) {
    double r0 = 0.0, j[3] = {0.0, 0.0, 0.0};
    for (int q = 0; q < NQ; ++q) {
      double v = f[(int64_t)q * nn + i];
      r0 += v;
      for (int d = 0; d < 3; ++d) j[d] += v * c->e[q][d];
    }
    rho[i] = r0;
    for (int d = 0; d < 3; ++d) u[d * nn + i] = (j[d] - 0.5 * p->force[d]) / r0;
  }
}
