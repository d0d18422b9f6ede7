// cm_stream.cuh -- streaming of the 3D cuboid central-moment LBM: the pull
// sources of a node with the wall rules (halfway bounce-back, Eq. 69 lid,
// free-slip), the isotropic density gradient of FULL_FD, and the store
// policies (own node, AA reversed / push, peer-memory halo).  "P:Lnnn"
// cites /root/reference/PAPER.md line nnn.
#pragma once

#include "cm_common.cuh"

namespace lbm {

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

// is node (x, y, z) next to a wall face (bounce-back, moving or free-slip)?
// (the predicate of PullSrc::wall)
__device__ __forceinline__ bool wall_adjacent(const Consts& c, int x, int y, int z) {
  if (!c.has_walls) return false;
  auto w = [](int fk) { return fk >= FK_BOUNCE && fk <= FK_SLIP; };
  return (x == 0 && w(c.face[0])) || (x == c.nx - 1 && w(c.face[1])) || (y == 0 && w(c.face[2])) ||
         (y == c.ny - 1 && w(c.face[3])) || (z == 0 && w(c.face[4])) || (z == c.nzl - 1 && w(c.face[5]));
}

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
    if (REV) {
      // AA odd step: 26 of the node's 27 slots belong to the neighbour threads
      // that pull from them and then push into them (the bijection of k_aa), so
      // they may already be overwritten; rho_f = sum f~(x_f, t), formed by the
      // even step that stored them (StoreRev), or by k_aa_lid_rho after
      // init/set_populations, in the same q order as below
      rho_f = c.aa_lid_rho[z * nx + x];
    } else {
#pragma unroll
      for (int q = 0; q < 27; ++q) rho_f += ldg(LBM_CHECK_LD(src, p0 + q * c.nxy + own, c));
    }
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
// neighbour across a wall face is its mirror image in the halfway wall: the
// offset along the crossed axes is zeroed (zero-normal-gradient ghost).  rf has
// the population-buffer plane structure: rf[(z_local + 1) * nxy + y * nx + x].
// rho_at(i, j, k) = density at offset (i-1, j-1, k-1) from the node (never
// called for a neighbour across a wall); identical arithmetic for every source.
// NOWALL: the caller knows no face of the node is a wall (no mirror images)
template <class RhoAt, bool NOWALL = false>
__device__ __forceinline__ void density_gradient_g(const Consts& c, int x, int y, int z, RhoAt rho_at, double& gx,
                                                   double& gy, double& gz) {
  auto is_wall = [](int fk) { return fk >= FK_BOUNCE && fk <= FK_SLIP; };
  const bool cx[3] = {!NOWALL && x == 0 && is_wall(c.face[0]), false, !NOWALL && x == c.nx - 1 && is_wall(c.face[1])};
  const bool cy[3] = {!NOWALL && y == 0 && is_wall(c.face[2]), false, !NOWALL && y == c.ny - 1 && is_wall(c.face[3])};
  const bool cz[3] = {!NOWALL && z == 0 && is_wall(c.face[4]), false,
                      !NOWALL && z == c.nzl - 1 && is_wall(c.face[5])};
  double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        if (i == 1 && j == 1 && k == 1) continue;
        const double v = rho_at(cx[i] ? 1 : i, cy[j] ? 1 : j, cz[k] ? 1 : k);
        // explicit fused multiply-adds: the same rounding in every kernel that
        // inlines this, whatever the compiler's contraction choices
        if (i != 1) sx = __fma_rn((i == 2 ? 1.0 : -1.0) * c.phy[j] * c.phz[k], v, sx);
        if (j != 1) sy = __fma_rn((j == 2 ? 1.0 : -1.0) * c.phx[i] * c.phz[k], v, sy);
        if (k != 1) sz = __fma_rn((k == 2 ? 1.0 : -1.0) * c.phx[i] * c.phy[j], v, sz);
      }
  gx = 0.5 * sx;
  gy = c.h1y * sy;
  gz = c.h1z * sz;
}

__device__ __forceinline__ void density_gradient(const double* __restrict__ rf, const Consts& c, int x, int y,
                                                 int z, double& gx, double& gy, double& gz) {
  const int nx = c.nx;
  // warp-uniform interior: no lane wraps a periodic face or touches a wall, so
  // the 26 neighbours are the node's address plus warp-uniform offsets
  const bool inner = x > 0 && x < nx - 1 && y > 0 && y < c.ny - 1 && !(z == 0 && c.face[4] == FK_WRAP) &&
                     !(z == c.nzl - 1 && c.face[5] == FK_WRAP) && !wall_adjacent(c, x, y, z);
  if (__all_sync(__activemask(), inner)) {
    const double* b = rf + (long long)(z + 1) * c.nxy + (y * nx + x);
    auto at = [&](int i, int j, int k) { return __ldg(b + ((long long)(k - 1) * c.nxy + ((j - 1) * nx + (i - 1)))); };
    density_gradient_g<decltype(at), true>(c, x, y, z, at, gx, gy, gz);
    return;
  }
  const int xs[3] = {(x == 0) ? nx - 1 : x - 1, x, (x == nx - 1) ? 0 : x + 1};
  const int ys[3] = {((y == 0) ? c.ny - 1 : y - 1) * nx, y * nx, ((y == c.ny - 1) ? 0 : y + 1) * nx};
  int zm = z - 1, zp = z + 1;
  if (z == 0 && c.face[4] == FK_WRAP) zm = c.nzl - 1;
  if (z == c.nzl - 1 && c.face[5] == FK_WRAP) zp = 0;
  const long long zb[3] = {(long long)(zm + 1) * c.nxy, (long long)(z + 1) * c.nxy, (long long)(zp + 1) * c.nxy};
  density_gradient_g(
      c, x, y, z, [&](int i, int j, int k) { return __ldg(rf + zb[k] + ys[j] + xs[i]); }, gx, gy, gz);
}

// --------------------------------------------------------- store policies
// Where the post-collision populations f~_q(x) go:
//   StoreOwn  (two-buffer "AB" pull scheme): own node, slot q of the other buffer;
//   StoreRev  (AA even step): own node, slot 26 - q of the same buffer;
//   StorePush (AA odd step): the slot whose next pull reads it (push with the
//             wall rules; the exact inverse of gather()).
// RHO (the density-gradient kernels only): also form the node's density for
// FULL_FD_LAG's next step as the sum of the STORED values in q order (what
// k_stored_rho forms after a set_populations, so a checkpoint resumes bit for
// bit); rho_out == nullptr at run time for the same-time FULL_FD.  A
// compile-time flag, so the plain kernels carry no per-store test.
template <typename T, bool RHO = false>
struct StoreOwn {
  T* base;
  T* out;
  int nxy;
  const Consts* c;
  double* rho_out = nullptr;
  double acc = 0.0;
  __device__ __forceinline__ void begin(double) {}
  __device__ __forceinline__ void operator()(int q, double v) {
    stcs<T>(LBM_CHECK_ST(base, out + q * nxy, *c), v);
    if constexpr (RHO) {
      if (rho_out) {
        acc += (double)(T)v;
        if (q == 26) *rho_out = acc;
      }
    }
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


}  // namespace lbm
