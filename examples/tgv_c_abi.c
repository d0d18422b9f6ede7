/* Plain-C use of the C ABI (include/lbm_cuboid.h), no Python, no torch:
 * BASELINE config 1 (Taylor-Green vortex, 32x32x16, r = 1, s = 2, nu = 0.01),
 * library-owned stream and buffers.  Writes rho and u after `steps` steps as raw
 * fp64 to the output file and prints the kinetic-energy ratio.
 *
 *   gcc -O2 -std=c99 -I include examples/tgv_c_abi.c -o build/tgv_c_abi \
 *       -L paper_2107_14774_b200 -llbm_cuboid -Wl,-rpath,$PWD/paper_2107_14774_b200 -lm
 *   ./build/tgv_c_abi 200 out.bin
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "lbm_cuboid.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    int rc_ = (x);                                                            \
    if (rc_ != LBM_OK) {                                                      \
      fprintf(stderr, "%s failed: %d %s\n", #x, rc_, lbm_cuboid_last_error()); \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(int argc, char **argv) {
  const int steps = argc > 1 ? atoi(argv[1]) : 200;
  const char *out = argc > 2 ? argv[2] : NULL;
  lbm_cuboid_params p;
  lbm_cuboid_default_params(&p);
  p.nx = 32;
  p.ny = 32;
  p.nz = 16;
  p.r = 1.0;
  p.s = 2.0;
  p.cs2 = 1.0 / 3.0;
  p.omega_nu = 1.0 / (0.01 / p.cs2 + 0.5); /* Eq. 53 */
  lbm_cuboid_t *h = NULL;
  CHECK(lbm_cuboid_create(&p, &h));
  const size_t n = (size_t)p.nx * p.ny * p.nz;
  double *rho = malloc(n * sizeof(double)), *u = malloc(3 * n * sizeof(double));
  const double pi = acos(-1.0), u0 = 0.02;
  for (int z = 0; z < p.nz; ++z)
    for (int y = 0; y < p.ny; ++y)
      for (int x = 0; x < p.nx; ++x) {
        const size_t i = ((size_t)z * p.ny + y) * p.nx + x;
        const double X = 2 * pi * x / p.nx, Y = 2 * pi * y / p.ny, Z = 2 * pi * z / p.nz;
        u[i] = u0 * sin(X) * cos(Y) * cos(Z);
        u[n + i] = -u0 * cos(X) * sin(Y) * cos(Z);
        u[2 * n + i] = 0.0;
        rho[i] = 1.0 + (u0 * u0 / 16.0) * (cos(2 * X) + cos(2 * Y)) * (cos(2 * Z) + 2.0) / p.cs2;
      }
  CHECK(lbm_cuboid_init_fields(h, rho, u));
  double d0[7], d1[7];
  CHECK(lbm_cuboid_check(h, d0));
  CHECK(lbm_cuboid_step(h, steps));
  CHECK(lbm_cuboid_sync(h));
  CHECK(lbm_cuboid_check(h, d1));
  CHECK(lbm_cuboid_get_macroscopic(h, rho, u));
  printf("{\"steps\": %d, \"ke_ratio\": %.12f, \"mass_change\": %.3e}\n", steps, d1[4] / d0[4], d1[0] - d0[0]);
  if (out) {
    FILE *fh = fopen(out, "wb");
    fwrite(rho, sizeof(double), n, fh);
    fwrite(u, sizeof(double), 3 * n, fh);
    fclose(fh);
  }
  CHECK(lbm_cuboid_destroy(h));
  free(rho);
  free(u);
  return 0;
}
