// Practical ceiling of the D3Q27 pull pattern on this GPU: the same 27 shifted
// loads and 27 coalesced stores per node as k_collide_stream_paper (same layout,
// grid, block size), with no arithmetic (f_out[q](x) = f_in[q](x - e_q), periodic).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/pull_copy_ceiling.cu -o build/pull_copy_ceiling
#include <cstdio>
#include <cuda_runtime.h>

template <bool COMPUTE_NOTHING>
__global__ void __launch_bounds__(128) pull_copy(const double* __restrict__ src, double* __restrict__ dst, int nx,
                                                 int ny, int nz) {
  const int nxy = nx * ny;
  const int idx = blockIdx.x * 128 + threadIdx.x;
  if (idx >= nxy) return;
  const int y = idx / nx, x = idx - y * nx, z = blockIdx.y;
  const long long plane = 27LL * nxy;
  const int sx[3] = {x == nx - 1 ? 0 : x + 1, x, x == 0 ? nx - 1 : x - 1};
  const int sy[3] = {(y == ny - 1 ? 0 : y + 1) * nx, y * nx, (y == 0 ? ny - 1 : y - 1) * nx};
  const int zz[3] = {z == nz - 1 ? 0 : z + 1, z, z == 0 ? nz - 1 : z - 1};
  double f[27];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int q = i + 3 * j + 9 * k;
        f[q] = __ldg(src + (zz[k] + 1) * plane + q * nxy + sy[j] + sx[i]);
      }
  double* out = dst + (z + 1) * plane + idx;
#pragma unroll
  for (int q = 0; q < 27; ++q) __stcs(out + q * nxy, f[q]);
}

// plain vectorized copy of the same number of bytes (16-B loads/stores)
__global__ void __launch_bounds__(256) plain_copy(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * (size_t)256 + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * 256;
  for (; i < n; i += stride) __stcs(dst + i, __ldg(src + i));
}

// 27 aligned streams (no shifts), same structure as the pull copy
__global__ void __launch_bounds__(128) aligned27(const double* __restrict__ src, double* __restrict__ dst, int nx,
                                                 int ny) {
  const int nxy = nx * ny;
  const int idx = blockIdx.x * 128 + threadIdx.x;
  if (idx >= nxy) return;
  const long long plane = 27LL * nxy;
  const double* in = src + (blockIdx.y + 1) * plane + idx;
  double f[27];
#pragma unroll
  for (int q = 0; q < 27; ++q) f[q] = __ldg(in + q * nxy);
  double* out = dst + (blockIdx.y + 1) * plane + idx;
#pragma unroll
  for (int q = 0; q < 27; ++q) __stcs(out + q * nxy, f[q]);
}

int main() {
  const int nx = 512, ny = 512, nz = 512;
  const size_t elems = 27ull * nx * ny * (nz + 2);
  double *a, *b;
  if (cudaMalloc(&a, elems * 8) || cudaMalloc(&b, elems * 8)) { printf("alloc failed\n"); return 1; }
  cudaMemset(a, 0, elems * 8);
  cudaMemset(b, 0, elems * 8);
  dim3 g((nx * ny + 127) / 128, nz);
  for (int w = 0; w < 3; ++w) pull_copy<true><<<g, 128>>>(a, b, nx, ny, nz);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 40;
  cudaEventRecord(e0);
  for (int t = 0; t < n; ++t) pull_copy<true><<<g, 128>>>((t & 1) ? b : a, (t & 1) ? a : b, nx, ny, nz);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double nodes = double(nx) * ny * nz;
  {
    const size_t n2 = size_t(27) * nx * ny * nz / 2;
    cudaEvent_t a0, a1;
    cudaEventCreate(&a0);
    cudaEventCreate(&a1);
    for (int w = 0; w < 2; ++w) plain_copy<<<148 * 16, 256>>>((const double2*)a, (double2*)b, n2);
    cudaEventRecord(a0);
    for (int t = 0; t < 20; ++t) plain_copy<<<148 * 16, 256>>>((const double2*)((t & 1) ? b : a), (double2*)((t & 1) ? a : b), n2);
    cudaEventRecord(a1);
    cudaEventSynchronize(a1);
    float m2 = 0;
    cudaEventElapsedTime(&m2, a0, a1);
    printf("{\"kernel\": \"plain 16B copy, same bytes\", \"ms\": %.4f, \"GBps\": %.1f}\n", m2 / 20,
           432.0 * nodes * 20 / (m2 * 1e-3) / 1e9);
    for (int w = 0; w < 2; ++w) aligned27<<<g, 128>>>(a, b, nx, ny);
    cudaEventRecord(a0);
    for (int t = 0; t < 20; ++t) aligned27<<<g, 128>>>((t & 1) ? b : a, (t & 1) ? a : b, nx, ny);
    cudaEventRecord(a1);
    cudaEventSynchronize(a1);
    cudaEventElapsedTime(&m2, a0, a1);
    printf("{\"kernel\": \"27 aligned streams, no shift\", \"ms\": %.4f, \"GBps\": %.1f}\n", m2 / 20,
           432.0 * nodes * 20 / (m2 * 1e-3) / 1e9);
  }
  printf("{\"kernel\": \"pull_copy (no arithmetic)\", \"ms_per_step\": %.4f, \"mlups\": %.1f, \"GBps_432B\": %.1f, \"err\": \"%s\"}\n",
         ms / n, nodes * n / (ms * 1e-3) / 1e6, 432.0 * nodes * n / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
