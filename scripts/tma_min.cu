// Minimal TMA check (3D tiled box -> shared memory with an mbarrier): which
// construct the B200 accepts.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap map, float* out, int x0, int y0, int z0, int doff) {
  __shared__ __align__(128) float bufa[512];
  float* buf = bufa + doff;
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    if (MODE >= 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(136 * 4) : "memory");
    if (MODE == 2) asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(buf)),
        "l"(&map), "r"(x0), "r"(y0), "r"(z0), "r"(smem_u32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          smem_u32(&bar)),
      "r"(0)
      : "memory");
  for (int i = threadIdx.x; i < 136; i += blockDim.x) out[i] = buf[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int nx = 256, ny = 4, np = 6;
  float* d;
  cudaMalloc(&d, sizeof(float) * nx * ny * np);
  float* h = (float*)malloc(sizeof(float) * nx * ny * np);
  for (int i = 0; i < nx * ny * np; ++i) h[i] = (float)i;
  cudaMemcpy(d, h, sizeof(float) * nx * ny * np, cudaMemcpyHostToDevice);
  float* out;
  cudaMalloc(&out, 136 * sizeof(float));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  CUtensorMap map;
  cuuint64_t dims[3] = {nx, ny, np};
  cuuint64_t str[2] = {nx * 4ull, nx * ny * 4ull};
  cuuint32_t box[3] = {136, 1, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  struct { int x, doff; } cases[] = {{0, 0}, {124, 0}, {-4, 0}, {248, 0}, {0, 4}, {0, 8}, {0, 16}, {0, 32}};
  for (auto& c : cases) {
    k<1><<<1, 128>>>(map, out, c.x, 1, 2, c.doff);
    cudaError_t e = cudaDeviceSynchronize();
    float o[136];
    cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    const float base = (float)((2 * ny + 1) * nx + c.x);
    printf("x0 %d smem+%dB: %s  out[0]=%g (expect %g if in range) out[4]=%g out[135]=%g\n", c.x, c.doff * 4,
           cudaGetErrorString(e), o[0], base, o[4], o[135]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
