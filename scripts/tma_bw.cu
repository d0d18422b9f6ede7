// TMA pipeline throughput on the B200 (no arithmetic): a persistent grid of
// CTAs with one producer thread issuing NB boxes of BW fp64 elements per tile
// (3D tensor, 1D boxes = rows) into a ring of ST stages, 128 consumer threads
// reading them from shared memory.  Reports GB/s moved by TMA, to separate the
// box-rate limit of the TMA unit from the collide-stream kernel's other costs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   smem_u32(bar)), "r"(parity) : "memory");
}

template <int BW, int NB, int ST, int ROWS>
__global__ void __launch_bounds__(160) k(const __grid_constant__ CUtensorMap map, double* out, long long ntiles, int ny,
                                         int npq) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int BOX = ((BW * ROWS * 8 + 127) / 128) * 128;
  constexpr int STAGE = NB * BOX;
  unsigned long long* full = (unsigned long long*)(sm + ST * STAGE);
  unsigned long long* empty = full + ST;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= 128) {
    if (threadIdx.x == 128) {
      int i = 0;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int s = i % ST;
        const unsigned n = i / ST;
        if (n > 0) mbar_wait(&empty[s], (n - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                     "r"(NB * BW * ROWS * 8) : "memory");
        const int y = int(t % (ny / ROWS)) * ROWS;
        const int pq = int((t / (ny / ROWS)) % (npq - NB));
        for (int b = 0; b < NB; ++b)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                  smem_u32(sm + s * STAGE + b * BOX)),
              "l"(&map), "r"(0), "r"(y), "r"(pq + b), "r"(smem_u32(&full[s]))
              : "memory");
      }
    }
    return;
  }
  double acc = 0;
  int i = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
    const int s = i % ST;
    mbar_wait(&full[s], (i / ST) & 1);
    const double* b = (const double*)(sm + s * STAGE);
#pragma unroll
    for (int q = 0; q < NB; ++q) acc += b[q * (BOX / 8) + threadIdx.x];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])));
  }
  if (acc == 12345.0) out[0] = acc;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int BW, int NB, int ST, int ROWS>
void run(Enc enc, double* d, int nx, int ny, int npq) {
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)npq};
  cuuint64_t str[2] = {nx * 8ull, (cuuint64_t)nx * ny * 8ull};
  cuuint32_t box[3] = {BW, ROWS, 1}, es[3] = {1, 1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  constexpr int BOX = ((BW * ROWS * 8 + 127) / 128) * 128;
  const int smem = ST * NB * BOX + 2 * ST * 8;
  auto fn = k<BW, NB, ST, ROWS>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 160, smem);
  const int grid = per * 148;
  const long long ntiles = 200000;
  double* out;
  cudaMalloc(&out, 8);
  fn<<<grid, 160, smem>>>(map, out, ntiles, ny, npq);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  fn<<<grid, 160, smem>>>(map, out, ntiles, ny, npq);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = double(ntiles) * NB * BW * ROWS * 8;
  printf("box %3d x %d fp64, %2d boxes/stage, %d stages, %d CTA/SM: %7.1f GB/s  %6.1f Gbox/s  (%s)\n", BW, ROWS, NB,
         ST, per, bytes / ms / 1e6, double(ntiles) * NB / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int nx = 512, ny = 512, npq = 27 * 8;  // 453 MB
  double* d;
  cudaMalloc(&d, sizeof(double) * nx * ny * npq);
  cudaMemset(d, 0, sizeof(double) * nx * ny * npq);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  run<128, 27, 2, 1>(enc, d, nx, ny, npq);
  run<128, 27, 3, 1>(enc, d, nx, ny, npq);
  run<128, 9, 4, 1>(enc, d, nx, ny, npq);
  run<256, 27, 1, 1>(enc, d, nx, ny, npq);
  run<128, 27, 1, 2>(enc, d, nx, ny, npq);
  run<128, 9, 3, 4>(enc, d, nx, ny, npq);
  run<64, 27, 3, 1>(enc, d, nx, ny, npq);
  run<256, 9, 3, 2>(enc, d, nx, ny, npq);
  return 0;
}
