// FP64 FMA peak of the B200: register-resident DFMA chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/fp64_peak.cu -o build/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void __launch_bounds__(256) dfma_chains(double* out, long iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 1 << 20);
  const int blocks = 4 * sms, threads = 256;
  const long iters = 200000;
  constexpr int CH = 8;
  dfma_chains<CH><<<blocks, threads>>>(out, 1000, 0.999999, 1e-7);  // warm up
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_chains<CH><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * CH * (double)iters * blocks * threads;
    printf("{\"rep\": %d, \"ms\": %.3f, \"fp64_tflops\": %.3f, \"dfma_per_clk_per_sm_at_1965MHz\": %.2f}\n", rep, ms,
           flops / ms / 1e9, flops / 2.0 / (ms * 1e-3) / sms / 1.965e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
