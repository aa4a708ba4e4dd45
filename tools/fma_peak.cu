// FP64 FMA throughput ceiling of the CUDA cores (the bound of the Gram and
// GEMM kernels of the recycle update, which stay off the tensor cores for
// bitwise reproducibility): independent __fma_rn chains per thread, all SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fma_peak tools/fma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k_fma(double *out, int iters, double b) {
  double a[C];
#pragma unroll
  for (int i = 0; i < C; ++i) a[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) a[i] = __fma_rn(a[i], b, 1e-12);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += a[i];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int C>
static void run(int blocks_per_sm, int threads) {
  double *d;
  cudaMalloc(&d, 1024 * sizeof(double));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, grid = sms * blocks_per_sm;
  k_fma<C><<<grid, threads>>>(d, iters, 0.999999);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_fma<C><<<grid, threads>>>(d, iters, 0.999999);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fma = 5.0 * grid * threads * (double)iters * C;
  printf("chains %2d  %d x %4d threads/SM: %.2f TFLOP/s fp64 (%.1f fma/clk/SM at 1965 MHz)\n", C,
         blocks_per_sm, threads, 2 * fma / (ms * 1e-3) / 1e12,
         fma / (ms * 1e-3) / sms / 1.965e9);
  cudaFree(d);
}

int main() {
  run<8>(4, 256);
  run<16>(4, 256);
  run<16>(8, 256);
  run<32>(2, 256);
  return 0;
}
