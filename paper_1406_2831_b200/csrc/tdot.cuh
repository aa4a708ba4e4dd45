// Canonical projection-dot block (shared by the standalone and the graph
// variants of the kernel).
#pragma once

#include "ctx.cuh"

namespace krb {

// Projection dots out[j] = (M[:,j], v) (self: ||M[:,j]||), j < k.
// Grid (gx, ceil(k/kTdotCG)): CTA (bx, cy) owns columns [cy*CG, cy*CG+CG) of
// canonical blocks b = bx, bx+gx, ...; every (block, column) gets its own
// canonical block partial part[j*nb + b]; the last CTA to finish runs the
// canonical final stage for all k columns (one warp per column).
constexpr int kTdotCG = 4;

template <int kE, bool kSelf, bool kSqrt = kSelf>
__device__ __forceinline__ void tdot_body(int64_t n, int64_t nb, int k,
                                          const double *__restrict__ M,
                                          int64_t ldm,
                                          const double *__restrict__ v,
                                          double *__restrict__ part,
                                          double *__restrict__ out,
                                          unsigned int *counter) {
  __shared__ double sm[kTdotCG][8];
  __shared__ int last_flag;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = blockIdx.y * kTdotCG;
  const int nj = min(kTdotCG, k - j0);
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const int64_t base = b * (256 * kE) + threadIdx.x;
    double vr[kE];
    if (!kSelf) {
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        int64_t i = base + 256 * e;
        vr[e] = i < n ? __ldg(v + i) : 0.0;
      }
    }
#pragma unroll
    for (int jj = 0; jj < kTdotCG; ++jj) {
      if (jj < nj) {
        const double *col = M + (int64_t)(j0 + jj) * ldm;
        double acc = 0.0;
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          int64_t i = base + 256 * e;
          if (i < n) {
            double m = __ldg(col + i);
            acc = __fma_rn(m, kSelf ? m : vr[e], acc);
          }
        }
        double w = warp_tree(acc);
        if (lane == 0) sm[jj][warp] = w;
      }
    }
    __syncthreads();
    if (threadIdx.x < nj) {
      double a[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) a[t] = sm[threadIdx.x][t];
#pragma unroll
      for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
        for (int t = 0; t < off; ++t) a[t] = __dadd_rn(a[t], a[t + off]);
      part[(int64_t)(j0 + threadIdx.x) * nb + b] = a[0];
    }
    __syncthreads();
  }
  // last CTA of the whole (gx x gy) grid: canonical final stage per column
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    last_flag = (prev == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!last_flag) return;
  __threadfence();
  for (int j = warp; j < k; j += (blockDim.x >> 5)) {
    double r = warp_final_volatile(part + (int64_t)j * nb, nb);
    if (lane == 0) out[j] = kSqrt ? __dsqrt_rn(r) : r;
  }
  if (threadIdx.x == 0) *counter = 0;
}

}  // namespace krb
