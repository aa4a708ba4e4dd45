// Canonical projection dots (shared by the standalone kernel, the graph
// kernels and the persistent solver).
#pragma once

#include "ctx.cuh"

namespace krb {

// Projection dots out[j] = (M[:,j], v) (self: ||M[:,j]|| or its square), j < k.
// Work unit = (canonical block b, group of kTdotCG columns from j0), done by
// one 1024-thread CTA: each lane runs the canonical per-lane fma chain for the
// group's columns, one transposed warp tree reduces all of them together
// (warp_tree_multi), then warp c runs the canonical 32-warp tree of column c
// -> part[j*nb + b].
constexpr int kTdotCG = 8;

template <int kE, bool kSelf, int kU = 4, int kCG = kTdotCG>
__device__ __forceinline__ void tdot_unit(int64_t n, int64_t nb, int k,
                                          const double *__restrict__ M,
                                          int64_t ldm,
                                          const double *__restrict__ v,
                                          double *__restrict__ part, int64_t b,
                                          int j0, double (*red)[32],
                                          bool keep = false) {
  const uint64_t pol = l2_policy(keep);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  static_assert(kCG <= kTdotCG, "column group larger than the reduction buffer");
  const int nj = min(kCG, k - j0);
  const int64_t base = b * ((int64_t)kLanes * kE) + threadIdx.x;
  double acc[kCG];
#pragma unroll
  for (int c = 0; c < kCG; ++c) acc[c] = 0.0;
#pragma unroll(kE < kU ? kE : kU)
  for (int e = 0; e < kE; ++e) {
    const int64_t i = base + (int64_t)kLanes * e;
    if (i < n) {
      const double vi = kSelf ? 0.0 : v[i];
      double m[kCG];
#pragma unroll
      for (int c = 0; c < kCG; ++c)
        m[c] = c < nj ? ldg_pol(M + (int64_t)(j0 + c) * ldm + i, pol) : 0.0;
#pragma unroll
      for (int c = 0; c < kCG; ++c)
        acc[c] = __fma_rn(m[c], kSelf ? m[c] : vi, acc[c]);
    }
  }
  int col;
  double w = warp_tree_multi<kCG>(acc, col);
  if ((lane & (32 / kCG - 1)) == 0) red[col][warp] = w;
  __syncthreads();
  if (warp < nj) {
    double r = warp_tree(red[warp][lane]);
    if (lane == 0) part[(int64_t)(j0 + warp) * nb + b] = r;
  }
  __syncthreads();
}

// canonical final stage of k columns (partials part[j*nb + b]) by the warps
// of one CTA
template <bool kSqrt>
__device__ __forceinline__ void tdot_finals(int64_t nb, int k,
                                            const double *part, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < k; j += (blockDim.x >> 5)) {
    double r = warp_final_volatile(part + (int64_t)j * nb, nb);
    if (lane == 0) out[j] = kSqrt ? __dsqrt_rn(r) : r;
  }
}

// Grid (gx, ceil(k/kTdotCG)): CTA (x, y) takes column group y of blocks x,
// x + gx, ...  A 1-D grid instead takes the contiguous unit range
// [c U / G, (c+1) U / G) of the units u = b * ng + g (groups of kCG columns):
// equal unit counts (+-1) and the same mix of groups per CTA -- for block
// counts too small to balance a 2-D grid (C3: 256 blocks).  The last CTA to
// finish runs the final stage.
template <int kE, bool kSelf, bool kSqrt = kSelf, int kU = 4, int kCG = kTdotCG>
__device__ __forceinline__ void tdot_body(int64_t n, int64_t nb, int k,
                                          const double *__restrict__ M,
                                          int64_t ldm,
                                          const double *__restrict__ v,
                                          double *__restrict__ part,
                                          double *__restrict__ out,
                                          unsigned int *counter,
                                          bool keep = false) {
  __shared__ double red[kTdotCG][32];
  __shared__ int last_flag;
  if (gridDim.y == 1 && gridDim.x > 1) {
    const int64_t ng = (k + kCG - 1) / kCG, U = nb * ng, G = gridDim.x;
    const int64_t u1 = (blockIdx.x + 1) * U / G;
    for (int64_t u = blockIdx.x * U / G; u < u1; ++u)
      tdot_unit<kE, kSelf, kU, kCG>(n, nb, k, M, ldm, v, part, u / ng, (int)(u % ng) * kCG,
                                    red, keep);
  } else {
    const int j0 = blockIdx.y * kCG;
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x)
      tdot_unit<kE, kSelf, kU, kCG>(n, nb, k, M, ldm, v, part, b, j0, red, keep);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    last_flag = (prev == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!last_flag) return;
  __threadfence();
  tdot_finals<kSqrt>(nb, k, part, out);
  if (threadIdx.x == 0) *counter = 0;
}

}  // namespace krb
