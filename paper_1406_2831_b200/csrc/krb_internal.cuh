// Internal helpers shared by the libkrb translation units (sm_100a).
//
// Floating-point policy: the library is compiled with -fmad=false, so no
// multiply/add pair is ever contracted by the compiler.  Fused multiply-adds
// appear only where the canonical order (oracle/canon.c) asks for them, via
// explicit __fma_rn.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/krb.h"

// Device sparse matrix (CSR + optional SELL-32 + lazily built transpose).
struct krb_matrix {
  int64_t n = 0, nnz = 0;
  int format = 0;  // 1 CSR, 2 SELL
  int64_t *rp = nullptr;
  int32_t *ci = nullptr;
  double *val = nullptr;
  // SELL-32
  int64_t nslices = 0, sell_elems = 0;
  int64_t *sl_ptr = nullptr;
  int32_t *rlen = nullptr;
  int32_t *s_col = nullptr;
  double *s_val = nullptr;
  krb_matrix *T = nullptr;  // lazily built transpose
  int64_t bytes = 0;
};


namespace krb {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
int64_t &launch_counter();

#define KRB_CHECK_CUDA(call)                                                \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess) {                                                \
      krb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                     cudaGetErrorString(e_));                               \
      return KRB_ECUDA;                                                     \
    }                                                                       \
  } while (0)

#define KRB_CHECK_LAUNCH()                                                  \
  do {                                                                      \
    krb::launch_counter()++;                                                \
    cudaError_t e_ = cudaGetLastError();                                    \
    if (e_ != cudaSuccess) {                                                \
      krb::set_error("%s:%d launch: %s", __FILE__, __LINE__,                \
                     cudaGetErrorString(e_));                               \
      return KRB_ECUDA;                                                     \
    }                                                                       \
  } while (0)

#define KRB_REQUIRE(cond, msg)                                              \
  do {                                                                      \
    if (!(cond)) {                                                          \
      krb::set_error("%s", msg);                                            \
      return KRB_EINVAL;                                                    \
    }                                                                       \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------- canonical order
constexpr int kLanes = 256;            // threads per canonical block
constexpr int kTargetBlocks = 1184;    // 148 SMs x 8
constexpr int kNumSMs = 148;

inline int64_t canon_E(int64_t n) {
  int64_t t = (n + (int64_t)kLanes * kTargetBlocks - 1) /
              ((int64_t)kLanes * kTargetBlocks);
  int64_t E = 4;  /* >= 4 lanes-elements amortise the shuffle tree */
  while (E < t && E < 16) E *= 2;
  return E;
}
inline int64_t canon_nblocks(int64_t n) {
  int64_t B = kLanes * canon_E(n);
  return n <= 0 ? 0 : (n + B - 1) / B;
}
inline int64_t canon_R(int64_t n) {
  int64_t t = (n + 65535) / 65536;
  if (t < 1) t = 1;
  return 64 * t;
}

// lane 0 receives the canonical 32-lane tree (offsets 16,8,4,2,1)
__device__ __forceinline__ double warp_tree(double a) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
    a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, off));
  return a;
}

// canonical 8-warp tree over w[0..7] held by lanes 0..7 of one warp
__device__ __forceinline__ double warp8_tree(double a) {
#pragma unroll
  for (int off = 4; off >= 1; off >>= 1)
    a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, off));
  return a;
}

// Block stage of the canonical dot: every thread of a 256-thread CTA passes
// its lane accumulator; returns the block partial on thread 0.  `sm` needs 8
// doubles.  Contains __syncthreads (call uniformly).
__device__ __forceinline__ double block_tree(double acc, double *sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double w = warp_tree(acc);
  __syncthreads();
  if (lane == 0) sm[warp] = w;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    double v = lane < 8 ? sm[lane] : 0.0;
    r = warp8_tree(v);
  }
  return r;
}

// Final stage over nb block partials (one warp): lane L sums b = L, L+32, ...
// in order, then the 32-lane tree.  Result on lane 0.
__device__ __forceinline__ double warp_final(const double *P, int64_t nb) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  int64_t b = lane;
  for (; b + 7 * 32 < nb; b += 8 * 32) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = P[b + 32 * u];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
  }
  for (; b < nb; b += 32) acc = __dadd_rn(acc, P[b]);
  return warp_tree(acc);
}

// Same, reading through volatile loads (partials written by other CTAs of
// the same kernel, consumed by the last CTA after a fence).
__device__ __forceinline__ double warp_final_volatile(const double *P,
                                                      int64_t nb) {
  // L2-coherent loads (ld.global.cg), issued 8 at a time so the partials of
  // one lane stream in parallel; the adds stay in the canonical order.
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  int64_t b = lane;
  for (; b + 7 * 32 < nb; b += 8 * 32) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(P + b + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
  }
  for (; b < nb; b += 32) acc = __dadd_rn(acc, __ldcg(P + b));
  return warp_tree(acc);
}

// "last CTA" election: every CTA calls after writing its partials; returns
// true on exactly one CTA, which then sees all partials.
__device__ __forceinline__ bool elect_last_cta(unsigned int *counter,
                                               int *sflag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    *sflag = (prev == gridDim.x - 1);
  }
  __syncthreads();
  bool last = *sflag != 0;
  if (last) __threadfence();
  return last;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#define KRB_DISPATCH_E(E, ...)                 \
  switch (E) {                                 \
    case 1: { constexpr int kE = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int kE = 2; __VA_ARGS__; } break;   \
    case 4: { constexpr int kE = 4; __VA_ARGS__; } break;   \
    case 8: { constexpr int kE = 8; __VA_ARGS__; } break;   \
    default: { constexpr int kE = 16; __VA_ARGS__; } break; \
  }

inline int grid_for(int64_t nb, int per_sm = 8) {
  int64_t g = (int64_t)kNumSMs * per_sm;
  if (nb < g) g = nb;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace krb
