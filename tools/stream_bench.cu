// Micro-benchmark: how fast can 148 CTAs x 1024 threads stream the recycle
// block (n x k column-major, the projection-phase access pattern of the fused
// persistent kernel) out of HBM?  Variants:
//   0  plain loads, 8 columns per round, CTA-owned 1024-row blocks
//   1  per-thread cp.async 3-stage pipeline (as in persist.cu)
//   2  all k columns of an element loaded at once (k registers)
//   3  grid-stride double2 stream over the whole matrix (pure bandwidth)
//   4  like 0 but 256 threads/CTA x 4 CTAs/SM, rows split across CTAs
// Several copies of the matrix rotate so each launch reads from HBM, not L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bench tools/stream_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ void cp_async8(double *smem, const double *g) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async8p(double *smem, const double *g, uint64_t pol) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, 8, %2;\n" ::"r"(s), "l"(g), "l"(pol) : "memory");
}
template <int P> __device__ __forceinline__ uint64_t mkpol() {
  uint64_t p;
  if (P == 0) asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  if (P == 1) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  if (P == 2) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <int N> __device__ __forceinline__ void wait_g() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(1024, 1) v0(const double *M, int64_t n, int k, int64_t nb,
                                             double *out) {
  double acc = 0;
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    int64_t i = b * 1024 + threadIdx.x;
    for (int j0 = 0; j0 < k; j0 += 8) {
      double m[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) m[c] = (j0 + c < k) ? __ldg(M + (j0 + c) * n + i) : 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) acc += m[c];
    }
  }
  out[blockIdx.x * 1024 + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(1024, 1) v1(const double *M, int64_t n, int k, int64_t nb,
                                             double *out) {
  extern __shared__ double st[];
  const int ncg = (k + 7) / 8;
  const int nown = blockIdx.x < nb ? (int)((nb - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int T = nown * ncg;
  auto issue = [&](int t) {
    int bi = t / ncg, g = t % ncg;
    int64_t i = (blockIdx.x + (int64_t)bi * gridDim.x) * 1024 + threadIdx.x;
    double *d = st + (size_t)(t % 3) * 8 * 1024 + threadIdx.x;
    for (int c = 0; c < 8; ++c)
      if (g * 8 + c < k) cp_async8(d + c * 1024, M + (g * 8 + c) * n + i);
  };
  for (int t = 0; t < 3; ++t) { if (t < T) issue(t); commit(); }
  double acc = 0;
  for (int t = 0; t < T; ++t) {
    wait_g<2>();
    const double *s = st + (size_t)(t % 3) * 8 * 1024 + threadIdx.x;
    int g = t % ncg;
#pragma unroll
    for (int c = 0; c < 8; ++c) if (g * 8 + c < k) acc += s[c * 1024];
    if (t + 3 < T) issue(t + 3);
    commit();
  }
  out[blockIdx.x * 1024 + threadIdx.x] = acc;
}

// v1 + L2 cache-policy operand (P: 0 normal, 1 first, 2 last) + optional
// per-tile 1024-thread tree with two CTA barriers (as in persist.cu)
template <int P, bool kTree>
__global__ void __launch_bounds__(1024, 1) v5(const double *M, int64_t n, int k, int64_t nb,
                                             double *out) {
  extern __shared__ double st[];
  __shared__ double red[8][32];
  const uint64_t pol = P == 3 ? 0 : mkpol<P>();
  const int ncg = (k + 7) / 8;
  const int nown = blockIdx.x < nb ? (int)((nb - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int T = nown * ncg;
  auto issue = [&](int t) {
    int bi = t / ncg, g = t % ncg;
    int64_t i = (blockIdx.x + (int64_t)bi * gridDim.x) * 1024 + threadIdx.x;
    double *d = st + (size_t)(t % 3) * 8 * 1024 + threadIdx.x;
    for (int c = 0; c < 8; ++c)
      if (g * 8 + c < k) { if (P == 3) cp_async8(d + c * 1024, M + (g * 8 + c) * n + i); else cp_async8p(d + c * 1024, M + (g * 8 + c) * n + i, pol); }
  };
  for (int t = 0; t < 3; ++t) { if (t < T) issue(t); commit(); }
  double tot = 0;
  for (int t = 0; t < T; ++t) {
    wait_g<2>();
    const double *s = st + (size_t)(t % 3) * 8 * 1024 + threadIdx.x;
    int g = t % ncg;
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = (g * 8 + c < k) ? s[c * 1024] : 0.0;
    if (t + 3 < T) issue(t + 3);
    commit();
    if (kTree) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) acc[c] += __shfl_xor_sync(~0u, acc[c], off);
      if ((threadIdx.x & 31) < 8) red[threadIdx.x & 7][threadIdx.x >> 5] = acc[threadIdx.x & 7];
      __syncthreads();
      if (threadIdx.x < 256) {
        double r = red[threadIdx.x >> 5][threadIdx.x & 31];
        for (int off = 16; off >= 1; off >>= 1) r += __shfl_xor_sync(~0u, r, off);
        tot += r;
      }
      __syncthreads();
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) tot += acc[c];
    }
  }
  out[blockIdx.x * 1024 + threadIdx.x] = tot;
}

template <int K>
__global__ void __launch_bounds__(1024, 1) v2(const double *M, int64_t n, int k, int64_t nb,
                                             double *out) {
  double acc = 0;
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    int64_t i = b * 1024 + threadIdx.x;
    double m[K];
#pragma unroll
    for (int c = 0; c < K; ++c) m[c] = __ldg(M + c * n + i);
#pragma unroll
    for (int c = 0; c < K; ++c) acc += m[c];
  }
  out[blockIdx.x * 1024 + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(1024) v3(const double2 *M, int64_t n2, double *out) {
  double acc = 0;
  for (int64_t i = blockIdx.x * 1024 + threadIdx.x; i < n2; i += (int64_t)gridDim.x * 1024) {
    double2 v = __ldg(M + i);
    acc += v.x + v.y;
  }
  out[blockIdx.x * 1024 + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(256) v4(const double *M, int64_t n, int k, double *out) {
  double acc = 0;
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
    for (int j0 = 0; j0 < k; j0 += 8) {
      double m[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) m[c] = (j0 + c < k) ? __ldg(M + (j0 + c) * n + i) : 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) acc += m[c];
    }
  }
  out[blockIdx.x * 256 + threadIdx.x] = acc;
}

// persistent: R passes (rotating copies), grid barrier between passes
struct Mats { const double *m[6]; };
template <int kMode>
__global__ void __launch_bounds__(1024, 1) vp(Mats M, int copies, int R, int64_t n, int k,
                                             int64_t nb, double *out) {
  extern __shared__ double st[];
  cg::grid_group grid = cg::this_grid();
  double tot = 0;
  const int ncg = (k + 7) / 8;
  const int nown = blockIdx.x < nb ? (int)((nb - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  for (int rep = 0; rep < R; ++rep) {
    const double *A = M.m[rep % copies];
    if (kMode == 4) {   // cp.async 3-stage, next pass's prologue issued before the barrier
      const int T = nown * ncg;
      const double *An = M.m[(rep + 1) % copies];
      auto issue = [&](const double *Src, int t) {
        int bi = t / ncg, g = t % ncg;
        int64_t i = (blockIdx.x + (int64_t)bi * gridDim.x) * 1024 + threadIdx.x;
        double *d = st + (size_t)(t % 3) * 8 * 1024 + threadIdx.x;
        for (int c = 0; c < 8; ++c)
          if (g * 8 + c < k) cp_async8(d + c * 1024, Src + (g * 8 + c) * n + i);
      };
      if (rep == 0) { for (int t = 0; t < 3; ++t) { if (t < T) issue(A, t); commit(); } }
      for (int t = 0; t < T; ++t) {
        wait_g<2>();
        const double *s = st + (size_t)(t % 3) * 8 * 1024 + threadIdx.x;
        int g = t % ncg;
#pragma unroll
        for (int c = 0; c < 8; ++c) if (g * 8 + c < k) tot += s[c * 1024];
        if (t + 3 < T) issue(A, t + 3);
        commit();
      }
      for (int t = 0; t < 3; ++t) { if (t < T) issue(An, t); commit(); }
    } else if (kMode == 7 || kMode == 8) {   // as 5 / 6 but the resident blocks via cp.async (+hint)
      uint64_t keep = 0, drop = 0;
      if (kMode == 7) {
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(drop));
      } else {
        asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(keep));
        drop = keep;
      }
      const double *Ares = M.m[rep & 1];
      const double *noise = M.m[2 + (rep % 2)];
      for (int bi = 0; bi < nown; ++bi) {
        const int64_t b = blockIdx.x + (int64_t)bi * gridDim.x;
        for (int c0 = 0; c0 < k; c0 += 8) {
          for (int c = c0; c < k && c < c0 + 8; ++c) {
            unsigned sa = (unsigned)__cvta_generic_to_shared(st + (c - c0) * 1024 + threadIdx.x);
            asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(Ares + c * n + b * 1024 + threadIdx.x), "l"(keep) : "memory");
          }
          commit();
          wait_g<0>();
          for (int c = c0; c < k && c < c0 + 8; ++c) tot += st[(c - c0) * 1024 + threadIdx.x];
        }
      }
      const int64_t nn = (40ll << 20) / 8;
      for (int64_t i = blockIdx.x * 1024 + threadIdx.x; i < nn; i += (int64_t)gridDim.x * 1024) {
        double v;
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(noise + i), "l"(drop));
        tot += v;
      }
    } else if (kMode == 5 || kMode == 6) {   // 2 resident blocks + 40 MB noise; 5: hints, 6: none
      uint64_t keep = 0, drop = 0;
      if (kMode == 5) {
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(drop));
      } else {
        asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(keep));
        drop = keep;
      }
      const double *Ares = M.m[rep & 1];
      const double *noise = M.m[2 + (rep % 2)];
      for (int bi = 0; bi < nown; ++bi) {
        const int64_t b = blockIdx.x + (int64_t)bi * gridDim.x;
        for (int c = 0; c < k; ++c) {
          double v;
          asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(Ares + c * n + b * 1024 + threadIdx.x), "l"(keep));
          tot += v;
        }
      }
      // noise: 40 MB streamed with the drop policy
      const int64_t nn = (40ll << 20) / 8;
      for (int64_t i = blockIdx.x * 1024 + threadIdx.x; i < nn; i += (int64_t)gridDim.x * 1024) {
        double v;
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(noise + i), "l"(drop));
        tot += v;
      }
    } else if (kMode == 0) {   // cp.async 3-stage
      const int T = nown * ncg;
      auto issue = [&](int t) {
        int bi = t / ncg, g = t % ncg;
        int64_t i = (blockIdx.x + (int64_t)bi * gridDim.x) * 1024 + threadIdx.x;
        double *d = st + (size_t)(t % 3) * 8 * 1024 + threadIdx.x;
        for (int c = 0; c < 8; ++c)
          if (g * 8 + c < k) cp_async8(d + c * 1024, A + (g * 8 + c) * n + i);
      };
      for (int t = 0; t < 3; ++t) { if (t < T) issue(t); commit(); }
      for (int t = 0; t < T; ++t) {
        wait_g<2>();
        const double *s = st + (size_t)(t % 3) * 8 * 1024 + threadIdx.x;
        int g = t % ncg;
#pragma unroll
        for (int c = 0; c < 8; ++c) if (g * 8 + c < k) tot += s[c * 1024];
        if (t + 3 < T) issue(t + 3);
        commit();
      }
    } else if (kMode == 2) {   // grid-stride double2 over the whole block
      const double2 *A2 = (const double2 *)A;
      const int64_t n2 = n * k / 2;
      for (int64_t i = blockIdx.x * 1024 + threadIdx.x; i < n2; i += (int64_t)gridDim.x * 1024) {
        double2 v = __ldg(A2 + i);
        tot += v.x + v.y;
      }
    } else if (kMode == 3) {   // owned blocks, column loop, double2 (512 threads/row pair)
      for (int bi = 0; bi < nown; ++bi) {
        const int64_t b = blockIdx.x + (int64_t)bi * gridDim.x;
#pragma unroll 4
        for (int c = 0; c < k; ++c) {
          const double2 *col = (const double2 *)(A + c * n + b * 1024);
          if (threadIdx.x < 512) { double2 v = __ldg(col + threadIdx.x); tot += v.x + v.y; }
        }
      }
    } else {            // plain loads, all 20 columns of both blocks at once
      double m[2][20];
#pragma unroll
      for (int bi = 0; bi < 2; ++bi)
#pragma unroll
        for (int c = 0; c < 20; ++c) {
          int64_t i = (blockIdx.x + (int64_t)bi * gridDim.x) * 1024 + threadIdx.x;
          m[bi][c] = (bi < nown) ? __ldg(A + c * n + i) : 0.0;
        }
#pragma unroll
      for (int bi = 0; bi < 2; ++bi)
#pragma unroll
        for (int c = 0; c < 20; ++c) tot += m[bi][c];
    }
    grid.sync();
  }
  out[blockIdx.x * 1024 + threadIdx.x] = tot;
}

int main(int argc, char **argv) {
  int64_t n = argc > 1 ? atoll(argv[1]) : 262144;
  int k = argc > 2 ? atoi(argv[2]) : 20;
  const int copies = argc > 4 ? atoi(argv[4]) : 6;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  size_t bytes = (size_t)n * k * 8;
  double *M[8];
  double *all;
  CK(cudaMalloc(&all, bytes * copies));   // one allocation: copies are adjacent
  CK(cudaMemset(all, 0, bytes * copies));
  for (int c = 0; c < copies; ++c) M[c] = all + (size_t)c * n * k;
  const int window = argc > 5 ? atoi(argv[5]) : 0;   // MB set aside for persisting
  double *out;
  CK(cudaMalloc(&out, (size_t)sms * 4096 * 8 * 4));
  int64_t nb = (n + 1023) / 1024;
  CK(cudaFuncSetAttribute(v1, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8 * 1024 * 8));
  CK(cudaFuncSetAttribute(v5<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8 * 1024 * 8));
  CK(cudaFuncSetAttribute(v5<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8 * 1024 * 8));
  CK(cudaFuncSetAttribute(v5<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8 * 1024 * 8));
  CK(cudaFuncSetAttribute(v5<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8 * 1024 * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char *names[] = {"v0 plain 8/round", "v1 cp.async 3-stage", "v2 all-k regs",
                         "v3 grid-stride double2", "v4 256thr x4/SM",
                         "v5 cp.async+evict_normal", "v6 cp.async+evict_first",
                         "v7 cp.async+evict_last", "v8 cp.async+tree"};
  const int vmax = argc > 3 ? atoi(argv[3]) : 9;
  for (int v = 0; v < vmax; ++v) {
    if (v >= 5 && v <= 7) continue;
    float best = 1e9, tot = 0;
    const int reps = 30;
    for (int r = 0; r < reps + 3; ++r) {
      const double *m = M[r % copies];
      cudaEventRecord(e0);
      if (v == 0) v0<<<sms, 1024>>>(m, n, k, nb, out);
      if (v == 1) v1<<<sms, 1024, 3 * 8 * 1024 * 8>>>(m, n, k, nb, out);
      if (v == 2) {
        if (k == 20) v2<20><<<sms, 1024>>>(m, n, k, nb, out);
        else v2<10><<<sms, 1024>>>(m, n, k, nb, out);
      }
      if (v == 3) v3<<<sms, 1024>>>((const double2 *)m, (int64_t)(bytes / 16), out);
      if (v == 4) v4<<<sms * 4, 256>>>(m, n, k, out);
      if (v == 5) v5<0, false><<<sms, 1024, 3 * 8 * 1024 * 8>>>(m, n, k, nb, out);
      if (v == 6) v5<1, false><<<sms, 1024, 3 * 8 * 1024 * 8>>>(m, n, k, nb, out);
      if (v == 7) v5<2, false><<<sms, 1024, 3 * 8 * 1024 * 8>>>(m, n, k, nb, out);
      if (v == 8) v5<3, true><<<sms, 1024, 3 * 8 * 1024 * 8>>>(m, n, k, nb, out);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 3) { best = ms < best ? ms : best; tot += ms; }
    }
    printf("%-26s n=%lld k=%d  best %.2f us (%.0f GB/s)  mean %.2f us\n", names[v],
           (long long)n, k, best * 1e3, bytes / (best * 1e-3) / 1e9, tot / reps * 1e3);
  }
  // persistent variants
  CK(cudaFuncSetAttribute(vp<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8 * 1024 * 8));
  Mats mats;
  for (int c = 0; c < copies; ++c) mats.m[c] = M[c];
  CK(cudaFuncSetAttribute(vp<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8 * 1024 * 8));
  CK(cudaFuncSetAttribute(vp<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8 * 1024 * 8));
  CK(cudaFuncSetAttribute(vp<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8 * 1024 * 8));
  for (int mode = 0; mode < 9; ++mode) {
    if (argc > 6 && mode < 5) continue;
    for (int R : {1, 50}) {
      int cp = copies;
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(sms);
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = (mode == 0 || mode == 4 || mode >= 7) ? 3 * 8 * 1024 * 8 : 0;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (window > 0) {
          size_t lim = (size_t)window << 20;
          CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim));
          at[1].id = cudaLaunchAttributeAccessPolicyWindow;
          at[1].val.accessPolicyWindow.base_ptr = all;
          at[1].val.accessPolicyWindow.num_bytes = bytes * copies;
          float hr = (float)((double)lim / (double)(bytes * copies));
          at[1].val.accessPolicyWindow.hitRatio = hr > 1.f ? 1.f : hr;
          at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
          at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
          cfg.numAttrs = 2;
        }
        cudaEventRecord(e0);
        if (mode == 1) CK(cudaLaunchKernelEx(&cfg, vp<1>, mats, cp, R, n, k, nb, out));
        else if (mode == 2) CK(cudaLaunchKernelEx(&cfg, vp<2>, mats, cp, R, n, k, nb, out));
        else if (mode == 3) CK(cudaLaunchKernelEx(&cfg, vp<3>, mats, cp, R, n, k, nb, out));
        else if (mode == 4) CK(cudaLaunchKernelEx(&cfg, vp<4>, mats, cp, R, n, k, nb, out));
        else if (mode == 5) CK(cudaLaunchKernelEx(&cfg, vp<5>, mats, cp, R, n, k, nb, out));
        else if (mode == 6) CK(cudaLaunchKernelEx(&cfg, vp<6>, mats, cp, R, n, k, nb, out));
        else if (mode == 7) CK(cudaLaunchKernelEx(&cfg, vp<7>, mats, cp, R, n, k, nb, out));
        else if (mode == 8) CK(cudaLaunchKernelEx(&cfg, vp<8>, mats, cp, R, n, k, nb, out));
        else CK(cudaLaunchKernelEx(&cfg, vp<0>, mats, cp, R, n, k, nb, out));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("persistent mode %d R=%d: %.2f us per pass (%.0f GB/s)\n", mode, R,
             best * 1e3 / R, bytes * R / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
