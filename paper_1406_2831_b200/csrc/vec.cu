// Canonical-order dense primitives for sm_100a: dots, tall-skinny projection
// dots (M^T v), projection updates (v -/+ M y), Grams (X^T Y), basis
// combinations (X Z), column norms, and the PCG64 shadow-vector draw.
//
// All are HBM-bound (<= 0.25 flop/B except the Gram, ~m/8 flop/B): they are
// written as grid-stride loops over canonical blocks of 256*E elements with
// coalesced 256-thread x 8 B sweeps, and every reduction follows the order of
// oracle/canon.c exactly (block stage: per-lane fma chain over E elements,
// 32-lane shuffle tree, 8-warp tree; final stage: 32-lane strided sum then
// tree).
#include "ctx.cuh"
#include "tdot.cuh"

namespace krb {

template <int kE>
__global__ void __launch_bounds__(1024) k_dot_part(int64_t n, int64_t nb,
                                                   const double *__restrict__ x,
                                                   const double *__restrict__ y,
                                                   double *__restrict__ part) {
  __shared__ double red[1][32];
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const int64_t base = b * ((int64_t)kLanes * kE) + threadIdx.x;
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < kE; ++e) {
      int64_t i = base + (int64_t)kLanes * e;
      if (i < n) acc = __fma_rn(__ldg(x + i), __ldg(y + i), acc);
    }
    double r = block_tree(acc, red);
    if (threadIdx.x == 0) part[b] = r;
  }
}

__global__ void k_final(int ndots, int64_t nb, const double *__restrict__ part,
                        double *__restrict__ out) {
  int d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (d >= ndots) return;
  double r = warp_final(part + d * nb, nb);
  if ((threadIdx.x & 31) == 0) out[d] = r;
}

__global__ void k_final_sqrt(int ndots, int64_t nb,
                             const double *__restrict__ part,
                             double *__restrict__ out) {
  int d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (d >= ndots) return;
  double r = warp_final(part + d * nb, nb);
  if ((threadIdx.x & 31) == 0) out[d] = __dsqrt_rn(r);
}

template <int kE, bool kSelf, bool kSqrt>
__global__ void __launch_bounds__(1024) k_tdot(
    int64_t n, int64_t nb, int k, const double *__restrict__ M, int64_t ldm,
    const double *__restrict__ v, double *__restrict__ part,
    double *__restrict__ out, unsigned int *counter) {
  tdot_body<kE, kSelf, kSqrt>(n, nb, k, M, ldm, v, part, out, counter);
}

// Ritz eigen-residual combination (recycling.py:351-352 as real arithmetic):
// Are <- Are - (Yre*thr - Yim*thi) ; Aim <- Aim - (Yre*thi + Yim*thr)
__global__ void k_ritz_combine(int64_t n, int m, const double *__restrict__ Yre,
                               const double *__restrict__ Yim, double *Are,
                               double *Aim, int64_t ld,
                               const double *__restrict__ thr,
                               const double *__restrict__ thi) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       idx < n * m; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = idx / n, i = idx % n;
    int64_t o = c * ld + i;
    double yr = Yre[o], yi = Yim[o], tr = thr[c], ti = thi[c];
    Are[o] = __dsub_rn(Are[o], __dsub_rn(__dmul_rn(yr, tr), __dmul_rn(yi, ti)));
    Aim[o] = __dsub_rn(Aim[o], __dadd_rn(__dmul_rn(yr, ti), __dmul_rn(yi, tr)));
  }
}

// out[i] = base[i] + sign * (sum_j M[i,j] y[j])  (sequential fma from 0.0)
__global__ void __launch_bounds__(256) k_gemv(int64_t n, int k,
                                              const double *__restrict__ M,
                                              int64_t ldm,
                                              const double *__restrict__ y,
                                              const double *base, int sign,
                                              double *out) {
  extern __shared__ double ys[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) ys[j] = y[j];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < k; ++j) acc = __fma_rn(__ldg(M + (int64_t)j * ldm + i), ys[j], acc);
    double o;
    if (base == nullptr)
      o = acc;
    else if (sign < 0)
      o = __dsub_rn(base[i], acc);
    else
      o = __dadd_rn(base[i], acc);
    out[i] = o;
  }
}

// ---- Gram: chunk partials (R rows sequential per entry) -----------------
// One CTA per chunk; 64-row tiles of X (na cols) and Y (nc cols) staged in
// shared memory; each thread owns entries e = tid, tid+256, ... (row-major
// a*nc + c) and walks the chunk rows in order with fma.
constexpr int kGramTile = 64;
constexpr int kGramMaxEnt = 16;  // entries per thread => na*nc <= 4096

__global__ void __launch_bounds__(256) k_gram_part(
    int64_t n, int64_t R, int64_t nch, int na, int nc,
    const double *__restrict__ X, int64_t ldx, const double *__restrict__ Y,
    int64_t ldy, double *__restrict__ part) {
  extern __shared__ double sm[];
  double *xs = sm;                     // [kGramTile][na]
  double *ys = sm + kGramTile * na;    // [kGramTile][nc]
  const int ne = na * nc;
  for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    double acc[kGramMaxEnt];
#pragma unroll
    for (int t = 0; t < kGramMaxEnt; ++t) acc[t] = 0.0;
    const int64_t r0 = ch * R;
    const int64_t r1 = min(n, r0 + R);
    for (int64_t t0 = r0; t0 < r1; t0 += kGramTile) {
      const int rows = (int)min((int64_t)kGramTile, r1 - t0);
      __syncthreads();
      for (int idx = threadIdx.x; idx < kGramTile * na; idx += blockDim.x) {
        int a = idx / kGramTile, rr = idx % kGramTile;
        xs[rr * na + a] = rr < rows ? __ldg(X + (int64_t)a * ldx + t0 + rr) : 0.0;
      }
      for (int idx = threadIdx.x; idx < kGramTile * nc; idx += blockDim.x) {
        int c = idx / kGramTile, rr = idx % kGramTile;
        ys[rr * nc + c] = rr < rows ? __ldg(Y + (int64_t)c * ldy + t0 + rr) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int t = 0; t < kGramMaxEnt; ++t) {
        int e = threadIdx.x + 256 * t;
        if (e < ne) {
          int a = e / nc, c = e % nc;
          double s = acc[t];
          for (int rr = 0; rr < rows; ++rr)
            s = __fma_rn(xs[rr * na + a], ys[rr * nc + c], s);
          acc[t] = s;
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kGramMaxEnt; ++t) {
      int e = threadIdx.x + 256 * t;
      if (e < ne) part[(int64_t)e * nch + ch] = acc[t];
    }
  }
}

// Register-tiled Gram chunk partials (same order as k_gram_part): a 16 x 16
// thread grid, thread (ty, tx) owning the T x T entries (ty + 16 i, tx + 16 j)
// and running their sequential fma chains over the chunk's rows.  Row
// sub-tiles of kGT rows are staged column-major in shared memory with an odd
// stride (conflict-free: the 16 distinct columns a warp reads hit distinct
// banks) by per-thread cp.async, double-buffered so the next sub-tile loads
// while this one is consumed.  FP64-FMA bound (m x m x n fma per Gram).
constexpr int kGT = 64;
constexpr int kGS = kGT + 1;   // odd column stride in shared memory
template <int T>
__global__ void __launch_bounds__(256) k_gram_rt(int64_t n, int64_t R, int64_t nch, int na,
                                                 int nc, const double *__restrict__ X,
                                                 int64_t ldx, const double *__restrict__ Y,
                                                 int64_t ldy, double *__restrict__ part) {
  extern __shared__ double sm[];
  constexpr int W = 16 * T;                 // staged columns of X and of Y
  constexpr int kBuf = 2 * W * kGS;         // doubles per buffer (X then Y)
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const uint64_t pol = l2_policy(false);
  for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    const int64_t r0 = ch * R;
    const int64_t r1 = min(n, r0 + R);
    const int nsub = (int)((r1 - r0 + kGT - 1) / kGT);
    auto stage = [&](int sub, int buf) {
      const int64_t t0 = r0 + (int64_t)sub * kGT;
      const int rows = (int)min((int64_t)kGT, r1 - t0);
      double *xs = sm + buf * kBuf, *ys = xs + W * kGS;
      for (int idx = tid; idx < W * kGT; idx += 256) {
        const int a = idx >> 6, rr = idx & (kGT - 1);
        const bool okx = a < na && rr < rows, oky = a < nc && rr < rows;
        cp_async8(xs + a * kGS + rr, X + (okx ? (int64_t)a * ldx + t0 + rr : 0), okx, pol);
        cp_async8(ys + a * kGS + rr, Y + (oky ? (int64_t)a * ldy + t0 + rr : 0), oky, pol);
      }
      cp_async_commit();
    };
    double acc[T][T];
#pragma unroll
    for (int i = 0; i < T; ++i)
#pragma unroll
      for (int j = 0; j < T; ++j) acc[i][j] = 0.0;
    __syncthreads();   // previous chunk's readers are done with both buffers
    stage(0, 0);
    for (int sub = 0; sub < nsub; ++sub) {
      if (sub + 1 < nsub) {
        stage(sub + 1, (sub + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double *xs = sm + (sub & 1) * kBuf, *ys = xs + W * kGS;
      const int rows = (int)min((int64_t)kGT, r1 - (r0 + (int64_t)sub * kGT));
      for (int rr = 0; rr < rows; ++rr) {
        double xv[T], yv[T];
#pragma unroll
        for (int i = 0; i < T; ++i) xv[i] = xs[(ty + 16 * i) * kGS + rr];
#pragma unroll
        for (int j = 0; j < T; ++j) yv[j] = ys[(tx + 16 * j) * kGS + rr];
#pragma unroll
        for (int i = 0; i < T; ++i)
#pragma unroll
          for (int j = 0; j < T; ++j) acc[i][j] = __fma_rn(xv[i], yv[j], acc[i][j]);
      }
      __syncthreads();   // buffer (sub & 1) is refilled two sub-tiles later
    }
#pragma unroll
    for (int i = 0; i < T; ++i)
#pragma unroll
      for (int j = 0; j < T; ++j) {
        const int a = ty + 16 * i, c = tx + 16 * j;
        if (a < na && c < nc) part[(int64_t)(a * nc + c) * nch + ch] = acc[i][j];
      }
  }
}

// Gram chunk partials, 64-thread groups (same order as k_gram_part): each
// group of 64 threads (an 8 x 8 grid) owns one chunk at a time, thread
// (ty, tx) the T x T entries (ty + 8 i, tx + 8 j), so a row costs 2T
// shared-memory doubles for T^2 fmas (T = 6 at m = 47: 12 per 36, vs 6 per
// 9 with 256 threads per chunk).  Rows are read in pairs as 16-byte loads
// from kGT2-row sub-tiles staged column-major with stride kGT2 + 2 (odd in
// 16-byte units: the 8 distinct columns a warp reads fall in distinct bank
// groups), double-buffered per group by per-thread cp.async; groups
// synchronise on their own named barrier, so the G groups of a CTA run
// independently.  kGT2 = 16 and <= 128 registers keep two CTAs (16 warps)
// per SM.
template <int T, int G, int kGT2>
__global__ void __launch_bounds__(64 * G, 2) k_gram_g(int64_t n, int64_t R, int64_t nch, int na,
                                                   int nc, const double *__restrict__ X,
                                                   int64_t ldx, const double *__restrict__ Y,
                                                   int64_t ldy, double *__restrict__ part) {
  extern __shared__ double2 sm2[];
  constexpr int kGS2 = kGT2 + 2;
  constexpr int W = 8 * T;                  // staged columns of X and of Y
  constexpr int kBuf = 2 * W * kGS2;        // doubles per buffer (X then Y)
  const int g = threadIdx.x >> 6, lt = threadIdx.x & 63, tx = lt & 7, ty = lt >> 3;
  double *gsm = reinterpret_cast<double *>(sm2) + (size_t)g * 2 * kBuf;
  const uint64_t pol = l2_policy(false);
  auto gsync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(g + 1) : "memory"); };
  for (int64_t ch = (int64_t)blockIdx.x * G + g; ch < nch; ch += (int64_t)gridDim.x * G) {
    const int64_t r0 = ch * R;
    const int64_t r1 = min(n, r0 + R);
    const int nsub = (int)((r1 - r0 + kGT2 - 1) / kGT2);
    auto stage = [&](int sub, int buf) {
      const int64_t t0 = r0 + (int64_t)sub * kGT2;
      const int rows = (int)min((int64_t)kGT2, r1 - t0);
      double *xs = gsm + buf * kBuf, *ys = xs + W * kGS2;
      for (int idx = lt; idx < W * kGT2; idx += 64) {
        const int a = idx / kGT2, rr = idx % kGT2;
        const bool okx = a < na && rr < rows, oky = a < nc && rr < rows;
        cp_async8(xs + a * kGS2 + rr, X + (okx ? (int64_t)a * ldx + t0 + rr : 0), okx, pol);
        cp_async8(ys + a * kGS2 + rr, Y + (oky ? (int64_t)a * ldy + t0 + rr : 0), oky, pol);
      }
      cp_async_commit();
    };
    double acc[T][T];
#pragma unroll
    for (int i = 0; i < T; ++i)
#pragma unroll
      for (int j = 0; j < T; ++j) acc[i][j] = 0.0;
    gsync();   // the group's previous chunk readers are done with both buffers
    stage(0, 0);
    for (int sub = 0; sub < nsub; ++sub) {
      if (sub + 1 < nsub) {
        stage(sub + 1, (sub + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      gsync();
      const double *xs = gsm + (sub & 1) * kBuf, *ys = xs + W * kGS2;
      const int rows = (int)min((int64_t)kGT2, r1 - (r0 + (int64_t)sub * kGT2));
      int rr = 0;
      for (; rr + 1 < rows; rr += 2) {
        // y column by column: its loads overlap the previous column's fmas
        double2 xv[T];
#pragma unroll
        for (int i = 0; i < T; ++i)
          xv[i] = *reinterpret_cast<const double2 *>(xs + (ty + 8 * i) * kGS2 + rr);
#pragma unroll
        for (int j = 0; j < T; ++j) {
          const double2 yv = *reinterpret_cast<const double2 *>(ys + (tx + 8 * j) * kGS2 + rr);
#pragma unroll
          for (int i = 0; i < T; ++i) acc[i][j] = __fma_rn(xv[i].x, yv.x, acc[i][j]);
#pragma unroll
          for (int i = 0; i < T; ++i) acc[i][j] = __fma_rn(xv[i].y, yv.y, acc[i][j]);
        }
      }
      if (rr < rows) {
#pragma unroll
        for (int i = 0; i < T; ++i)
#pragma unroll
          for (int j = 0; j < T; ++j)
            acc[i][j] = __fma_rn(xs[(ty + 8 * i) * kGS2 + rr], ys[(tx + 8 * j) * kGS2 + rr],
                                 acc[i][j]);
      }
      gsync();   // buffer (sub & 1) is refilled two sub-tiles later
    }
#pragma unroll
    for (int i = 0; i < T; ++i)
#pragma unroll
      for (int j = 0; j < T; ++j) {
        const int a = ty + 8 * i, c = tx + 8 * j;
        if (a < na && c < nc) part[(int64_t)(a * nc + c) * nch + ch] = acc[i][j];
      }
  }
}

template <int T, int G, int S>
static int launch_gram_g(int64_t n, int64_t R, int64_t nch, int na, int nc, const double *X,
                         int64_t ldx, const double *Y, int64_t ldy, double *part,
                         cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)G * 2 * 2 * 8 * T * (S + 2);   // G x 2 buffers x (X, Y)
  static int per_sm = 0;   // per instantiation: the opt-in and the occupancy query run once
  if (per_sm == 0) {
    KRB_CHECK_CUDA(cudaFuncSetAttribute(k_gram_g<T, G, S>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int q = 0;
    KRB_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, k_gram_g<T, G, S>, 64 * G,
                                                                 smem));
    per_sm = q < 1 ? 1 : q;
  }
  const int64_t want = (nch + G - 1) / G;
  const int64_t cap = (int64_t)kNumSMs * per_sm;
  const int grid = (int)(want < cap ? want : cap);
  k_gram_g<T, G, S><<<grid, 64 * G, smem, st>>>(n, R, nch, na, nc, X, ldx, Y, ldy, part);
  return KRB_OK;
}

// out[i + c*ldo] = sum_j X[i + j*ldx] Z[j*nc + c]  (sequential fma, j order)
// One thread per row, kCT output columns per pass (X is re-read once per
// pass: ceil(nc / kCT) passes), Z in shared memory with an even row stride
// so a row's kCT coefficients are kCT / 2 broadcast 16-byte loads.
constexpr int kGemmCT2 = 24;
__global__ void __launch_bounds__(256, 2) k_gemm(int64_t n, int m, int nc,
                                                 const double *__restrict__ X,
                                                 int64_t ldx,
                                                 const double *__restrict__ Z,
                                                 double *__restrict__ out,
                                                 int64_t ldo) {
  extern __shared__ double2 zs2[];
  double *zs = reinterpret_cast<double *>(zs2);
  const int ncp = ((nc + kGemmCT2 - 1) / kGemmCT2) * kGemmCT2;   // padded stride
  for (int idx = threadIdx.x; idx < m * ncp; idx += blockDim.x) {
    const int j = idx / ncp, c = idx - j * ncp;
    zs[idx] = c < nc ? Z[j * nc + c] : 0.0;
  }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int c0 = 0; c0 < nc; c0 += kGemmCT2) {
      double acc[kGemmCT2];
#pragma unroll
      for (int t = 0; t < kGemmCT2; ++t) acc[t] = 0.0;
      const double *xp = X + i;
      const double2 *zrow = zs2 + (c0 >> 1);
#pragma unroll 2
      for (int j = 0; j < m; ++j) {
        const double xv = __ldg(xp + (int64_t)j * ldx);
        const double2 *zr = zrow + j * (ncp >> 1);
#pragma unroll
        for (int t = 0; t < kGemmCT2 / 2; ++t) {
          const double2 z = zr[t];
          acc[2 * t] = __fma_rn(xv, z.x, acc[2 * t]);
          acc[2 * t + 1] = __fma_rn(xv, z.y, acc[2 * t + 1]);
        }
      }
#pragma unroll
      for (int t = 0; t < kGemmCT2; ++t)
        if (c0 + t < nc) out[(int64_t)(c0 + t) * ldo + i] = acc[t];
    }
  }
}

// Tiled variant (same sums, same order): a CTA streams tiles of T rows of
// X (all m columns) into shared memory with TMA bulk copies (one 8T-byte
// copy per column, one elected thread, completion on an mbarrier), double
// buffered, so the next tile is in flight while the current one is
// consumed; thread (row r, column group g) accumulates its kCT outputs from
// the staged tile (conflict-free rows) and the broadcast Z.  X is read from
// HBM exactly once.  Needs 16-byte aligned columns (X, ldx even); the
// partial last tile goes through plain loads.
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_1d(double *dst, const double *src, unsigned bytes,
                                       uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

// Two adjacent rows per thread (i, i + 1): each broadcast Z load feeds 2 x 2
// fmas instead of 2, the X pair is one 16-byte load.  Same per-entry order.
template <int kCT>
__device__ __forceinline__ void gemm_tile_rows2(const double *xs, int T, int r, int g, int m,
                                                int nc, int ncp, const double2 *dsm2,
                                                double *out, int64_t ldo, int64_t i,
                                                int64_t nrows) {
  const int c0 = g * kCT;
  double a0[kCT], a1[kCT];
#pragma unroll
  for (int t = 0; t < kCT; ++t) a0[t] = a1[t] = 0.0;
  const double2 *zrow = dsm2 + (c0 >> 1);
#pragma unroll 2
  for (int j = 0; j < m; ++j) {
    const double2 xv = *reinterpret_cast<const double2 *>(xs + j * T + r);
    const double2 *zr = zrow + j * (ncp >> 1);
#pragma unroll
    for (int t = 0; t < kCT / 2; ++t) {
      const double2 z = zr[t];
      a0[2 * t] = __fma_rn(xv.x, z.x, a0[2 * t]);
      a0[2 * t + 1] = __fma_rn(xv.x, z.y, a0[2 * t + 1]);
      a1[2 * t] = __fma_rn(xv.y, z.x, a1[2 * t]);
      a1[2 * t + 1] = __fma_rn(xv.y, z.y, a1[2 * t + 1]);
    }
  }
#pragma unroll
  for (int t = 0; t < kCT; ++t)
    if (c0 + t < nc) {
      if (nrows > 0) out[(int64_t)(c0 + t) * ldo + i] = a0[t];
      if (nrows > 1) out[(int64_t)(c0 + t) * ldo + i + 1] = a1[t];
    }
}

template <int kCT>
__device__ __forceinline__ void gemm_tile_rows(const double *xs, int T, int r, int g, int m,
                                               int nc, int ncp, const double2 *dsm2,
                                               double *out, int64_t ldo, int64_t i) {
  const int c0 = g * kCT;
  double acc[kCT];
#pragma unroll
  for (int t = 0; t < kCT; ++t) acc[t] = 0.0;
  const double2 *zrow = dsm2 + (c0 >> 1);
#pragma unroll 2
  for (int j = 0; j < m; ++j) {
    const double xv = xs[j * T + r];
    const double2 *zr = zrow + j * (ncp >> 1);
#pragma unroll
    for (int t = 0; t < kCT / 2; ++t) {
      const double2 z = zr[t];
      acc[2 * t] = __fma_rn(xv, z.x, acc[2 * t]);
      acc[2 * t + 1] = __fma_rn(xv, z.y, acc[2 * t + 1]);
    }
  }
#pragma unroll
  for (int t = 0; t < kCT; ++t)
    if (c0 + t < nc) out[(int64_t)(c0 + t) * ldo + i] = acc[t];
}

template <int kCT, int RPT>
__global__ void __launch_bounds__(256, 2) k_gemm_t(int64_t n, int m, int nc, int lgT,
                                                   const double *__restrict__ X, int64_t ldx,
                                                   const double *__restrict__ Z,
                                                   double *__restrict__ out, int64_t ldo) {
  extern __shared__ double2 dsm2[];
  __shared__ uint64_t bar[2];
  double *dsm = reinterpret_cast<double *>(dsm2);
  const int T = 1 << lgT;
  const int ncp = ((nc + kCT - 1) / kCT) * kCT;
  double *zs = dsm;                                   // m x ncp (16-byte multiple)
  double *stage = dsm + (size_t)m * ncp;              // 2 x m x T
  for (int idx = threadIdx.x; idx < m * ncp; idx += blockDim.x) {
    const int j = idx / ncp, c = idx - j * ncp;
    zs[idx] = c < nc ? Z[j * nc + c] : 0.0;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nfull = n >> lgT;
  // row in tile (RPT adjacent rows per thread), column group
  const int r = (threadIdx.x & ((T / RPT) - 1)) * RPT, g = threadIdx.x >> (lgT - (RPT - 1));
  const int ngroups = ncp / kCT;
  const int per = m << lgT;
  const unsigned tile_bytes = (unsigned)per * 8u;
  auto issue = [&](int64_t t, int b) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bar[b], tile_bytes);
    const double *src = X + (t << lgT);
    double *dst = stage + (size_t)b * per;
    for (int j = 0; j < m; ++j) tma_1d(dst + (j << lgT), src + (int64_t)j * ldx, (unsigned)T * 8u, &bar[b]);
  };
  int64_t tile = blockIdx.x;
  unsigned ph = 0u;   // bit b: parity of buffer b's next completion
  if (threadIdx.x == 0 && tile < nfull) issue(tile, 0);
  int buf = 0;
  for (; tile < nfull; tile += gridDim.x, buf ^= 1) {
    if (threadIdx.x == 0 && tile + gridDim.x < nfull) issue(tile + gridDim.x, buf ^ 1);
    mbar_wait(&bar[buf], (ph >> buf) & 1u);
    ph ^= 1u << buf;
    if (g < ngroups) {
      if (RPT == 2)
        gemm_tile_rows2<kCT>(stage + (size_t)buf * per, T, r, g, m, nc, ncp, dsm2, out, ldo,
                             (tile << lgT) + r, 2);
      else
        gemm_tile_rows<kCT>(stage + (size_t)buf * per, T, r, g, m, nc, ncp, dsm2, out, ldo,
                            (tile << lgT) + r);
    }
    __syncthreads();   // every thread done with `buf` before it is refilled
  }
  // partial last tile: plain loads, by the CTA the tile loop would give it to
  const int64_t rem = n - (nfull << lgT);
  if (rem > 0 && blockIdx.x == (unsigned)(nfull % gridDim.x)) {
    double *xs = stage;
    for (int e = threadIdx.x; e < per; e += blockDim.x) {
      const int j = e >> lgT, rr = e & (T - 1);
      xs[e] = rr < rem ? X[(int64_t)j * ldx + (nfull << lgT) + rr] : 0.0;
    }
    __syncthreads();
    if (g < ngroups && r < rem) {
      if (RPT == 2)
        gemm_tile_rows2<kCT>(xs, T, r, g, m, nc, ncp, dsm2, out, ldo, (nfull << lgT) + r,
                             rem - r);
      else
        gemm_tile_rows<kCT>(xs, T, r, g, m, nc, ncp, dsm2, out, ldo, (nfull << lgT) + r);
    }
  }
}

template <int kCT, int RPT = 1>
static bool gemm_tiled(int64_t n, int64_t m, int64_t nc, const double *d_X, int64_t ldx,
                       const double *d_Z, double *d_out, int64_t ldo, cudaStream_t st,
                       int *rc) {
  const int64_t ncp = ((nc + kCT - 1) / kCT) * kCT;
  const int64_t groups = ncp / kCT;
  int lgT = 0;   // T = 2^lgT rows per tile, groups x T / RPT <= 256 threads
  while ((groups << (lgT + 1)) <= 256 * RPT) ++lgT;
  // RPT = 2: keep two CTAs per SM (tile stage + Z <= 110 KB) at the cost of threads
  while (RPT == 2 && lgT > 5 &&
         sizeof(double) * (size_t)(m * ncp + 2 * (m << lgT)) > 110 * 1024)
    --lgT;
  if (lgT < 5) return false;   // T >= 32 rows (idle threads when groups does not divide 256)
  if ((ldx & 1) || (reinterpret_cast<uintptr_t>(d_X) & 15)) return false;   // TMA alignment
  const int threads = (int)((groups << lgT) / RPT);
  const size_t smem = sizeof(double) * (size_t)(m * ncp + 2 * (m << lgT));
  if (smem > 200 * 1024) return false;
  *rc = KRB_OK;
  static size_t attr_smem = 0;   // largest dynamic smem opted in so far
  if (smem > attr_smem) {
    if (cudaFuncSetAttribute(k_gemm_t<kCT, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024) != cudaSuccess) {
      set_error("krb_gemm: cudaFuncSetAttribute failed");
      *rc = KRB_ECUDA;
      return true;
    }
    attr_smem = 200 * 1024;
  }
  // resident CTAs per SM: shared memory (227 KB) and registers (2 x 256 threads)
  int per_sm = smem <= 110 * 1024 ? 2 : 1;
  if (RPT == 2) {
    // occupancy from the kernel's register count (queried once) and this
    // launch's shared memory / threads, without a per-call occupancy query
    static int regs = 0;
    if (regs == 0) {
      cudaFuncAttributes fa;
      regs = cudaFuncGetAttributes(&fa, k_gemm_t<kCT, RPT>) == cudaSuccess ? fa.numRegs : 255;
    }
    const int warps = (threads + 31) / 32;
    const int regs_per_warp = ((regs * 32 + 255) / 256) * 256;
    const int by_regs = 65536 / (regs_per_warp * warps);
    const int by_smem = (int)((228 * 1024) / (smem + 1024));
    const int by_thr = 2048 / threads;
    per_sm = by_regs < by_smem ? by_regs : by_smem;
    if (by_thr < per_sm) per_sm = by_thr;
    if (per_sm < 1) per_sm = 1;
  }
  const int64_t ntiles = (n + (1 << lgT) - 1) >> lgT;
  const int64_t cap = (int64_t)kNumSMs * per_sm;
  const int grid = (int)(ntiles < cap ? ntiles : cap);
  k_gemm_t<kCT, RPT><<<grid, RPT == 2 ? threads : 256, smem, st>>>(n, (int)m, (int)nc, lgT, d_X,
                                                                     ldx, d_Z, d_out, ldo);
  if (cudaGetLastError() != cudaSuccess) {
    set_error("krb_gemm: launch failed");
    *rc = KRB_ECUDA;
  }
  return true;
}

// X[:, j] /= s[j]: column j on blockIdx.y (no per-element index division);
// each thread divides four elements 256 apart, loads issued together
// Y[:, j] = X[:, j] / s[j] (Y == X: in place; otherwise Y must not overlap X)
__global__ void __launch_bounds__(256) k_colscale_div(int64_t n, int k, const double *X,
                                                      int64_t ldx,
                                                      const double *__restrict__ s,
                                                      double *Y, int64_t ldy) {
  const int j = blockIdx.y;
  const double *src = X + (int64_t)j * ldx;
  double *col = Y + (int64_t)j * ldy;
  const double d = __ldg(s + j);
  for (int64_t i0 = (int64_t)blockIdx.x * 1024 + threadIdx.x; i0 < n;
       i0 += (int64_t)gridDim.x * 1024) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + 256 * q;
      v[q] = i < n ? src[i] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + 256 * q;
      if (i < n) col[i] = __ddiv_rn(v[q], d);
    }
  }
}

// ---- PCG64 (numpy default_rng) -----------------------------------------
typedef unsigned __int128 u128;
__host__ __device__ inline u128 mk128(uint64_t hi, uint64_t lo) {
  return ((u128)hi << 64) | lo;
}
constexpr uint64_t kPcgMulHi = 0x2360ED051FC65DA4ull;
constexpr uint64_t kPcgMulLo = 0x4385DF649FCCF645ull;

// (A, C) such that LCG^steps(s) = A*s + C   (mod 2^128)
__host__ __device__ inline void pcg_jump(u128 mult, u128 inc, uint64_t steps,
                                         u128 *A, u128 *C) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = mult, cur_plus = inc;
  while (steps > 0) {
    if (steps & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    steps >>= 1;
  }
  *A = acc_mult;
  *C = acc_plus;
}

__device__ inline uint64_t pcg_out(u128 s) {
  uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

// element i uses state LCG^(i+1)(s0); thread g handles the run
// i = g L .. g L + L - 1: one jump to its start, then single LCG steps (a
// jump per element costs ~18 dependent 128-bit multiply-adds)
constexpr int kPcgRun = 16;
__global__ void k_pcg64_uniform(int64_t n, uint64_t s_hi, uint64_t s_lo,
                                uint64_t i_hi, uint64_t i_lo, double lo,
                                double range, double *out) {
  const u128 mult = mk128(kPcgMulHi, kPcgMulLo), inc = mk128(i_hi, i_lo);
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = g * kPcgRun;
  if (i0 >= n) return;
  u128 A, C;
  pcg_jump(mult, inc, (uint64_t)i0 + 1, &A, &C);
  u128 s = A * mk128(s_hi, s_lo) + C;
  const int64_t i1 = i0 + kPcgRun < n ? i0 + kPcgRun : n;
  for (int64_t i = i0; i < i1; ++i) {
    uint64_t r = pcg_out(s);
    double u = (double)(r >> 11) * (1.0 / 9007199254740992.0);
    out[i] = __dadd_rn(lo, __dmul_rn(range, u));
    s = mult * s + inc;
  }
}

// ---- host launchers ------------------------------------------------------
int launch_dot_partials(int64_t n, const double *x, const double *y,
                        double *part, cudaStream_t st) {
  int64_t nb = canon_nblocks(n);
  if (nb == 0) return KRB_OK;
  int grid = grid_for(nb);
  KRB_DISPATCH_E(canon_E(n), (k_dot_part<kE><<<grid, 1024, 0, st>>>(n, nb, x, y, part)));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int launch_final(int ndots, int64_t nb, const double *part, double *out,
                 cudaStream_t st) {
  if (ndots <= 0) return KRB_OK;
  k_final<<<(ndots + 7) / 8, 256, 0, st>>>(ndots, nb, part, out);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

// One wave: gx x gy = 148 x (resident CTAs per SM), so the column groups of
// a canonical block run at the same time (their shared v loads hit L2) and no
// CTA waits for a second wave.  (2 per SM assumed before; with 42-64
// registers only one 1024-thread CTA fits, so half the grid ran as a second
// wave that re-read v from DRAM.)
dim3 tdot_grid(int64_t nb, int64_t k, int per_sm) {
  int64_t gy = (k + kTdotCG - 1) / kTdotCG;
  int64_t want = (int64_t)kNumSMs * (per_sm > 0 ? per_sm : 1);
  int64_t gx = (want + gy - 1) / gy;
  if (gx > nb) gx = nb;
  if (gx < 1) gx = 1;
  return dim3((unsigned)gx, (unsigned)gy);
}

int launch_tdot(krb_context *ctx, int64_t n, int64_t k, const double *M,
                int64_t ldm, const double *v, bool self, double *out,
                const int *status, cudaStream_t st, bool self_sqrt) {
  (void)status;
  if (k <= 0) return KRB_OK;
  int64_t nb = canon_nblocks(n);
  if (nb == 0) {
    KRB_CHECK_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * k, st));
    return KRB_OK;
  }
  int rc = ctx_reserve_part(ctx, (size_t)(k * nb));
  if (rc) return rc;
  rc = ctx_reserve_counters(ctx, st);
  if (rc) return rc;
  static int per_sm = occupancy_1024(k_tdot<16, false, false>);
  dim3 grid = tdot_grid(nb, k, per_sm);
  unsigned int *cnt = ctx->counters + kCounterTdotStandalone;
  if (self) {
    if (self_sqrt) {
      KRB_DISPATCH_E(canon_E(n), (k_tdot<kE, true, true><<<grid, 1024, 0, st>>>(
                                     n, nb, (int)k, M, ldm, v, ctx->part, out, cnt)));
    } else {
      KRB_DISPATCH_E(canon_E(n), (k_tdot<kE, true, false><<<grid, 1024, 0, st>>>(
                                     n, nb, (int)k, M, ldm, v, ctx->part, out, cnt)));
    }
  } else {
    KRB_DISPATCH_E(canon_E(n), (k_tdot<kE, false, false><<<grid, 1024, 0, st>>>(
                                   n, nb, (int)k, M, ldm, v, ctx->part, out, cnt)));
  }
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int ctx_reserve_counters(krb_context *ctx, cudaStream_t st) {
  if (ctx->counters) return KRB_OK;
  KRB_CHECK_CUDA(cudaMalloc(&ctx->counters, sizeof(unsigned int) * kNumCounters));
  KRB_CHECK_CUDA(cudaMemsetAsync(ctx->counters, 0, sizeof(unsigned int) * kNumCounters, st));
  return KRB_OK;
}

int launch_gemv(int64_t n, int64_t k, const double *M, int64_t ldm,
                const double *y, const double *base, int sign, double *out,
                cudaStream_t st) {
  if (n == 0) return KRB_OK;
  int64_t blocks = (n + 255) / 256;
  int grid = (int)(blocks < kNumSMs * 16 ? blocks : kNumSMs * 16);
  k_gemv<<<grid, 256, sizeof(double) * (k > 0 ? k : 1), st>>>(n, (int)k, M, ldm, y, base, sign, out);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int ctx_reserve_part(krb_context *ctx, size_t doubles) {
  if (doubles <= ctx->part_cap) return KRB_OK;
  if (ctx->part) cudaFree(ctx->part);
  ctx->part = nullptr;
  size_t cap = doubles < 4096 ? 4096 : doubles;
  KRB_CHECK_CUDA(cudaMalloc(&ctx->part, cap * sizeof(double)));
  ctx->part_cap = cap;
  ctx->graph.reset();  // graphs bake the partial-buffer pointer
  return KRB_OK;
}

}  // namespace krb

using namespace krb;

extern "C" {

int krb_dot(krb_context *ctx, int64_t n, const double *d_x, const double *d_y,
            double *d_out, void *stream) {
  KRB_REQUIRE(ctx != nullptr, "krb_dot: NULL context");
  cudaStream_t st = as_stream(stream);
  int64_t nb = canon_nblocks(n);
  if (nb == 0) {
    KRB_CHECK_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), st));
    return KRB_OK;
  }
  int rc = ctx_reserve_part(ctx, (size_t)nb);
  if (rc) return rc;
  rc = launch_dot_partials(n, d_x, d_y, ctx->part, st);
  if (rc) return rc;
  return launch_final(1, nb, ctx->part, d_out, st);
}

int krb_tdot(krb_context *ctx, int64_t n, int64_t k, const double *d_M,
             int64_t ldm, const double *d_v, double *d_out, void *stream) {
  KRB_REQUIRE(ctx != nullptr, "krb_tdot: NULL context");
  KRB_REQUIRE(ldm >= n, "krb_tdot: ldm < n");
  return launch_tdot(ctx, n, k, d_M, ldm, d_v, false, d_out, nullptr,
                     as_stream(stream));
}

int krb_colnorms(krb_context *ctx, int64_t n, int64_t k, const double *d_X,
                 int64_t ldx, double *d_out, void *stream) {
  KRB_REQUIRE(ctx != nullptr, "krb_colnorms: NULL context");
  KRB_REQUIRE(ldx >= n, "krb_colnorms: ldx < n");
  return launch_tdot(ctx, n, k, d_X, ldx, nullptr, true, d_out, nullptr,
                     as_stream(stream), true);
}

int krb_colsq(krb_context *ctx, int64_t n, int64_t k, const double *d_X,
              int64_t ldx, double *d_out, void *stream) {
  KRB_REQUIRE(ctx != nullptr, "krb_colsq: NULL context");
  KRB_REQUIRE(ldx >= n, "krb_colsq: ldx < n");
  return launch_tdot(ctx, n, k, d_X, ldx, nullptr, true, d_out, nullptr,
                     as_stream(stream), false);
}

int krb_ritz_combine(int64_t n, int64_t m, const double *d_Yre,
                     const double *d_Yim, double *d_Are, double *d_Aim,
                     int64_t ld, const double *d_thr, const double *d_thi,
                     void *stream) {
  KRB_REQUIRE(ld >= n, "krb_ritz_combine: ld < n");
  if (n * m == 0) return KRB_OK;
  int64_t blocks = (n * m + 255) / 256;
  int grid = (int)(blocks < kNumSMs * 16 ? blocks : kNumSMs * 16);
  k_ritz_combine<<<grid, 256, 0, as_stream(stream)>>>(n, (int)m, d_Yre, d_Yim, d_Are,
                                                      d_Aim, ld, d_thr, d_thi);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int krb_gemv(int64_t n, int64_t k, const double *d_M, int64_t ldm,
             const double *d_y, const double *d_base, int sign, double *d_out,
             void *stream) {
  KRB_REQUIRE(ldm >= n || k == 0, "krb_gemv: ldm < n");
  return launch_gemv(n, k, d_M, ldm, d_y, d_base, sign, d_out,
                     as_stream(stream));
}

int krb_gram(krb_context *ctx, int64_t n, int64_t na, int64_t nc,
             const double *d_X, int64_t ldx, const double *d_Y, int64_t ldy,
             double *d_G, void *stream) {
  KRB_REQUIRE(ctx != nullptr, "krb_gram: NULL context");
  KRB_REQUIRE(na * nc <= 256 * kGramMaxEnt, "krb_gram: na*nc > 4096");
  KRB_REQUIRE(ldx >= n && ldy >= n, "krb_gram: leading dimension < n");
  cudaStream_t st = as_stream(stream);
  int64_t ne = na * nc;
  if (ne == 0) return KRB_OK;
  int64_t R = canon_R(n);
  int64_t nch = n <= 0 ? 0 : (n + R - 1) / R;
  if (nch == 0) {
    KRB_CHECK_CUDA(cudaMemsetAsync(d_G, 0, sizeof(double) * ne, st));
    return KRB_OK;
  }
  int rc = ctx_reserve_part(ctx, (size_t)(ne * nch));
  if (rc) return rc;
  // m <= 48: 64-thread groups (k_gram_g, 6 x 6 tiles at m = 47: 135 -> 114 us
  // at 262144 rows); m <= 64: 256 threads per chunk (k_gram_rt: 16 x 16 tiles
  // of 4 x 4 hold their own at m = 60, 9.0 ms vs 9.4 ms at C5's 16.8 M rows)
  const int64_t T8 = ((na > nc ? na : nc) + 7) / 8;
  if (T8 <= 6) {
    int rc = KRB_OK;
#define KRB_GRAM_G(TT)                                                                      \
  rc = launch_gram_g<TT, 4, 16>(n, R, nch, (int)na, (int)nc, d_X, ldx, d_Y, ldy, ctx->part, st)
    switch (T8) {
      case 1: KRB_GRAM_G(1); break;
      case 2: KRB_GRAM_G(2); break;
      case 3: KRB_GRAM_G(3); break;
      case 4: KRB_GRAM_G(4); break;
      case 5: KRB_GRAM_G(5); break;
      default: KRB_GRAM_G(6); break;
    }
#undef KRB_GRAM_G
    if (rc) return rc;
    KRB_CHECK_LAUNCH();
    return launch_final((int)ne, nch, ctx->part, d_G, st);
  }
  const int64_t T = ((na > nc ? na : nc) + 15) / 16;
  if (T <= 4) {
    const size_t smem = sizeof(double) * 2 * 2 * 16 * T * kGS;
    int grid = (int)(nch < kNumSMs * 2 ? nch : kNumSMs * 2);
#define KRB_GRAM_RT(TT)                                                                  \
  do {                                                                                   \
    KRB_CHECK_CUDA(cudaFuncSetAttribute(k_gram_rt<TT>,                                   \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                        (int)smem));                                     \
    k_gram_rt<TT><<<grid, 256, smem, st>>>(n, R, nch, (int)na, (int)nc, d_X, ldx, d_Y, ldy, \
                                           ctx->part);                                   \
  } while (0)
    switch (T) {
      case 1: KRB_GRAM_RT(1); break;
      case 2: KRB_GRAM_RT(2); break;
      case 3: KRB_GRAM_RT(3); break;
      default: KRB_GRAM_RT(4); break;
    }
#undef KRB_GRAM_RT
  } else {
    size_t smem = sizeof(double) * kGramTile * (na + nc);
    KRB_CHECK_CUDA(cudaFuncSetAttribute(k_gram_part,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    int grid = (int)(nch < kNumSMs * 4 ? nch : kNumSMs * 4);
    k_gram_part<<<grid, 256, smem, st>>>(n, R, nch, (int)na, (int)nc, d_X, ldx,
                                         d_Y, ldy, ctx->part);
  }
  KRB_CHECK_LAUNCH();
  return launch_final((int)ne, nch, ctx->part, d_G, st);
}

int krb_gemm(int64_t n, int64_t m, int64_t nc, const double *d_X, int64_t ldx,
             const double *d_Z, double *d_out, int64_t ldo, void *stream) {
  KRB_REQUIRE(ldx >= n && ldo >= n, "krb_gemm: leading dimension < n");
  KRB_REQUIRE(m * nc <= 8192, "krb_gemm: m*nc > 8192");
  cudaStream_t st = as_stream(stream);
  if (n == 0 || nc == 0) return KRB_OK;
  const int64_t ncp = ((nc + kGemmCT2 - 1) / kGemmCT2) * kGemmCT2;
  {
    // tiled kernels (tuning "gemm_mode" = 0 off, 8 / 12 / 24: columns per
    // thread, 122: 12 columns x 2 rows per thread; default: 122 for m <= 64
    // and nc >= 4 (47 x 47 at 262144 rows 97 -> 85 us, 26 x 26 54 -> 38 us),
    // else 12)
    const int tm = tuning().gemm_mode;
    const int mode = tm >= 0 ? tm : (m <= 64 && nc >= 4 ? 122 : 12);
    int rc = KRB_OK;
    if (m > 0 && mode == 8 && gemm_tiled<8>(n, m, nc, d_X, ldx, d_Z, d_out, ldo, st, &rc)) return rc;
    if (m > 0 && mode == 12 && gemm_tiled<12>(n, m, nc, d_X, ldx, d_Z, d_out, ldo, st, &rc)) return rc;
    if (m > 0 && mode == 24 && gemm_tiled<24>(n, m, nc, d_X, ldx, d_Z, d_out, ldo, st, &rc)) return rc;
    if (m > 0 && mode == 122 && gemm_tiled<12, 2>(n, m, nc, d_X, ldx, d_Z, d_out, ldo, st, &rc)) return rc;
  }
  size_t smem = sizeof(double) * (m * ncp > 0 ? m * ncp : 2);
  KRB_REQUIRE(smem <= 200 * 1024, "krb_gemm: Z too large for shared memory");
  KRB_CHECK_CUDA(cudaFuncSetAttribute(k_gemm,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  int64_t blocks = (n + 255) / 256;
  int grid = (int)(blocks < kNumSMs * 2 ? blocks : kNumSMs * 2);
  k_gemm<<<grid, 256, smem, st>>>(n, (int)m, (int)nc, d_X, ldx, d_Z, d_out, ldo);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int krb_colscale_div(int64_t n, int64_t k, double *d_X, int64_t ldx,
                     const double *d_s, void *stream) {
  KRB_REQUIRE(ldx >= n, "krb_colscale_div: ldx < n");
  if (n * k == 0) return KRB_OK;
  // one pass: every element has its thread (grid.y <= 65535 columns)
  KRB_REQUIRE(k <= 65535, "krb_colscale_div: more than 65535 columns");
  const int64_t blocks = (n + 1023) / 1024;
  dim3 grid((unsigned)(blocks < 65535 ? blocks : 65535), (unsigned)k);
  k_colscale_div<<<grid, 256, 0, as_stream(stream)>>>(n, (int)k, d_X, ldx, d_s, d_X, ldx);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int krb_colscale_div_to(int64_t n, int64_t k, const double *d_X, int64_t ldx,
                        const double *d_s, double *d_Y, int64_t ldy, void *stream) {
  KRB_REQUIRE(ldx >= n && ldy >= n, "krb_colscale_div_to: leading dimension < n");
  if (n * k == 0) return KRB_OK;
  KRB_REQUIRE(k <= 65535, "krb_colscale_div_to: more than 65535 columns");
  const int64_t blocks = (n + 1023) / 1024;
  dim3 grid((unsigned)(blocks < 65535 ? blocks : 65535), (unsigned)k);
  k_colscale_div<<<grid, 256, 0, as_stream(stream)>>>(n, (int)k, d_X, ldx, d_s, d_Y, ldy);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int krb_uniform_pcg64(int64_t n, uint64_t state_hi, uint64_t state_lo,
                      uint64_t inc_hi, uint64_t inc_lo, double lo, double hi,
                      double *d_out, void *stream) {
  if (n <= 0) return KRB_OK;
  const int64_t threads = (n + kPcgRun - 1) / kPcgRun;
  const int64_t grid = (threads + 255) / 256;
  KRB_REQUIRE(grid < (int64_t)1 << 31, "krb_uniform_pcg64: n too large");
  k_pcg64_uniform<<<(unsigned)grid, 256, 0, as_stream(stream)>>>(
      n, state_hi, state_lo, inc_hi, inc_lo, lo, hi - lo, d_out);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

}  // extern "C"
