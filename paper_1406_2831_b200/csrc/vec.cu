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

// Register-tiled Gram chunk partials (same order as k_gram_part): each thread
// owns a 4 x 4 tile of entries and runs their 16 sequential fma chains over
// the chunk's rows, so a row costs 8 shared loads for 16 fma instead of 2
// per fma.  Sub-tiles of kGT rows are staged column-major (padded stride)
// with coalesced loads.  Requires ceil(na/4) * ceil(nc/4) <= 256.
constexpr int kGemmCT = 8;
constexpr int kGT = 64;
constexpr int kGS = kGT + 1;   // padded column stride in shared memory
__global__ void __launch_bounds__(256) k_gram_tiled(
    int64_t n, int64_t R, int64_t nch, int na, int nc,
    const double *__restrict__ X, int64_t ldx, const double *__restrict__ Y,
    int64_t ldy, double *__restrict__ part) {
  extern __shared__ double sm[];
  const int na4 = (na + 3) & ~3, nc4 = (nc + 3) & ~3;
  double *xs = sm;                  // [na4][kGS]
  double *ys = sm + na4 * kGS;      // [nc4][kGS]
  const int ntc = nc4 >> 2, ntile = (na4 >> 2) * ntc;
  const int tid = threadIdx.x;
  const int a0 = (tid / ntc) * 4, c0 = (tid % ntc) * 4;
  for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    const int64_t r0 = ch * R;
    const int64_t r1 = min(n, r0 + R);
    for (int64_t t0 = r0; t0 < r1; t0 += kGT) {
      const int rows = (int)min((int64_t)kGT, r1 - t0);
      __syncthreads();
      for (int idx = tid; idx < na4 * kGT; idx += blockDim.x) {
        const int a = idx / kGT, rr = idx - a * kGT;
        xs[a * kGS + rr] = (a < na && rr < rows) ? __ldg(X + (int64_t)a * ldx + t0 + rr) : 0.0;
      }
      for (int idx = tid; idx < nc4 * kGT; idx += blockDim.x) {
        const int c = idx / kGT, rr = idx - c * kGT;
        ys[c * kGS + rr] = (c < nc && rr < rows) ? __ldg(Y + (int64_t)c * ldy + t0 + rr) : 0.0;
      }
      __syncthreads();
      if (tid < ntile) {
        for (int rr = 0; rr < rows; ++rr) {
          double xv[4], yv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) xv[i] = xs[(a0 + i) * kGS + rr];
#pragma unroll
          for (int j = 0; j < 4; ++j) yv[j] = ys[(c0 + j) * kGS + rr];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(xv[i], yv[j], acc[i][j]);
        }
      }
    }
    if (tid < ntile) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (a0 + i < na && c0 + j < nc)
            part[(int64_t)((a0 + i) * nc + c0 + j) * nch + ch] = acc[i][j];
    }
  }
}

// out[i + c*ldo] = sum_j X[i + j*ldx] Z[j*nc + c]  (sequential fma, j order)
__global__ void __launch_bounds__(256) k_gemm(int64_t n, int m, int nc,
                                              const double *__restrict__ X,
                                              int64_t ldx,
                                              const double *__restrict__ Z,
                                              double *__restrict__ out,
                                              int64_t ldo) {
  extern __shared__ double zs[];
  for (int idx = threadIdx.x; idx < m * nc; idx += blockDim.x) zs[idx] = Z[idx];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int c0 = 0; c0 < nc; c0 += kGemmCT) {
      double acc[kGemmCT];
#pragma unroll
      for (int t = 0; t < kGemmCT; ++t) acc[t] = 0.0;
      for (int j = 0; j < m; ++j) {
        double xv = __ldg(X + (int64_t)j * ldx + i);
#pragma unroll
        for (int t = 0; t < kGemmCT; ++t)
          if (c0 + t < nc) acc[t] = __fma_rn(xv, zs[j * nc + c0 + t], acc[t]);
      }
#pragma unroll
      for (int t = 0; t < kGemmCT; ++t)
        if (c0 + t < nc) out[(int64_t)(c0 + t) * ldo + i] = acc[t];
    }
  }
}

__global__ void k_colscale_div(int64_t n, int k, double *X, int64_t ldx,
                               const double *__restrict__ s) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       idx < n * k; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = idx / n, i = idx % n;
    X[j * ldx + i] = __ddiv_rn(X[j * ldx + i], s[j]);
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

// element i uses state LCG^(i+1)(s0); thread g handles i = g, g+T, ...
__global__ void k_pcg64_uniform(int64_t n, uint64_t s_hi, uint64_t s_lo,
                                uint64_t i_hi, uint64_t i_lo, double lo,
                                double range, double *out) {
  const u128 mult = mk128(kPcgMulHi, kPcgMulLo), inc = mk128(i_hi, i_lo);
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  u128 A, C, AT, CT;
  pcg_jump(mult, inc, (uint64_t)g + 1, &A, &C);
  u128 s = A * mk128(s_hi, s_lo) + C;
  pcg_jump(mult, inc, (uint64_t)T, &AT, &CT);
  for (int64_t i = g; i < n; i += T) {
    uint64_t r = pcg_out(s);
    double u = (double)(r >> 11) * (1.0 / 9007199254740992.0);
    out[i] = __dadd_rn(lo, __dmul_rn(range, u));
    s = AT * s + CT;
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

dim3 tdot_grid(int64_t nb, int64_t k) {
  int64_t gy = (k + kTdotCG - 1) / kTdotCG;
  int64_t want = (int64_t)kNumSMs * 2;
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
  dim3 grid = tdot_grid(nb, k);
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
  const int64_t na4 = (na + 3) & ~3, nc4 = (nc + 3) & ~3;
  if ((na4 / 4) * (nc4 / 4) <= 256) {
    size_t smem = sizeof(double) * kGS * (na4 + nc4);
    KRB_CHECK_CUDA(cudaFuncSetAttribute(k_gram_tiled,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    int grid = (int)(nch < kNumSMs * 4 ? nch : kNumSMs * 4);
    k_gram_tiled<<<grid, 256, smem, st>>>(n, R, nch, (int)na, (int)nc, d_X, ldx, d_Y, ldy,
                                          ctx->part);
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
  size_t smem = sizeof(double) * (m * nc > 0 ? m * nc : 1);
  KRB_CHECK_CUDA(cudaFuncSetAttribute(k_gemm,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  int64_t blocks = (n + 255) / 256;
  int grid = (int)(blocks < kNumSMs * 8 ? blocks : kNumSMs * 8);
  k_gemm<<<grid, 256, smem, st>>>(n, (int)m, (int)nc, d_X, ldx, d_Z, d_out, ldo);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int krb_colscale_div(int64_t n, int64_t k, double *d_X, int64_t ldx,
                     const double *d_s, void *stream) {
  KRB_REQUIRE(ldx >= n, "krb_colscale_div: ldx < n");
  if (n * k == 0) return KRB_OK;
  int64_t blocks = (n * k + 255) / 256;
  int grid = (int)(blocks < kNumSMs * 16 ? blocks : kNumSMs * 16);
  k_colscale_div<<<grid, 256, 0, as_stream(stream)>>>(n, (int)k, d_X, ldx, d_s);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int krb_uniform_pcg64(int64_t n, uint64_t state_hi, uint64_t state_lo,
                      uint64_t inc_hi, uint64_t inc_lo, double lo, double hi,
                      double *d_out, void *stream) {
  if (n <= 0) return KRB_OK;
  int64_t blocks = (n + 255) / 256;
  int grid = (int)(blocks < kNumSMs * 8 ? blocks : kNumSMs * 8);
  k_pcg64_uniform<<<grid, 256, 0, as_stream(stream)>>>(
      n, state_hi, state_lo, inc_hi, inc_lo, lo, hi - lo, d_out);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

}  // extern "C"
