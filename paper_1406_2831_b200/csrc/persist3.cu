// Fused persistent RBiCGSTAB for large systems (v3: canon_E >= 4, C3 / C5):
// the pass structure of the fused kernel in persist.cu -- five grid barriers
// per iteration,
//   A  p' on the fly; q' = A p'; Chat^T q' partials          | sync
//   B  q' -= C zeta; (rt0, q'), (q', q')                      | sync
//   C  s = r - alpha q' on the fly; (s, s); t = A s; Chat^T t | sync
//   D  t -= C gamma; (t, t), (t, s)                           | sync
//   E  x += alpha p' + omega s; r = s - omega t; dots         | sync
// (k = 0: B's and D's dots come with A and C, three barriers) -- but every
// CTA owns any number of canonical blocks (me, me + G, ...), and a block's
// E elements per thread round-trip through global memory (L1 / L2-hot: the
// owner just wrote them) instead of living in registers.  Fusing P into the
// SpMV and the projection dots into the SpMV phase turns nine streaming
// passes per iteration into five larger ones (HBM bandwidth grows with the
// bytes per pass, tools/read_bw.cu).  The recycle blocks stream through the
// same per-thread cp.async ring (3 x 64 KB).  Bit-identical to every other
// driver (same canonical blocks, lane chains, trees and scalar logic).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "iter.cuh"
#include "spmv.cuh"
#include "tdot.cuh"

namespace krb {
namespace p3 {

namespace cg = cooperative_groups;

constexpr int kStages = 3;
constexpr int kTile = 8;
constexpr int kMaxK = 32;
constexpr size_t kStageBytes = (size_t)kStages * kTile * kLanes * sizeof(double);

template <int kE>
__device__ __forceinline__ int64_t elem(int64_t b, int e) {
  return b * ((int64_t)kLanes * kE) + (int64_t)kLanes * e + threadIdx.x;
}

struct Pass {
  const double *M;
  int64_t ld, n, me, G;
  int k, ncg;
};

// tile t of a pass: kDot -> (owned block, group, e); else (owned block, e, group)
template <int kE, bool kDot>
__device__ __forceinline__ void issue(double *stage, const Pass &P, int t, uint64_t pol) {
  const int per = P.ncg * kE;
  const int bi = t / per, rem = t - bi * per;
  const int g = kDot ? rem / kE : rem % P.ncg;
  const int e = kDot ? rem % kE : rem / P.ncg;
  const int64_t i = elem<kE>(P.me + (int64_t)bi * P.G, e);
  const bool ok = i < P.n;
  const int j0 = g * kTile;
  const double *src = P.M + (int64_t)j0 * P.ld + (ok ? i : 0);
  double *dst = stage + ((size_t)(t % kStages) * kTile << 10) + threadIdx.x;
#pragma unroll
  for (int c = 0; c < kTile; ++c)
    if (j0 + c < P.k) cp_async8(dst + ((size_t)c << 10), src + (int64_t)c * P.ld, ok, pol);
}

template <int kE, bool kDot>
__device__ __forceinline__ void prologue(double *stage, const Pass &P, int T, uint64_t pol) {
#pragma unroll
  for (int t = 0; t < kStages; ++t) {
    if (t < T) issue<kE, kDot>(stage, P, t, pol);
    cp_async_commit();
  }
}

// Chat^T v partials of owned block bi (v read back from global: the owner
// wrote it this phase); consumes tiles [bi*ncg*kE, (bi+1)*ncg*kE)
template <int kE>
__device__ __forceinline__ void proj_block(double *stage, const Pass &P, int T, int bi,
                                           const double *v, double (*wred)[32],
                                           double *part, int64_t nb, uint64_t pol) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = P.me + (int64_t)bi * P.G;
  int t = bi * P.ncg * kE;
  for (int g = 0; g < P.ncg; ++g) {
    const int j0 = g * kTile;
    const int nj = min(kTile, P.k - j0);
    double acc[kTile];
#pragma unroll
    for (int c = 0; c < kTile; ++c) acc[c] = 0.0;
#pragma unroll 2
    for (int e = 0; e < kE; ++e, ++t) {
      const int64_t i = elem<kE>(b, e);
      const double vi = i < P.n ? v[i] : 0.0;
      cp_async_wait<kStages - 1>();
      const double *src = stage + ((size_t)(t % kStages) * kTile << 10) + threadIdx.x;
      if (i < P.n) {
#pragma unroll
        for (int c = 0; c < kTile; ++c)
          if (c < nj) acc[c] = __fma_rn(src[(size_t)c << 10], vi, acc[c]);
      }
      if (t + kStages < T) issue<kE, true>(stage, P, t + kStages, pol);
      cp_async_commit();
    }
    int col;
    double w = warp_tree_multi<kTile>(acc, col);
    if ((lane & 3) == 0 && col < nj) wred[j0 + col][warp] = w;
  }
  __syncthreads();
  for (int c = warp; c < P.k; c += 32) {
    double r = warp_tree(wred[c][lane]);
    if (lane == 0) part[(int64_t)c * nb + b] = r;
  }
  __syncthreads();
}

// v -= C coef for owned block bi, then the phase's two dots (block partials);
// kT: (t, t), (t, s) else (rt0, q), (q, q).  Tiles (bi, e, g).
template <int kE, bool kT>
__device__ __forceinline__ void correct_block(double *stage, const Pass &P, int T, int bi,
                                              const double *coef, double *v, const double *s,
                                              const double *rt0, double (*red)[32],
                                              double *part, int64_t nb, uint64_t pol) {
  const int64_t b = P.me + (int64_t)bi * P.G;
  int t = bi * P.ncg * kE;
  double acc[2] = {0.0, 0.0};
#pragma unroll 2
  for (int e = 0; e < kE; ++e) {
    const int64_t i = elem<kE>(b, e);
    const bool ok = i < P.n;
    double vi = ok ? v[i] : 0.0;
    const double w2 = ok ? (kT ? s[i] : rt0[i]) : 0.0;
    double cz = 0.0;
    for (int g = 0; g < P.ncg; ++g, ++t) {
      cp_async_wait<kStages - 1>();
      const double *src = stage + ((size_t)(t % kStages) * kTile << 10) + threadIdx.x;
      const int j0 = g * kTile;
      const int nj = min(kTile, P.k - j0);
      if (ok) {
#pragma unroll
        for (int c = 0; c < kTile; ++c)
          if (c < nj) cz = __fma_rn(src[(size_t)c << 10], coef[j0 + c], cz);
      }
      if (t + kStages < T) issue<kE, false>(stage, P, t + kStages, pol);
      cp_async_commit();
    }
    if (ok) {
      if (P.k > 0) {
        vi = __dsub_rn(vi, cz);   // solvers.py:307,329
        v[i] = vi;
      }
      if (kT) {
        acc[0] = __fma_rn(vi, vi, acc[0]);   // (t, t)
        acc[1] = __fma_rn(vi, w2, acc[1]);   // (t, s)
      } else {
        acc[0] = __fma_rn(w2, vi, acc[0]);   // (rt0, q)
        acc[1] = __fma_rn(vi, vi, acc[1]);   // (q, q)
      }
    }
  }
  double bp = block_tree_multi<2>(acc, red);
  const int warp = threadIdx.x >> 5;
  if (warp < 2 && (threadIdx.x & 31) == 0) part[warp * nb + b] = bp;
}

template <int ND>
__device__ __forceinline__ void block_partials(double (&acc)[2], double (*red)[32], double *part,
                                               int64_t nb, int64_t b, int row0) {
  double bp = block_tree_multi<ND>(acc, red);
  const int warp = threadIdx.x >> 5;
  if (warp < ND && (threadIdx.x & 31) == 0) part[(int64_t)(row0 + warp) * nb + b] = bp;
}

template <int kE, bool kSell>
__global__ void __launch_bounds__(1024, 1) k_persist3(const IterArgs *__restrict__ pa) {
  extern __shared__ double stage[];
  __shared__ double zeta[kMaxK], gamma[kMaxK], xc[kMaxK];
  __shared__ double wred[kMaxK][32];
  __shared__ double red[8][32];
  __shared__ double dfin[3];
  __shared__ SolveScalars L;
  cg::grid_group grid = cg::this_grid();
  const IterArgs &a = *pa;
  const int64_t G = gridDim.x, me = blockIdx.x;
  const int64_t n = a.n, nb = a.nb;
  const int k = a.k;
  const int ncg = (k + kTile - 1) / kTile;
  const int nown = me < nb ? (int)((nb - 1 - me) / G + 1) : 0;
  const int Tt = nown * ncg * kE;
  const bool writer = me == 0;
  const krb_matrix A = a.A;
  const uint64_t pol = l2_policy(false);
  Pass PZ{a.Chat, a.ld, n, me, G, k, ncg}, PC{a.C, a.ld, n, me, G, k, ncg};
  double *__restrict__ x = a.x;
  double *__restrict__ r = a.r;
  double *__restrict__ s = a.s;
  double *__restrict__ tv_ = a.t;
  const double *__restrict__ rt0 = a.rt0;
  double *po = a.p, *pn = a.p2, *qo = a.q, *qn = a.q2;
  if (threadIdx.x == 0) L = *a.S;
  for (int j = threadIdx.x; j < k; j += blockDim.x) xc[j] = a.xc[j];
  __syncthreads();
  double *pb[2] = {a.part, a.part2};
  int cur = 0;
  if (k > 0) prologue<kE, true>(stage, PZ, Tt, pol);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (;;) {
    if (L.status != KRB_RUNNING) break;
    const double omega0 = L.omega, beta = L.beta;
    // ---- A
    {
      const double *__restrict__ r_ = r;
      const double *po_ = po, *qo_ = qo;
      auto pf = [=](int64_t c) {
        return __dadd_rn(r_[c], __dmul_rn(beta, __dsub_rn(po_[c], __dmul_rn(omega0, qo_[c]))));
      };
      for (int bi = 0; bi < nown; ++bi) {
        const int64_t b = me + (int64_t)bi * G;
        double acc[2] = {0.0, 0.0};
#pragma unroll 2
        for (int e = 0; e < kE; ++e) {
          const int64_t i = elem<kE>(b, e);
          if (i < n) {
            pn[i] = pf(i);   // solvers.py:303
            const double qv = spmv_row_f<kSell>(i, A, pf);
            qn[i] = qv;
            if (k == 0) {
              acc[0] = __fma_rn(rt0[i], qv, acc[0]);   // (rt0, q)
              acc[1] = __fma_rn(qv, qv, acc[1]);       // (q, q)
            }
          }
        }
        if (k > 0)
          proj_block<kE>(stage, PZ, Tt, bi, qn, wred, pb[cur], nb, pol);
        else
          block_partials<2>(acc, red, pb[cur], nb, b, 0);
      }
    }
    if (k > 0) prologue<kE, false>(stage, PC, Tt, pol);
    grid.sync();
    if (k > 0) {
      tdot_finals<false>(nb, k, pb[cur], zeta);
      __syncthreads();
      cur ^= 1;
      // ---- B
      for (int bi = 0; bi < nown; ++bi)
        correct_block<kE, false>(stage, PC, Tt, bi, zeta, qn, s, rt0, red, pb[cur], nb, pol);
      prologue<kE, true>(stage, PZ, Tt, pol);
      grid.sync();
    }
    if (warp < 2) {
      double v = warp_final_volatile(pb[cur] + warp * nb, nb);
      if (lane == 0) dfin[warp] = v;
    }
    __syncthreads();
    cur ^= 1;
    if (threadIdx.x == 0) finalize<PH_PROJ_Q>(a, &L, dfin, writer);
    __syncthreads();
    if (L.status != KRB_RUNNING) break;
    const double alpha = L.alpha;
    // ---- C
    {
      const double *__restrict__ r_ = r;
      const double *qn_ = qn;
      auto sf = [=](int64_t c) { return __dsub_rn(r_[c], __dmul_rn(alpha, qn_[c])); };
      for (int bi = 0; bi < nown; ++bi) {
        const int64_t b = me + (int64_t)bi * G;
        double acc[2] = {0.0, 0.0}, acc2[2] = {0.0, 0.0};
#pragma unroll 2
        for (int e = 0; e < kE; ++e) {
          const int64_t i = elem<kE>(b, e);
          if (i < n) {
            const double sv = __dsub_rn(r[i], __dmul_rn(alpha, qn[i]));   // :313
            s[i] = sv;
            acc[0] = __fma_rn(sv, sv, acc[0]);
            const double tv = spmv_row_f<kSell>(i, A, sf);
            tv_[i] = tv;
            if (k == 0) {
              acc2[0] = __fma_rn(tv, tv, acc2[0]);   // (t, t)
              acc2[1] = __fma_rn(tv, sv, acc2[1]);   // (t, s)
            }
          }
        }
        block_partials<1>(acc, red, pb[cur], nb, b, k);   // (s, s) -> row k
        if (k > 0)
          proj_block<kE>(stage, PZ, Tt, bi, tv_, wred, pb[cur], nb, pol);
        else
          block_partials<2>(acc2, red, pb[cur], nb, b, 1);   // rows 1, 2
      }
    }
    if (k > 0) prologue<kE, false>(stage, PC, Tt, pol);
    grid.sync();
    {
      if (warp < k) {
        double v = warp_final_volatile(pb[cur] + warp * nb, nb);
        if (lane == 0) gamma[warp] = v;
      }
      if (k == 0 && warp < 2) {
        double v = warp_final_volatile(pb[cur] + (1 + warp) * nb, nb);
        if (lane == 0) dfin[1 + warp] = v;
      }
      if (warp == 31) {
        double v = warp_final_volatile(pb[cur] + (int64_t)k * nb, nb);
        if (lane == 0) dfin[0] = v;
      }
      __syncthreads();
      if (threadIdx.x == 0) finalize<PH_SUPD>(a, &L, dfin, writer);
      __syncthreads();
      cur ^= 1;
    }
    if (L.status != KRB_RUNNING) {
      // solvers.py:315-325: x += alpha p, xc += alpha zeta
      for (int bi = 0; bi < nown; ++bi)
        for (int e = 0; e < kE; ++e) {
          const int64_t i = elem<kE>(me + (int64_t)bi * G, e);
          if (i < n) x[i] = __dadd_rn(x[i], __dmul_rn(alpha, pn[i]));
        }
      for (int j = threadIdx.x; j < k; j += blockDim.x)
        xc[j] = __dadd_rn(xc[j], __dmul_rn(alpha, zeta[j]));
      __syncthreads();
      break;
    }
    // ---- D
    if (k > 0) {
      for (int bi = 0; bi < nown; ++bi)
        correct_block<kE, true>(stage, PC, Tt, bi, gamma, tv_, s, rt0, red, pb[cur], nb, pol);
      prologue<kE, true>(stage, PZ, Tt, pol);   // next A
      grid.sync();
      if (warp < 2) {
        double v = warp_final_volatile(pb[cur] + warp * nb, nb);
        if (lane == 0) dfin[warp] = v;
      }
      __syncthreads();
      cur ^= 1;
      if (threadIdx.x == 0) finalize<PH_PROJ_T>(a, &L, dfin, writer);
    } else if (threadIdx.x == 0) {
      finalize<PH_PROJ_T>(a, &L, dfin + 1, writer);
    }
    __syncthreads();
    if (L.status != KRB_RUNNING) break;
    const double omega = L.omega;
    // ---- E
    for (int bi = 0; bi < nown; ++bi) {
      const int64_t b = me + (int64_t)bi * G;
      double acc[2] = {0.0, 0.0};
#pragma unroll 2
      for (int e = 0; e < kE; ++e) {
        const int64_t i = elem<kE>(b, e);
        if (i < n) {
          const double sv = s[i];
          x[i] = __dadd_rn(__dadd_rn(x[i], __dmul_rn(alpha, pn[i])),
                           __dmul_rn(omega, sv));                       // :338
          const double rv = __dsub_rn(sv, __dmul_rn(omega, tv_[i]));   // :341
          r[i] = rv;
          acc[0] = __fma_rn(rv, rv, acc[0]);
          acc[1] = __fma_rn(rt0[i], rv, acc[1]);
        }
      }
      block_partials<2>(acc, red, pb[cur], nb, b, 0);
    }
    for (int j = threadIdx.x; j < k; j += blockDim.x)   // solvers.py:340
      xc[j] = __dadd_rn(__dadd_rn(xc[j], __dmul_rn(alpha, zeta[j])), __dmul_rn(omega, gamma[j]));
    grid.sync();
    if (warp < 2) {
      double v = warp_final_volatile(pb[cur] + warp * nb, nb);
      if (lane == 0) dfin[warp] = v;
    }
    __syncthreads();
    cur ^= 1;
    if (threadIdx.x == 0) finalize<PH_XR>(a, &L, dfin, writer);
    __syncthreads();
    double *tp = po; po = pn; pn = tp;
    double *tq = qo; qo = qn; qn = tq;
  }
  cp_async_wait<0>();
  if (writer) {
    if (threadIdx.x == 0) {
      L.bodies = L.itn;
      *a.S = L;
    }
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      a.xc[j] = xc[j];
      a.zeta[j] = zeta[j];
      a.gamma[j] = gamma[j];
    }
  }
}

template <int kE, bool kSell>
static int launch_t(const IterArgs *d, cudaStream_t st) {
  static int grid = 0;
  if (grid == 0) {
    KRB_CHECK_CUDA(cudaFuncSetAttribute(k_persist3<kE, kSell>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kStageBytes));
    int per_sm = 0;
    KRB_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, k_persist3<kE, kSell>, 1024, kStageBytes));
    int dev = 0, sms = kNumSMs;
    KRB_CHECK_CUDA(cudaGetDevice(&dev));
    KRB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = per_sm > 0 ? sms : 0;
    if (grid == 0) {
      set_error("large-n fused persistent kernel does not fit on an SM");
      return KRB_ECUDA;
    }
  }
  void *args[] = {(void *)&d};
  KRB_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)k_persist3<kE, kSell>,
                                             dim3(grid), dim3(1024), args, kStageBytes, st));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

}  // namespace p3

bool persist3_eligible(const IterArgs &h) {
  return h.A.perm == nullptr && h.k <= p3::kMaxK && canon_E(h.n) >= 4;
}

int persist3_launch(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  const bool sell = h.A.format == 2;
  switch (canon_E(h.n)) {
    case 4: return sell ? p3::launch_t<4, true>(d, st) : p3::launch_t<4, false>(d, st);
    case 8: return sell ? p3::launch_t<8, true>(d, st) : p3::launch_t<8, false>(d, st);
    default: return sell ? p3::launch_t<16, true>(d, st) : p3::launch_t<16, false>(d, st);
  }
}

}  // namespace krb
