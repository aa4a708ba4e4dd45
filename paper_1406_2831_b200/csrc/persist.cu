// Persistent (one cooperative kernel per solve) BiCGSTAB drivers.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "iter.cuh"
#include "spmv.cuh"
#include "tdot.cuh"

namespace krb {

namespace cg = cooperative_groups;

// ---------------------------------------------------------------------------
// persistent driver: the whole solve in one cooperative kernel
//
// Phases are separated by cooperative-groups grid barriers (~1.2 us on B200,
// one round trip).  After a barrier EVERY CTA runs the canonical final stage
// of the phase's dots and the scalar logic itself, on its own shared copy of
// the scalar block: the inputs are the same partials in the same order, so
// every copy is bit-identical and no second barrier is needed to broadcast
// the scalars.  CTA 0 alone writes the history and, at the end, the scalar
// block and xc back to global memory.
// ---------------------------------------------------------------------------
template <int ND>
__device__ __forceinline__ void local_finals(const IterArgs &a, const double *pb,
                                             double *dfin) {
  const int warp = threadIdx.x >> 5;
  if (warp < ND) {
    double v = warp_final_volatile(pb + warp * a.nb, a.nb);
    if ((threadIdx.x & 31) == 0) dfin[warp] = v;
  }
  __syncthreads();
}

template <int kE, bool kSell>
__global__ void __launch_bounds__(1024) k_persist(const IterArgs *__restrict__ pa) {
  __shared__ double zeta[512], gamma[512], xc[512];
  __shared__ double red[kTdotCG][32];
  __shared__ double dfin[3];
  __shared__ SolveScalars L;
  cg::grid_group grid = cg::this_grid();
  const IterArgs &a = *pa;
  const int64_t G = gridDim.x, me = blockIdx.x;
  const int64_t n = a.n, nb = a.nb;
  const int k = a.k;
  const int64_t ncg = (k + kTdotCG - 1) / kTdotCG;
  const bool writer = me == 0;
  const krb_matrix A = a.A;
  if (threadIdx.x == 0) L = *a.S;
  for (int j = threadIdx.x; j < k; j += blockDim.x) xc[j] = a.xc[j];
  __syncthreads();

  // Partials alternate between two buffers: a phase writes one while the
  // previous phase's partials (still being read by slower CTAs after their
  // barrier) stay intact in the other -- one barrier per phase.
  double *pb[2] = {a.part, a.part2};
  int cur = 0;
  uint64_t *prof = (writer && threadIdx.x == 0) ? a.prof : nullptr;
#define KRB_STAMP(slot)                                              \
  do {                                                               \
    if (prof && L.itn < a.prof_cap) prof[L.itn * 16 + (slot)] = globaltimer(); \
  } while (0)
  for (;;) {
    if (L.status != KRB_RUNNING) break;
    PhaseScal sc{L.alpha, L.omega, L.beta};
    KRB_STAMP(0);
    // P: p = r + beta (p - omega q)
    phase_blocks<kE, PH_PUPDATE>(a, sc, red, zeta, me, G, pb[cur]);
    grid.sync();
    KRB_STAMP(1);
    // M: q = A p
    for (int64_t i = me * blockDim.x + threadIdx.x; i < n; i += G * blockDim.x)
      a.q[(kSell && A.perm) ? A.perm[i] : i] = spmv_row<kSell, false>(i, A, a.p);
    grid.sync();
    KRB_STAMP(2);
    // Z: zeta = Chat^T q   (every CTA computes the k finals into smem)
    if (k > 0) {
      for (int64_t u = me; u < nb * ncg; u += G)
        tdot_unit<kE, false>(n, nb, k, a.Chat, a.ld, a.q, pb[cur], u % nb,
                             (int)(u / nb) * kTdotCG, red, a.l2keep != 0);
      grid.sync();
      tdot_finals<false>(nb, k, pb[cur], zeta);
      __syncthreads();
      cur ^= 1;
    }
    KRB_STAMP(3);
    // Q: q -= C zeta ; den, ||q|| -> alpha
    phase_blocks<kE, PH_PROJ_Q>(a, sc, red, zeta, me, G, pb[cur]);
    grid.sync();
    local_finals<2>(a, pb[cur], dfin);
    cur ^= 1;
    if (threadIdx.x == 0) finalize<PH_PROJ_Q>(a, &L, dfin, writer);
    __syncthreads();
    KRB_STAMP(4);
    if (L.status != KRB_RUNNING) break;
    sc.alpha = L.alpha;
    // S: s = r - alpha q ; ||s|| -> half-step exit
    phase_blocks<kE, PH_SUPD>(a, sc, red, zeta, me, G, pb[cur]);
    grid.sync();
    local_finals<1>(a, pb[cur], dfin);
    cur ^= 1;
    if (threadIdx.x == 0) finalize<PH_SUPD>(a, &L, dfin, writer);
    __syncthreads();
    KRB_STAMP(5);
    if (L.status != KRB_RUNNING) {
      // solvers.py:315-325: x += alpha p, xc += alpha zeta
      for (int64_t i = me * blockDim.x + threadIdx.x; i < n; i += G * blockDim.x)
        a.x[i] = __dadd_rn(a.x[i], __dmul_rn(sc.alpha, a.p[i]));
      for (int j = threadIdx.x; j < k; j += blockDim.x)
        xc[j] = __dadd_rn(xc[j], __dmul_rn(sc.alpha, zeta[j]));
      __syncthreads();
      break;
    }
    // M: t = A s
    for (int64_t i = me * blockDim.x + threadIdx.x; i < n; i += G * blockDim.x)
      a.t[(kSell && A.perm) ? A.perm[i] : i] = spmv_row<kSell, false>(i, A, a.s);
    grid.sync();
    KRB_STAMP(6);
    // Z: gamma = Chat^T t
    if (k > 0) {
      for (int64_t u = me; u < nb * ncg; u += G)
        tdot_unit<kE, false>(n, nb, k, a.Chat, a.ld, a.t, pb[cur], u % nb,
                             (int)(u / nb) * kTdotCG, red, a.l2keep != 0);
      grid.sync();
      tdot_finals<false>(nb, k, pb[cur], gamma);
      __syncthreads();
      cur ^= 1;
    }
    KRB_STAMP(7);
    // T: t -= C gamma ; (t,t), (t,s) -> omega
    phase_blocks<kE, PH_PROJ_T>(a, sc, red, gamma, me, G, pb[cur]);
    grid.sync();
    local_finals<2>(a, pb[cur], dfin);
    cur ^= 1;
    if (threadIdx.x == 0) finalize<PH_PROJ_T>(a, &L, dfin, writer);
    __syncthreads();
    KRB_STAMP(8);
    if (L.status != KRB_RUNNING) break;
    sc.omega = L.omega;
    // X: x, r ; ||r||, (rt0, r) -> record, convergence, rho, beta
    phase_blocks<kE, PH_XR>(a, sc, red, zeta, me, G, pb[cur]);
    for (int j = threadIdx.x; j < k; j += blockDim.x)   // solvers.py:340
      xc[j] = __dadd_rn(__dadd_rn(xc[j], __dmul_rn(sc.alpha, zeta[j])),
                        __dmul_rn(sc.omega, gamma[j]));
    grid.sync();
    local_finals<2>(a, pb[cur], dfin);
    cur ^= 1;
    KRB_STAMP(9);
    if (threadIdx.x == 0) finalize<PH_XR>(a, &L, dfin, writer);
    __syncthreads();
  }
#undef KRB_STAMP
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
static int persist_launch(const IterArgs *d, cudaStream_t st) {
  static int grid = 0;
  if (grid == 0) {
    int per_sm = 0;
    KRB_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, k_persist<kE, kSell>, 1024, 0));
    int dev = 0, sms = kNumSMs;
    KRB_CHECK_CUDA(cudaGetDevice(&dev));
    KRB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = (per_sm > 0 ? per_sm : 1) * sms;
  }
  void *args[] = {(void *)&d};
  KRB_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)k_persist<kE, kSell>,
                                             dim3(grid), dim3(1024), args, 0, st));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

// ---------------------------------------------------------------------------
// fused persistent driver (v2): five grid barriers per iteration
//
// Every CTA owns canonical blocks me, me + G (G = one CTA per SM >= nb / 2):
// the rows of its blocks for the SpMV, the elements of its blocks for every
// vector update and dot.  Owning the rows of a block lets one phase compute
// q = A p and, from registers, that block's partials of Chat^T q, so the
// projection needs no barrier of its own; and the vector updates that feed a
// SpMV (p = r + beta (p - omega q), s = r - alpha q) are recomputed on the fly
// for every gathered column instead of being written and fenced first (same
// formula, same bits).  p and q are double-buffered because the owner writes
// the new value while other CTAs still gather the old one.
//
//   A  p' = r + beta (p - omega q);  q' = A p';  Chat^T q' partials | sync
//   B  q' -= C zeta;  (rt0, q'), (q', q')  -> alpha                   | sync
//   C  s = r - alpha q';  (s, s);  t = A s;  Chat^T t partials         | sync
//   D  t -= C gamma;  (t, t), (t, s) -> omega                          | sync
//   E  x += alpha p' + omega s;  r = s - omega t;  (r, r), (rt0, r)    | sync
//
// The recycle blocks Chat / C stream through a 3-stage per-thread cp.async
// pipeline in shared memory (8 columns x 1024 elements = 64 KB per stage):
// each thread copies exactly the elements it consumes, so the copies need no
// CTA barrier and keep ~190 KB per SM in flight without occupying registers.
// The canonical block reductions are split so the streaming loops never
// synchronise the CTA: each warp runs its 32-lane trees as soon as its lane
// partials are complete and parks the results in shared memory (wred); one
// __syncthreads per phase then lets the warps run all the 32-warp trees.
// Every phase issues the next phase's tile prologue before its grid barrier,
// so those copies overlap the barrier and the final reductions.
// ---------------------------------------------------------------------------
#ifndef KRB_STAGES
#define KRB_STAGES 3
#endif
constexpr int kStages = KRB_STAGES;
constexpr int kMaxOwn = 2;       // canonical blocks per CTA (nb <= 2 G)
constexpr int kTileCols = 8;
constexpr int kV2MaxK = 32;      // recycle dimension limit of the fused kernel
constexpr int kWRow = kV2MaxK + 1;   // wred rows per owned block (k dots + 1)
constexpr size_t kStageBytes = (size_t)kStages * kTileCols * kLanes * sizeof(double);

template <int kE>
__device__ __forceinline__ int64_t owned_elem(int64_t b, int e) {
  return b * ((int64_t)kLanes * kE) + (int64_t)kLanes * e + threadIdx.x;
}

// stage tile (b, e, column group g) of M into slot `slot`
template <int kE>
__device__ __forceinline__ void issue_tile(double *stage, const double *M, int64_t ld,
                                           int64_t n, int k, int64_t b, int e, int g,
                                           int slot, uint64_t pol) {
  const int64_t i = owned_elem<kE>(b, e);
  const bool ok = i < n;
  const int j0 = g * kTileCols;
  const double *src = M + (int64_t)j0 * ld + (ok ? i : 0);
  double *dst = stage + ((size_t)slot * kTileCols << 10) + threadIdx.x;
#pragma unroll
  for (int c = 0; c < kTileCols; ++c)
    if (j0 + c < k) cp_async8(dst + ((size_t)c << 10), src + (int64_t)c * ld, ok, pol);
}

// tile t of a CTA's sequence; kDotOrder: (block, group, e) for projection
// dots, else (block, e, group) for C @ coef
template <int kE, bool kDotOrder>
__device__ __forceinline__ void issue_seq(double *stage, const double *M, int64_t ld,
                                          int64_t n, int k, int ncg, int64_t me,
                                          int64_t G, int t, uint64_t pol) {
  const int per = ncg * kE;
  const int bi = t >= per ? 1 : 0;   // kMaxOwn == 2
  const int rem = t - bi * per;
  const int g = kDotOrder ? (kE == 1 ? rem : rem >> 1) : (kE == 1 ? rem : rem % ncg);
  const int e = kDotOrder ? (kE == 1 ? 0 : rem & 1) : (kE == 1 ? 0 : rem / ncg);
  issue_tile<kE>(stage, M, ld, n, k, me + bi * G, e, g, t % kStages, pol);
}

template <int kE, bool kDotOrder>
__device__ __forceinline__ void prologue(double *stage, const double *M, int64_t ld,
                                         int64_t n, int k, int ncg, int64_t me, int64_t G,
                                         int T, uint64_t pol) {
#pragma unroll
  for (int t = 0; t < kStages; ++t) {
    if (t < T) issue_seq<kE, kDotOrder>(stage, M, ld, n, k, ncg, me, G, t, pol);
    cp_async_commit();
  }
}

// warp stage of ND (1 or 2) dots of owned block bi -> wred rows bi*kWRow + r0 + d
template <int ND>
__device__ __forceinline__ void warp_stage(double (&acc)[2], double (*wred)[32], int bi,
                                           int r0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (ND == 1) {
    double v = warp_tree(acc[0]);
    if (lane == 0) wred[bi * kWRow + r0][warp] = v;
  } else {
    int col;
    double v = warp_tree_multi<2>(acc, col);
    if ((lane & 15) == 0) wred[bi * kWRow + r0 + col][warp] = v;
  }
}

// CTA stage (after a __syncthreads): the 32-warp trees of `rows` dots per
// owned block; dot d of block b -> part[(p0 + d) * nb + b]
__device__ __forceinline__ void cta_stage(const double (*wred)[32], int nown, int rows,
                                          int r0, int p0, int64_t me, int64_t G, int64_t nb,
                                          double *part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int u = warp; u < nown * rows; u += 32) {
    const int bi = u / rows, d = u - bi * rows;
    double r = warp_tree(wred[bi * kWRow + r0 + d][lane]);
    if (lane == 0) part[(int64_t)(p0 + d) * nb + me + bi * G] = r;
  }
}

// Chat^T v of owned block bi, v in registers (vreg[bi][e]): lane partials
// and 32-lane trees per tile into wred rows 0..k-1 (no CTA barrier); consumes
// block bi's part of the tile sequence started by prologue<kE, true>.
template <int kE>
__device__ __forceinline__ void proj_block(double *stage, const double *M, int64_t ld,
                                           int64_t n, int k, int ncg, int64_t me,
                                           int64_t G, int nown, int bi,
                                           const double (&vreg)[kMaxOwn][kE],
                                           double (*wred)[32], uint64_t pol) {
  const int T = nown * ncg * kE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int t = bi * ncg * kE;
  const int64_t b = me + bi * G;
  for (int g = 0; g < ncg; ++g) {
    const int j0 = g * kTileCols;
    const int nj = min(kTileCols, k - j0);
    double acc[kTileCols];
#pragma unroll
    for (int c = 0; c < kTileCols; ++c) acc[c] = 0.0;
#pragma unroll
    for (int e = 0; e < kE; ++e, ++t) {
      cp_async_wait<kStages - 1>();
      const double *src = stage + ((size_t)(t % kStages) * kTileCols << 10) + threadIdx.x;
      if (owned_elem<kE>(b, e) < n) {
        const double vi = vreg[bi][e];
#pragma unroll
        for (int c = 0; c < kTileCols; ++c)
          if (c < nj) acc[c] = __fma_rn(src[(size_t)c << 10], vi, acc[c]);
      }
      if (t + kStages < T)
        issue_seq<kE, true>(stage, M, ld, n, k, ncg, me, G, t + kStages, pol);
      cp_async_commit();
    }
    int col;
    double w = warp_tree_multi<kTileCols>(acc, col);
    if ((lane & 3) == 0 && col < nj) wred[bi * kWRow + j0 + col][warp] = w;
  }
}

// v -= C coef for the owned elements (v in registers, written back), then the
// lane partials and warp trees of the phase's two dots into wred rows
// kV2MaxK - 1, kV2MaxK; consumes the tile sequence of prologue<kE, false>.
// kT: (t, t), (t, s) else (rt0, q), (q, q).
template <int kE, bool kT>
__device__ __forceinline__ void correct_warps(double *stage, const double *Cm, int64_t ld,
                                              int64_t n, int k, int ncg, int64_t me,
                                              int64_t G, int nown,
                                              double (&vreg)[kMaxOwn][kE],
                                              const double (&sreg)[kMaxOwn][kE],
                                              const double *coef, double *v,
                                              const double *rt0, double (*wred)[32],
                                              uint64_t pol) {
  const int T = nown * ncg * kE;
  int t = 0;
  double rt[kMaxOwn][kE];   // (rt0, q): loads issued before the tile waits
  if (!kT) {
#pragma unroll
    for (int bi = 0; bi < kMaxOwn; ++bi)
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        const int64_t i = owned_elem<kE>(me + bi * G, e);
        rt[bi][e] = (bi < nown && i < n) ? rt0[i] : 0.0;
      }
  }
#pragma unroll
  for (int bi = 0; bi < kMaxOwn; ++bi) {
    if (bi >= nown) break;
    const int64_t b = me + bi * G;
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int e = 0; e < kE; ++e) {
      const int64_t i = owned_elem<kE>(b, e);
      double cz = 0.0;
      for (int g = 0; g < ncg; ++g, ++t) {
        cp_async_wait<kStages - 1>();
        const double *src = stage + ((size_t)(t % kStages) * kTileCols << 10) + threadIdx.x;
        const int j0 = g * kTileCols;
        const int nj = min(kTileCols, k - j0);
        if (i < n) {
#pragma unroll
          for (int c = 0; c < kTileCols; ++c)
            if (c < nj) cz = __fma_rn(src[(size_t)c << 10], coef[j0 + c], cz);
        }
        if (t + kStages < T)
          issue_seq<kE, false>(stage, Cm, ld, n, k, ncg, me, G, t + kStages, pol);
        cp_async_commit();
      }
      if (i < n) {
        double vi = vreg[bi][e];
        if (k > 0) {
          vi = __dsub_rn(vi, cz);   // v - C @ coef   (solvers.py:307,329)
          v[i] = vi;
          vreg[bi][e] = vi;
        }
        if (kT) {
          acc[0] = __fma_rn(vi, vi, acc[0]);           // (t, t)
          acc[1] = __fma_rn(vi, sreg[bi][e], acc[1]);  // (t, s)
        } else {
          acc[0] = __fma_rn(rt[bi][e], vi, acc[0]);    // (rt0, q)
          acc[1] = __fma_rn(vi, vi, acc[1]);           // (q, q)
        }
      }
    }
    warp_stage<2>(acc, wred, bi, kV2MaxK - 1);
  }
}

template <int kE, bool kSell>
__global__ void __launch_bounds__(1024, 1) k_persist2(const IterArgs *__restrict__ pa) {
  extern __shared__ double stage[];   // kStages x kTileCols x 1024
  __shared__ double zeta[kV2MaxK], gamma[kV2MaxK], xc[kV2MaxK];
  __shared__ double wred[kMaxOwn * kWRow][32];
  __shared__ double dfin[3];
  __shared__ SolveScalars L;
  cg::grid_group grid = cg::this_grid();
  const IterArgs &a = *pa;
  const int64_t G = gridDim.x, me = blockIdx.x;
  const int64_t n = a.n, nb = a.nb, ld = a.ld;
  const int k = a.k;
  const int ncg = (k + kTileCols - 1) / kTileCols;
  const int nown = me < nb ? (int)((nb - 1 - me) / G + 1) : 0;
  const int Tt = nown * ncg * kE;   // tiles per projection / correction pass
  const bool writer = me == 0;
  const krb_matrix A = a.A;
  const uint64_t pol = l2_policy(a.l2keep);
  // matrix entries: evict_first when the recycle blocks are kept (l2keep)
  const uint64_t polm = a.l2keep ? l2_policy_first() : l2_policy(false);
  const double *__restrict__ Chat = a.Chat;
  const double *__restrict__ Cm = a.C;
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
  if (k > 0) prologue<kE, true>(stage, Chat, ld, n, k, ncg, me, G, Tt, pol);
  double preg[kMaxOwn][kE], qreg[kMaxOwn][kE], sreg[kMaxOwn][kE], treg[kMaxOwn][kE];
  // profiling: CTA 0 stamps each sub-phase after a CTA barrier (so a stamp
  // marks the slowest warp of CTA 0, not thread 0's own progress)
  const bool profiling = writer && a.prof != nullptr;
  uint64_t *prof = (profiling && threadIdx.x == 0) ? a.prof : nullptr;
#define KRB_STAMP(slot)                                                        \
  do {                                                                         \
    if (profiling) __syncthreads();                                            \
    if (prof && L.itn < a.prof_cap) prof[L.itn * 16 + (slot)] = globaltimer(); \
  } while (0)
  for (;;) {
    if (L.status != KRB_RUNNING) break;
    const double omega0 = L.omega, beta = L.beta;
    KRB_STAMP(0);
    // ---- A: p' = r + beta (p - omega q); q' = A p'; Chat^T q' partials
    // (per owned block: its rows' SpMV, then its projection tiles, so the
    // next block's tiles stream in while this block's SpMV runs)
    {
      const double *__restrict__ r_ = r;
      const double *po_ = po, *qo_ = qo;
      auto pf = [=](int c) {
        return __dadd_rn(r_[c], __dmul_rn(beta, __dsub_rn(po_[c], __dmul_rn(omega0, qo_[c]))));
      };
#pragma unroll
      for (int bi = 0; bi < kMaxOwn; ++bi) {
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          preg[bi][e] = qreg[bi][e] = 0.0;
          const int64_t i = owned_elem<kE>(me + bi * G, e);
          if (bi < nown && i < n) {
            const double pv = pf((int)i);   // solvers.py:303
            pn[i] = pv;
            preg[bi][e] = pv;
            const double qv = spmv_row_f<kSell, 4, true>(i, A, pf, polm);
            qn[i] = qv;
            qreg[bi][e] = qv;
          }
        }
        if (k > 0 && bi < nown)
          proj_block<kE>(stage, Chat, ld, n, k, ncg, me, G, nown, bi, qreg, wred, pol);
      }
    }
    KRB_STAMP(6);
    if (k > 0) {
      prologue<kE, false>(stage, Cm, ld, n, k, ncg, me, G, Tt, pol);
      __syncthreads();
      cta_stage(wred, nown, k, 0, 0, me, G, nb, pb[cur]);
    } else {
      // k = 0: nothing to project, so B's (rt0, q), (q, q) come straight from
      // the registers holding q -- phase B and its barrier disappear
#pragma unroll
      for (int bi = 0; bi < kMaxOwn; ++bi) {
        if (bi >= nown) break;
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          const int64_t i = owned_elem<kE>(me + bi * G, e);
          if (i < n) {
            const double vi = qreg[bi][e];
            acc[0] = __fma_rn(rt0[i], vi, acc[0]);   // (rt0, q)
            acc[1] = __fma_rn(vi, vi, acc[1]);       // (q, q)
          }
        }
        warp_stage<2>(acc, wred, bi, kV2MaxK - 1);
      }
      __syncthreads();
      cta_stage(wred, nown, 2, kV2MaxK - 1, 0, me, G, nb, pb[cur]);
    }
    KRB_STAMP(7);
    grid.sync();
    KRB_STAMP(8);
    if (k > 0) {
      tdot_finals<false>(nb, k, pb[cur], zeta);
      __syncthreads();
      cur ^= 1;
      KRB_STAMP(1);
      // ---- B: q' -= C zeta; (rt0, q'), (q', q') -> alpha
      correct_warps<kE, false>(stage, Cm, ld, n, k, ncg, me, G, nown, qreg, sreg, zeta, qn,
                               rt0, wred, pol);
      prologue<kE, true>(stage, Chat, ld, n, k, ncg, me, G, Tt, pol);
      __syncthreads();
      cta_stage(wred, nown, 2, kV2MaxK - 1, 0, me, G, nb, pb[cur]);
      KRB_STAMP(12);
      grid.sync();
      KRB_STAMP(13);
    }
    local_finals<2>(a, pb[cur], dfin);
    cur ^= 1;
    if (threadIdx.x == 0) finalize<PH_PROJ_Q>(a, &L, dfin, writer);
    __syncthreads();
    KRB_STAMP(2);
    if (L.status != KRB_RUNNING) break;
    const double alpha = L.alpha;
    // ---- C: s = r - alpha q'; (s, s); t = A s; Chat^T t partials
    {
      const double *__restrict__ r_ = r;
      const double *qn_ = qn;
      auto sf = [=](int c) { return __dsub_rn(r_[c], __dmul_rn(alpha, qn_[c])); };
#pragma unroll
      for (int bi = 0; bi < kMaxOwn; ++bi) {
        if (bi >= nown) break;
        double acc[2] = {0.0, 0.0}, acc2[2] = {0.0, 0.0};
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          sreg[bi][e] = treg[bi][e] = 0.0;
          const int64_t i = owned_elem<kE>(me + bi * G, e);
          if (i < n) {
            const double sv = __dsub_rn(r[i], __dmul_rn(alpha, qreg[bi][e]));  // :313
            s[i] = sv;
            sreg[bi][e] = sv;
            acc[0] = __fma_rn(sv, sv, acc[0]);
            const double tv = spmv_row_f<kSell, 4, true>(i, A, sf, polm);
            tv_[i] = tv;
            treg[bi][e] = tv;
            if (k == 0) {   // D's dots, straight from registers
              acc2[0] = __fma_rn(tv, tv, acc2[0]);   // (t, t)
              acc2[1] = __fma_rn(tv, sv, acc2[1]);   // (t, s)
            }
          }
        }
        warp_stage<1>(acc, wred, bi, kV2MaxK);
        if (k == 0) warp_stage<2>(acc2, wred, bi, 0);
        if (k > 0) proj_block<kE>(stage, Chat, ld, n, k, ncg, me, G, nown, bi, treg, wred, pol);
      }
    }
    KRB_STAMP(9);
    if (k > 0) prologue<kE, false>(stage, Cm, ld, n, k, ncg, me, G, Tt, pol);
    __syncthreads();
    cta_stage(wred, nown, 1, kV2MaxK, k, me, G, nb, pb[cur]);   // (s, s) -> row k
    if (k > 0) cta_stage(wred, nown, k, 0, 0, me, G, nb, pb[cur]);
    else cta_stage(wred, nown, 2, 0, 1, me, G, nb, pb[cur]);      // (t,t), (t,s) -> rows 1, 2
    KRB_STAMP(10);
    grid.sync();
    KRB_STAMP(11);
    {
      // gamma columns on warps 0..k-1, ||s|| on warp 31 (after its column
      // when k == 32): both L2 round trips in parallel
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (warp < k) {
        double v = warp_final_volatile(pb[cur] + (int64_t)warp * nb, nb);
        if (lane == 0) gamma[warp] = v;
      }
      if (k == 0 && warp < 2) {
        double v = warp_final_volatile(pb[cur] + (int64_t)(1 + warp) * nb, nb);
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
    KRB_STAMP(3);
    if (L.status != KRB_RUNNING) {
      // solvers.py:315-325: x += alpha p, xc += alpha zeta
#pragma unroll
      for (int bi = 0; bi < kMaxOwn; ++bi)
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          const int64_t i = owned_elem<kE>(me + bi * G, e);
          if (bi < nown && i < n) x[i] = __dadd_rn(x[i], __dmul_rn(alpha, preg[bi][e]));
        }
      for (int j = threadIdx.x; j < k; j += blockDim.x)
        xc[j] = __dadd_rn(xc[j], __dmul_rn(alpha, zeta[j]));
      __syncthreads();
      break;
    }
    // ---- D: t -= C gamma; (t, t), (t, s) -> omega   (k = 0: dots done in C)
    if (k > 0) {
      correct_warps<kE, true>(stage, Cm, ld, n, k, ncg, me, G, nown, treg, sreg, gamma, tv_,
                              rt0, wred, pol);
      prologue<kE, true>(stage, Chat, ld, n, k, ncg, me, G, Tt, pol);  // next A
      __syncthreads();
      cta_stage(wred, nown, 2, kV2MaxK - 1, 0, me, G, nb, pb[cur]);
      grid.sync();
      local_finals<2>(a, pb[cur], dfin);
      cur ^= 1;
      if (threadIdx.x == 0) finalize<PH_PROJ_T>(a, &L, dfin, writer);
    } else if (threadIdx.x == 0) {
      finalize<PH_PROJ_T>(a, &L, dfin + 1, writer);
    }
    __syncthreads();
    KRB_STAMP(4);
    if (L.status != KRB_RUNNING) break;
    const double omega = L.omega;
    // ---- E: x += alpha p' + omega s; r = s - omega t; (r, r), (rt0, r)
#pragma unroll
    for (int bi = 0; bi < kMaxOwn; ++bi) {
      if (bi >= nown) break;
      double acc[2] = {0.0, 0.0};
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        const int64_t i = owned_elem<kE>(me + bi * G, e);
        if (i < n) {
          const double sv = sreg[bi][e];
          x[i] = __dadd_rn(__dadd_rn(x[i], __dmul_rn(alpha, preg[bi][e])),
                           __dmul_rn(omega, sv));                      // :338
          const double rv = __dsub_rn(sv, __dmul_rn(omega, treg[bi][e]));  // :341
          r[i] = rv;
          acc[0] = __fma_rn(rv, rv, acc[0]);
          acc[1] = __fma_rn(rt0[i], rv, acc[1]);
        }
      }
      warp_stage<2>(acc, wred, bi, kV2MaxK - 1);
    }
    for (int j = threadIdx.x; j < k; j += blockDim.x)   // solvers.py:340
      xc[j] = __dadd_rn(__dadd_rn(xc[j], __dmul_rn(alpha, zeta[j])),
                        __dmul_rn(omega, gamma[j]));
    __syncthreads();
    cta_stage(wred, nown, 2, kV2MaxK - 1, 0, me, G, nb, pb[cur]);
    grid.sync();
    local_finals<2>(a, pb[cur], dfin);
    cur ^= 1;
    KRB_STAMP(5);
    if (threadIdx.x == 0) finalize<PH_XR>(a, &L, dfin, writer);
    __syncthreads();
    double *tp = po; po = pn; pn = tp;
    double *tq = qo; qo = qn; qn = tq;
  }
#undef KRB_STAMP
  cp_async_wait<0>();   // speculative prologue of an iteration that never ran
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
static int persist2_launch(const IterArgs *d, int64_t nb, cudaStream_t st) {
  static int grid = 0;
  if (grid == 0) {
    KRB_CHECK_CUDA(cudaFuncSetAttribute(k_persist2<kE, kSell>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kStageBytes));
    int per_sm = 0;
    KRB_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, k_persist2<kE, kSell>, 1024, kStageBytes));
    int dev = 0, sms = kNumSMs;
    KRB_CHECK_CUDA(cudaGetDevice(&dev));
    KRB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = (per_sm > 0 ? 1 : 0) * sms;
    if (grid == 0) {
      set_error("fused persistent kernel does not fit on an SM");
      return KRB_ECUDA;
    }
  }
  if ((int64_t)grid * kMaxOwn < nb) {
    set_error("fused persistent kernel: %lld blocks > %d x %d CTAs", (long long)nb, kMaxOwn, grid);
    return KRB_EINVAL;
  }
  // small systems: one CTA per canonical block (fewer CTAs make every grid
  // barrier and final-stage read cheaper; idle CTAs would only add arrivals)
  const int g = nb < grid ? (int)(nb > 0 ? nb : 1) : grid;
  void *args[] = {(void *)&d};
  KRB_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)k_persist2<kE, kSell>,
                                             dim3(g), dim3(1024), args, kStageBytes, st));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

static bool persist2_eligible(const IterArgs &h) {
  return h.A.perm == nullptr && h.k <= kV2MaxK;
}

bool cluster_eligible(const IterArgs &h);
int cluster_launch(const IterArgs &h, const IterArgs *d, cudaStream_t st);
bool persist0_eligible(const IterArgs &h);
int persist0_launch(const IterArgs &h, const IterArgs *d, cudaStream_t st);

int launch_persistent(const IterArgs &h, const IterArgs *d, cudaStream_t st, int *driver) {
  *driver = KRB_DRIVER_PERSISTENT;
  if (h.n == 0) return KRB_OK;
  const bool sell = h.A.format == 2;
  // tiny systems: one thread-block cluster, everything on chip (cluster.cu);
  // KRB_EINVAL = clusters of this size unavailable -> grid-wide kernel
  if (cluster_eligible(h)) {
    const int rc = cluster_launch(h, d, st);
    if (rc != KRB_EINVAL) {
      *driver = KRB_DRIVER_CLUSTER;
      return rc;
    }
  }
  // k = 0, canon_E == 1: the fused kernel with the operator on chip
  // (persist0.cu; tuning "persist0" = 0 disables)
  if (persist0_eligible(h)) {
    *driver = KRB_DRIVER_FUSED;
    return persist0_launch(h, d, st);
  }
  // fused v2 unless the rows are sigma-permuted (tuning "persist_v1" forces v1)
  const bool v2 = persist2_eligible(h) && !tuning().persist_v1;
  if (v2) {
    *driver = KRB_DRIVER_FUSED;
    switch (canon_E(h.n)) {
      case 1: return sell ? persist2_launch<1, true>(d, h.nb, st) : persist2_launch<1, false>(d, h.nb, st);
      case 2: return sell ? persist2_launch<2, true>(d, h.nb, st) : persist2_launch<2, false>(d, h.nb, st);
      default: break;
    }
    *driver = KRB_DRIVER_PERSISTENT;
  }
  // small systems only (E <= 2, n <= 606208): larger ones run the graph
  switch (canon_E(h.n)) {
    case 1: return sell ? persist_launch<1, true>(d, st) : persist_launch<1, false>(d, st);
    case 2: return sell ? persist_launch<2, true>(d, st) : persist_launch<2, false>(d, st);
    default:
      set_error("persistent driver supports n <= %d (canon_E <= 2)", 2 * kLanes * kTargetBlocks);
      return KRB_EINVAL;
  }
}


}  // namespace krb
