// Deflated BiCGSTAB (Algorithm 2 of arXiv 1406.2831) on sm_100a.
//
// Restates rbicgstab_solve (reference solvers.py:245-361; bicgstab_solve
// solvers.py:156-242 is the k = 0 case) as a chain of fused, HBM-streaming
// phases.  All scalar logic (alpha, omega, beta, rho, breakdown and
// convergence predicates, history records) runs on the device, in the
// reference's order, in the one CTA that finishes a phase's reduction last.
//
// Two drivers share the phase bodies below:
//  * persistent (default): ONE cooperative kernel runs the whole solve; the
//    phases are separated by grid barriers whose last-arriving CTA ("leader")
//    does the phase's final reduction and scalar logic before releasing the
//    others -- no kernel launches and no host round trips per iteration;
//  * graph: each phase is its own kernel, the iteration is captured once into
//    a CUDA graph whose WHILE conditional node is re-armed by the device
//    (cudaGraphSetConditional) until the status leaves RUNNING;
//  * host loop (debug / per-kernel profiling).
// Every per-solve pointer lives in a device descriptor, so the graph and the
// persistent kernel serve every solve of the same shape.
//
// Per iteration (k > 0; Z vanishes and Q/T skip the update for k = 0):
//   P  p = r + beta (p - omega q)                      3 read, 1 write
//   M  q = A p                                         SpMV
//   Z  zeta = Chat^T q  (block x column-group units)   n x k + n read
//   Q  q -= C zeta ; (rt0,q), (q,q) -> den, alpha       n x k + 2 read, 1 write
//   S  s = r - alpha q ; (s,s) -> half-step exit        2 read, 1 write
//   M  t = A s ;  Z gamma = Chat^T t
//   T  t -= C gamma ; (t,t), (t,s) -> omega             n x k + 2 read, 1 write
//   X  x = x + alpha p + omega s ; r = s - omega t ;
//      (r,r), (rt0,r) -> record, converge, rho, beta    5 read, 2 write
//      (on a half-step exit instead: x += alpha p, xc += alpha zeta)
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "ctx.cuh"
#include "spmv.cuh"
#include "tdot.cuh"

namespace krb {

namespace cg = cooperative_groups;

enum Phase {
  PH_PUPDATE = 0,
  PH_PROJ_Q,
  PH_SUPD,
  PH_PROJ_T,
  PH_XR,
  PH_BNORM,
  PH_INIT,
  PH_TRUE,
  PH_RINIT,
};

struct IterArgs {
  krb_matrix A;  // copy of the matrix handle (device pointers)
  int64_t n, nb, ld;
  int k;
  int use_cond;
  cudaGraphConditionalHandle cond;
  const double *C, *Chat, *U;
  double *x, *r, *p, *q, *s, *t, *rt0, *b;
  double *zeta, *gamma, *xc;
  double *part, *part2;   // part2: second partial buffer (persistent kernel)
  uint64_t *prof;         // optional per-phase %globaltimer stamps (16/iter)
  int64_t prof_cap;
  unsigned int *counters;
  SolveScalars *S;
  double *hist_r;
  int64_t *hist_m;
  uint64_t *hist_t;
};

struct GridSync {
  unsigned int count;
  unsigned int gen;
};

// S: the scalar block to update (global, or a CTA's shared copy in the
// persistent kernel); only the writer CTA stores the history entries.
__device__ __forceinline__ void record(const IterArgs &a, SolveScalars *S,
                                       double rn, bool writer) {
  int64_t h = S->hist_len;
  if (writer) {
    a.hist_r[h] = rn;
    a.hist_m[h] = S->matvecs;
    a.hist_t[h] = globaltimer();
  }
  S->hist_len = h + 1;
}

__host__ __device__ constexpr int ndots_of(int PH) {
  return PH == PH_PROJ_Q ? 2 : PH == PH_SUPD ? 1 : PH == PH_PROJ_T ? 2
       : PH == PH_XR ? 2 : PH == PH_BNORM ? 1 : PH == PH_INIT ? 3
       : PH == PH_TRUE ? 2 : 0;
}

// Scalar logic of each phase, executed by thread 0 of the finishing CTA once
// the dot products d[] are final.  Mirrors solvers.py:288-356 line by line.
template <int PH>
__device__ __noinline__ void finalize(const IterArgs &a, SolveScalars *S, const double *d,
                                     bool writer = true) {
  if (PH == PH_BNORM) {
    S->bnorm = __dsqrt_rn(d[0]);
    S->tol_abs = __dmul_rn(S->tol_abs, S->bnorm);  // tol_abs held tol
  } else if (PH == PH_INIT) {
    double rn = __dsqrt_rn(d[0]);
    record(a, S, rn, writer);
    S->rnorm = rn;
    S->rho = d[1];
    S->nrt0 = __dsqrt_rn(d[2]);
    S->beta = 0.0;
    S->omega = 0.0;
    if (rn <= S->tol_abs)
      S->status = KRB_CONVERGED;
    else if (S->max_itn <= 0)
      S->status = KRB_MAX_ITN;
  } else if (PH == PH_PROJ_Q) {
    S->matvecs += 1;
    double den = d[0];
    double nq = __dsqrt_rn(d[1]);
    S->den = den;
    S->qnorm = nq;
    if (fabs(den) <= __dmul_rn(__dmul_rn(S->breakdown_tol, S->nrt0), nq))
      S->status = KRB_BREAKDOWN_SERIOUS;
    else
      S->alpha = __ddiv_rn(S->rho, den);
  } else if (PH == PH_SUPD) {
    double sn = __dsqrt_rn(d[0]);
    S->snorm = sn;
    if (sn <= S->tol_abs) {
      record(a, S, sn, writer);
      S->early = 1;
      S->status = KRB_CONVERGED;
    }
  } else if (PH == PH_PROJ_T) {
    S->matvecs += 1;
    double tt = d[0];
    S->tt = tt;
    S->ts = d[1];
    if (tt == 0.0) {
      S->status = KRB_BREAKDOWN_OMEGA;
    } else {
      double om = __ddiv_rn(d[1], tt);
      if (om == 0.0)
        S->status = KRB_BREAKDOWN_OMEGA;
      else
        S->omega = om;
    }
  } else if (PH == PH_XR) {
    double rn = __dsqrt_rn(d[0]);
    S->rnorm = rn;
    record(a, S, rn, writer);
    S->itn += 1;
    if (rn <= S->tol_abs) {
      S->status = KRB_CONVERGED;
    } else {
      double rho_new = d[1];
      if (fabs(rho_new) <= __dmul_rn(__dmul_rn(S->breakdown_tol, S->nrt0), rn)) {
        S->status = KRB_BREAKDOWN_SERIOUS;
      } else {
        S->beta = __dmul_rn(__ddiv_rn(rho_new, S->rho), __ddiv_rn(S->alpha, S->omega));
        S->rho = rho_new;
      }
    }
    if (S->status == KRB_RUNNING && S->itn >= S->max_itn) S->status = KRB_MAX_ITN;
  } else if (PH == PH_TRUE) {
    double bn = __dsqrt_rn(d[1]);
    S->final_true_resid = __ddiv_rn(__dsqrt_rn(d[0]), bn > 0.0 ? bn : 1.0);
  }
}

struct PhaseScal {
  double alpha, omega, beta;
};

__device__ __forceinline__ PhaseScal load_scal(const SolveScalars *S) {
  return PhaseScal{S->alpha, S->omega, S->beta};
}

// Elementwise work + canonical block partials of one phase for canonical
// blocks blk = first, first + step, ...   `coef` (k values of zeta / gamma)
// must already be in shared memory for the projection phases.
template <int kE, int PH>
__device__ __forceinline__ void phase_blocks(const IterArgs &a, const PhaseScal sc,
                                             double (*red)[32],
                                             const double *coef, int64_t first,
                                             int64_t step, double *part_buf) {
  constexpr int ND = ndots_of(PH);
  const double alpha = sc.alpha, omega = sc.omega, beta = sc.beta;
  const int k = a.k;
  const int64_t n = a.n, nb = a.nb, ld = a.ld;
  double *__restrict__ x = a.x;
  double *__restrict__ r = a.r;
  double *__restrict__ p = a.p;
  double *__restrict__ q = a.q;
  double *__restrict__ s = a.s;
  double *__restrict__ t = a.t;
  const double *__restrict__ rt0 = a.rt0;
  const double *__restrict__ bvec = a.b;
  const double *__restrict__ Cm = a.C;
  double *__restrict__ part = part_buf;
  for (int64_t blk = first; blk < nb; blk += step) {
    const int64_t base = blk * ((int64_t)kLanes * kE) + threadIdx.x;
    double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll(kE < 4 ? kE : 4)
    for (int e = 0; e < kE; ++e) {
      const int64_t i = base + (int64_t)kLanes * e;
      if (i >= n) continue;
      if (PH == PH_PUPDATE) {
        // p = r + beta * (p - omega * q)          (solvers.py:303)
        double pv = __dsub_rn(p[i], __dmul_rn(omega, q[i]));
        p[i] = __dadd_rn(r[i], __dmul_rn(beta, pv));
      } else if (PH == PH_PROJ_Q || PH == PH_PROJ_T) {
        double *v = PH == PH_PROJ_Q ? q : t;
        double vi = v[i];
        if (k > 0) {
          // C @ zeta for this element: sequential fma over the columns, four
          // independent column loads in flight per step
          double cz = 0.0;
          int j = 0;
          for (; j + 4 <= k; j += 4) {
            double c0 = __ldg(Cm + (int64_t)j * ld + i);
            double c1 = __ldg(Cm + (int64_t)(j + 1) * ld + i);
            double c2 = __ldg(Cm + (int64_t)(j + 2) * ld + i);
            double c3 = __ldg(Cm + (int64_t)(j + 3) * ld + i);
            cz = __fma_rn(c0, coef[j], cz);
            cz = __fma_rn(c1, coef[j + 1], cz);
            cz = __fma_rn(c2, coef[j + 2], cz);
            cz = __fma_rn(c3, coef[j + 3], cz);
          }
          for (; j < k; ++j) cz = __fma_rn(__ldg(Cm + (int64_t)j * ld + i), coef[j], cz);
          vi = __dsub_rn(vi, cz);   // q - C @ zeta   (solvers.py:307,329)
          v[i] = vi;
        }
        if (PH == PH_PROJ_Q) {
          acc[0] = __fma_rn(rt0[i], vi, acc[0]);   // (rt0, q)
          acc[1] = __fma_rn(vi, vi, acc[1]);       // (q, q)
        } else {
          acc[0] = __fma_rn(vi, vi, acc[0]);       // (t, t)
          acc[1] = __fma_rn(vi, s[i], acc[1]);     // (t, s)
        }
      } else if (PH == PH_SUPD) {
        // s = r - alpha * q                       (solvers.py:313)
        double sv = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
        s[i] = sv;
        acc[0] = __fma_rn(sv, sv, acc[0]);
      } else if (PH == PH_XR) {
        // x = x + alpha*p + omega*s ; r = s - omega*t   (solvers.py:338,341)
        double sv = s[i];
        x[i] = __dadd_rn(__dadd_rn(x[i], __dmul_rn(alpha, p[i])),
                         __dmul_rn(omega, sv));
        double rv = __dsub_rn(sv, __dmul_rn(omega, t[i]));
        r[i] = rv;
        acc[0] = __fma_rn(rv, rv, acc[0]);
        acc[1] = __fma_rn(rt0[i], rv, acc[1]);
      } else if (PH == PH_BNORM) {
        double bv = bvec[i];
        acc[0] = __fma_rn(bv, bv, acc[0]);
      } else if (PH == PH_INIT) {
        double rv = r[i], tv = rt0[i];
        acc[0] = __fma_rn(rv, rv, acc[0]);
        acc[1] = __fma_rn(tv, rv, acc[1]);
        acc[2] = __fma_rn(tv, tv, acc[2]);
      } else if (PH == PH_TRUE) {
        // true residual b - A x_out   (solvers.py:147-153); A x_out in t
        double bv = bvec[i];
        double res = __dsub_rn(bv, t[i]);
        acc[0] = __fma_rn(res, res, acc[0]);
        acc[1] = __fma_rn(bv, bv, acc[1]);
      } else if (PH == PH_RINIT) {
        // r = b - A x_init            (recycling.py:200); A x_init in t
        r[i] = __dsub_rn(bvec[i], t[i]);
      }
    }
    if (ND > 0) {
      double bp = block_tree_multi<ND == 0 ? 1 : ND>(acc, red);
      const int warp = threadIdx.x >> 5;
      if (warp < ND && (threadIdx.x & 31) == 0) part[warp * nb + blk] = bp;
    }
  }
}

// Final stage + scalar logic of a phase, run by every thread of the one CTA
// that finished the phase last (all partials visible).
template <int PH>
__device__ __forceinline__ void phase_leader(const IterArgs &a, const PhaseScal sc) {
  constexpr int ND = ndots_of(PH);
  __shared__ double dfin[3];
  const int warp = threadIdx.x >> 5;
  if (warp < ND) {
    double v = warp_final_volatile(a.part + warp * a.nb, a.nb);
    if ((threadIdx.x & 31) == 0) dfin[warp] = v;
  }
  if (PH == PH_XR) {
    // xc = xc + alpha*zeta + omega*gamma     (solvers.py:340)
    for (int j = threadIdx.x; j < a.k; j += blockDim.x)
      a.xc[j] = __dadd_rn(__dadd_rn(a.xc[j], __dmul_rn(sc.alpha, a.zeta[j])),
                          __dmul_rn(sc.omega, a.gamma[j]));
  }
  __syncthreads();
  if (threadIdx.x == 0) finalize<PH>(a, a.S, dfin);
  __syncthreads();
}

// half-step exit (solvers.py:315-325): x += alpha p, xc += alpha zeta
__device__ __forceinline__ void half_exit_update(const IterArgs &a, double alpha,
                                                 int64_t first, int64_t step) {
  for (int64_t i = first * blockDim.x + threadIdx.x; i < a.n; i += step * blockDim.x)
    a.x[i] = __dadd_rn(a.x[i], __dmul_rn(alpha, a.p[i]));   // solvers.py:316
  if (first == 0)
    for (int j = threadIdx.x; j < a.k; j += blockDim.x)     // solvers.py:318
      a.xc[j] = __dadd_rn(a.xc[j], __dmul_rn(alpha, a.zeta[j]));
}

// ---------------------------------------------------------------------------
// graph / host-loop driver: one kernel per phase, last CTA finalizes
// ---------------------------------------------------------------------------
template <int kE, int PH>
__global__ void __launch_bounds__(1024) k_phase(const IterArgs *__restrict__ pa) {
  __shared__ double coef[512];
  __shared__ double red[4][32];
  __shared__ int last_flag;
  const IterArgs &a = *pa;
  SolveScalars *S = a.S;
  constexpr int ND = ndots_of(PH);
  constexpr bool kGated = (PH == PH_PUPDATE || PH == PH_PROJ_Q ||
                           PH == PH_SUPD || PH == PH_PROJ_T || PH == PH_XR);
  if (PH == PH_XR && blockIdx.x == 0 && threadIdx.x == 0) S->bodies += 1;
  const PhaseScal sc = load_scal(S);
  if (kGated && S->status != KRB_RUNNING) {
    if (PH == PH_PUPDATE) {
      // a half-step exit was applied by the previous X phase: mark consumed
      // (only matters for the host-driven loop, which may overshoot)
      if (blockIdx.x == 0 && threadIdx.x == 0 && S->early == 1) S->early = 2;
      return;
    }
    if (PH == PH_XR && S->early == 1) {
      half_exit_update(a, sc.alpha, blockIdx.x, gridDim.x);
      if (blockIdx.x == 0 && threadIdx.x == 0 && a.use_cond) cudaGraphSetConditional(a.cond, 0);
      return;
    }
    if (PH == PH_XR && a.use_cond && blockIdx.x == 0 && threadIdx.x == 0)
      cudaGraphSetConditional(a.cond, 0);
    return;
  }
  if (PH == PH_PROJ_Q || PH == PH_PROJ_T) {
    const double *src = PH == PH_PROJ_Q ? a.zeta : a.gamma;
    for (int j = threadIdx.x; j < a.k; j += blockDim.x) coef[j] = src[j];
    __syncthreads();
  }
  phase_blocks<kE, PH>(a, sc, red, coef, blockIdx.x, gridDim.x, a.part);
  if (ND == 0) return;
  if (!elect_last_cta(a.counters + PH, &last_flag)) return;
  phase_leader<PH>(a, sc);
  if (threadIdx.x == 0) {
    a.counters[PH] = 0;
    if (PH == PH_XR && a.use_cond)
      cudaGraphSetConditional(a.cond, S->status == KRB_RUNNING ? 1u : 0u);
  }
}

// projection dots inside the iteration: Chat^T v -> zeta / gamma
template <int kE, bool kGamma>
__global__ void __launch_bounds__(1024) k_proj_dot(const IterArgs *__restrict__ pa) {
  const IterArgs &a = *pa;
  if (a.S->status != KRB_RUNNING) return;
  tdot_body<kE, false>(a.n, a.nb, a.k, a.Chat, a.ld, kGamma ? a.t : a.q, a.part,
                       kGamma ? a.gamma : a.zeta, a.counters + kCounterTdotGraph);
}

// SpMV inside the iteration (matrix read from the descriptor)
template <bool kSell, bool kSecond>
__global__ void __launch_bounds__(256) k_iter_spmv(const IterArgs *__restrict__ pa) {
  const IterArgs &a = *pa;
  if (a.S->status != KRB_RUNNING) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.A.n) return;
  const double *x = kSecond ? a.s : a.p;
  double *y = kSecond ? a.t : a.q;
  y[(kSell && a.A.perm) ? a.A.perm[i] : i] = spmv_row<kSell>(i, a.A, x);
}

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
                             (int)(u / nb) * kTdotCG, red);
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
                             (int)(u / nb) * kTdotCG, red);
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

__global__ void k_init_scalars(SolveScalars *S, double tol, double btol,
                               int64_t max_itn, int k, int64_t mv0) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    SolveScalars z = {};
    z.tol_abs = tol;
    z.breakdown_tol = btol;
    z.max_itn = max_itn;
    z.k = k;
    z.matvecs = mv0;
    z.t_start = globaltimer();
    *S = z;
  }
}

#define KRB_TRY(x)          \
  do {                      \
    int rc_ = (x);          \
    if (rc_) return rc_;    \
  } while (0)

template <int PH>
static int launch_phase(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  if (h.nb == 0) return KRB_OK;
  int grid = grid_for(h.nb);
  KRB_DISPATCH_E(canon_E(h.n), (k_phase<kE, PH><<<grid, 1024, 0, st>>>(d)));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

template <bool kGamma>
static int launch_proj_dot(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  if (h.k <= 0 || h.nb == 0) return KRB_OK;
  dim3 grid = tdot_grid(h.nb, h.k);
  KRB_DISPATCH_E(canon_E(h.n), (k_proj_dot<kE, kGamma><<<grid, 1024, 0, st>>>(d)));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

template <bool kSecond>
static int launch_iter_spmv(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  if (h.n == 0) return KRB_OK;
  unsigned blocks = (unsigned)((h.n + 255) / 256);
  if (h.A.format == 2)
    k_iter_spmv<true, kSecond><<<blocks, 256, 0, st>>>(d);
  else
    k_iter_spmv<false, kSecond><<<blocks, 256, 0, st>>>(d);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

// one iteration (the graph body)
static int launch_iteration(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  KRB_TRY(launch_phase<PH_PUPDATE>(h, d, st));
  KRB_TRY(launch_iter_spmv<false>(h, d, st));
  KRB_TRY(launch_proj_dot<false>(h, d, st));
  KRB_TRY(launch_phase<PH_PROJ_Q>(h, d, st));
  KRB_TRY(launch_phase<PH_SUPD>(h, d, st));
  KRB_TRY(launch_iter_spmv<true>(h, d, st));
  KRB_TRY(launch_proj_dot<true>(h, d, st));
  KRB_TRY(launch_phase<PH_PROJ_T>(h, d, st));
  KRB_TRY(launch_phase<PH_XR>(h, d, st));
  return KRB_OK;
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

static int launch_persistent(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  if (h.n == 0) return KRB_OK;
  const bool sell = h.A.format == 2;
  // small systems only (E <= 2, n <= 606208): larger ones run the graph
  switch (canon_E(h.n)) {
    case 1: return sell ? persist_launch<1, true>(d, st) : persist_launch<1, false>(d, st);
    case 2: return sell ? persist_launch<2, true>(d, st) : persist_launch<2, false>(d, st);
    default:
      set_error("persistent driver supports n <= %d (canon_E <= 2)", 2 * kLanes * kTargetBlocks);
      return KRB_EINVAL;
  }
}

int ctx_reserve_vectors(krb_context *ctx, int64_t n, int64_t k) {
  if (n <= ctx->vec_n && k <= ctx->vec_k && ctx->desc) return KRB_OK;
  double **vecs[] = {&ctx->x, &ctx->r, &ctx->p, &ctx->q, &ctx->s,
                     &ctx->t, &ctx->rt0, &ctx->b, &ctx->w};
  int64_t nn = n > ctx->vec_n ? n : ctx->vec_n;
  int64_t kk = k > ctx->vec_k ? k : ctx->vec_k;
  for (double **v : vecs) {
    if (*v) cudaFree(*v);
    *v = nullptr;
    KRB_CHECK_CUDA(cudaMalloc(v, sizeof(double) * (nn > 0 ? nn : 1)));
  }
  if (ctx->kbuf) cudaFree(ctx->kbuf);
  KRB_CHECK_CUDA(cudaMalloc(&ctx->kbuf, sizeof(double) * 5 * (kk > 0 ? kk : 1)));
  if (!ctx->desc) KRB_CHECK_CUDA(cudaMalloc(&ctx->desc, sizeof(IterArgs)));
  if (!ctx->S) KRB_CHECK_CUDA(cudaMalloc(&ctx->S, sizeof(SolveScalars)));
  ctx->vec_n = nn;
  ctx->vec_k = kk;
  ctx->graph.reset();
  return KRB_OK;
}

static int build_graph(krb_context *ctx, const IterArgs &h, const IterArgs *d,
                       cudaStream_t capture) {
  GraphCache &G = ctx->graph;
  G.reset();
  cudaGraph_t g;
  KRB_CHECK_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hc;
  KRB_CHECK_CUDA(cudaGraphConditionalHandleCreate(&hc, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = hc;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  KRB_CHECK_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  KRB_CHECK_CUDA(cudaStreamBeginCaptureToGraph(capture, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeRelaxed));
  const int64_t c0 = launch_counter();
  int rc = launch_iteration(h, d, capture);
  G.kernels_per_body = launch_counter() - c0;
  launch_counter() = c0;  // captured, not executed: counted per body run
  cudaGraph_t out_body;
  cudaError_t e = cudaStreamEndCapture(capture, &out_body);
  if (rc) {
    cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    set_error("graph capture: %s", cudaGetErrorString(e));
    return KRB_ECUDA;
  }
  cudaGraphExec_t exec;
  e = cudaGraphInstantiate(&exec, g, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    set_error("graph instantiate: %s", cudaGetErrorString(e));
    return KRB_ECUDA;
  }
  G.graph = g;
  G.exec = exec;
  G.cond = hc;
  return KRB_OK;
}

static cudaStream_t capture_stream() {
  static thread_local cudaStream_t s = nullptr;
  if (!s) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  return s;
}

int rbicgstab(krb_context *ctx, const krb_matrix *A, const double *d_b,
              const double *d_x_init, const krb_space_view *R,
              const krb_solve_config *cfg, double *d_x_out, double *hist_r,
              int64_t *hist_m, uint64_t *hist_t, krb_solve_result *res,
              cudaStream_t st) {
  KRB_REQUIRE(ctx && A && d_b && cfg && d_x_out && hist_r && hist_m && hist_t && res,
              "krb_rbicgstab: NULL argument");
  const int64_t n = A->n;
  const int64_t k = (R && R->k > 0) ? R->k : 0;
  if (k > 0) {
    KRB_REQUIRE(R->n == n, "recycle space dimension does not match the operator");
    KRB_REQUIRE(R->ld >= n, "recycle space leading dimension < n");
    KRB_REQUIRE(R->U && R->C && R->Ct && R->Chat && R->Ccheck,
                "recycle space view has NULL blocks");
    KRB_REQUIRE(k <= 512, "recycle dimension > 512 unsupported");
  }
  KRB_TRY(ctx_reserve_vectors(ctx, n, k));
  KRB_TRY(ctx_reserve_counters(ctx, st));
  const int64_t l0 = launch_counter();
  int64_t per_body = 0;
  const int64_t nb = canon_nblocks(n);
  const size_t part_one = (size_t)(3 * nb > k * nb ? 3 * nb : k * nb) + 64;
  KRB_TRY(ctx_reserve_part(ctx, 2 * part_one));
  IterArgs h = {};
  h.A = *A;
  h.A.T = nullptr;
  h.n = n;
  h.nb = nb;
  h.k = (int)k;
  h.ld = k > 0 ? R->ld : n;
  h.C = k > 0 ? R->C : nullptr;
  h.Chat = k > 0 ? R->Chat : nullptr;
  h.U = k > 0 ? R->U : nullptr;
  h.x = ctx->x; h.r = ctx->r; h.p = ctx->p; h.q = ctx->q; h.s = ctx->s;
  h.t = ctx->t; h.rt0 = ctx->rt0; h.b = ctx->b;
  h.zeta = ctx->kbuf;
  h.gamma = ctx->kbuf + ctx->vec_k;
  h.xc = ctx->kbuf + 2 * ctx->vec_k;
  double *ybuf = ctx->kbuf + 3 * ctx->vec_k;
  h.part = ctx->part;
  h.part2 = ctx->part + part_one;
  h.counters = ctx->counters;
  h.S = ctx->S;
  h.hist_r = hist_r;
  h.hist_m = hist_m;
  h.hist_t = hist_t;
  h.prof = cfg->d_phase_stamps;
  h.prof_cap = cfg->d_phase_stamps ? cfg->phase_stamps_cap : 0;
  const int mode = cfg->use_graph;   // 0 host loop, 1 graph, 2 persistent
  const bool graph = mode == 1;
  GraphCache &G = ctx->graph;
  const bool hit = graph && G.exec && G.n == n && G.k == k && G.format == A->format;
  h.use_cond = graph ? 1 : 0;
  h.cond = hit ? G.cond : 0;
  IterArgs *d = reinterpret_cast<IterArgs *>(ctx->desc);

  // ---- setup (solvers.py:257-296) -------------------------------------
  if (graph && !hit) {
    KRB_CHECK_CUDA(cudaStreamSynchronize(st));
    KRB_TRY(build_graph(ctx, h, d, capture_stream()));
    G.n = n; G.k = k; G.format = A->format;
    h.cond = G.cond;
  }
  // the descriptor is written in stream order (the previous solve on this
  // stream has finished reading it)
  KRB_CHECK_CUDA(cudaMemcpyAsync(d, &h, sizeof(IterArgs), cudaMemcpyHostToDevice, st));
  KRB_CHECK_CUDA(cudaMemcpyAsync(h.b, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  k_init_scalars<<<1, 1, 0, st>>>(h.S, cfg->tol, cfg->breakdown_tol, cfg->max_itn,
                                  (int)k, d_x_init ? 1 : 0);
  KRB_CHECK_LAUNCH();
  KRB_TRY(launch_phase<PH_BNORM>(h, d, st));
  // shadow residual rt_{-1} (solvers.py:268-269)
  if (cfg->d_shadow)
    KRB_CHECK_CUDA(cudaMemcpyAsync(ctx->w, cfg->d_shadow, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
  else
    KRB_TRY(krb_uniform_pcg64(n, cfg->pcg_state_hi, cfg->pcg_state_lo, cfg->pcg_inc_hi,
                              cfg->pcg_inc_lo, -1.0, 1.0, ctx->w, st));
  // x0, r0 (project_initial, recycling.py:189-206)
  if (d_x_init) {
    KRB_CHECK_CUDA(cudaMemcpyAsync(h.x, d_x_init, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
    KRB_TRY(spmv_launch(A, h.x, h.t, nullptr, st));
    KRB_TRY(launch_phase<PH_RINIT>(h, d, st));
  } else {
    KRB_CHECK_CUDA(cudaMemsetAsync(h.x, 0, sizeof(double) * n, st));
    KRB_CHECK_CUDA(cudaMemcpyAsync(h.r, h.b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
  if (k > 0) {
    KRB_TRY(launch_tdot(ctx, n, k, R->Chat, R->ld, h.r, false, ybuf, nullptr, st));
    KRB_TRY(launch_gemv(n, k, R->U, R->ld, ybuf, h.x, +1, h.x, st));
    KRB_TRY(launch_gemv(n, k, R->C, R->ld, ybuf, h.r, -1, h.r, st));
    // rt0 = rt_{-1} - Ct (Ccheck^H rt_{-1})   (solvers.py:273)
    KRB_TRY(launch_tdot(ctx, n, k, R->Ccheck, R->ld, ctx->w, false, ybuf, nullptr, st));
    KRB_TRY(launch_gemv(n, k, R->Ct, R->ld, ybuf, ctx->w, -1, h.rt0, st));
    KRB_CHECK_CUDA(cudaMemsetAsync(h.xc, 0, sizeof(double) * k, st));
  } else {
    KRB_CHECK_CUDA(cudaMemcpyAsync(h.rt0, ctx->w, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
  }
  KRB_CHECK_CUDA(cudaMemsetAsync(h.p, 0, sizeof(double) * n, st));
  KRB_CHECK_CUDA(cudaMemsetAsync(h.q, 0, sizeof(double) * n, st));
  KRB_TRY(launch_phase<PH_INIT>(h, d, st));

  // ---- iterations (solvers.py:298-356) --------------------------------
  if (mode == 2) {
    KRB_TRY(launch_persistent(h, d, st));
  } else if (graph) {
    KRB_CHECK_CUDA(cudaGraphLaunch(G.exec, st));
    per_body = G.kernels_per_body;
  } else {
    // host-driven loop, status polled every 8 iterations (kernels no-op once
    // the status leaves RUNNING, so the overshoot is harmless)
    int32_t status = 0;
    for (int64_t it = 0; it < cfg->max_itn + 1; ++it) {
      KRB_TRY(launch_iteration(h, d, st));
      if ((it & 7) == 7 || it == cfg->max_itn) {
        KRB_CHECK_CUDA(cudaMemcpyAsync(&status, &h.S->status, sizeof(int32_t),
                                       cudaMemcpyDeviceToHost, st));
        KRB_CHECK_CUDA(cudaStreamSynchronize(st));
        if (status != KRB_RUNNING) break;
      }
    }
  }

  // ---- x_out = x - U xc (solvers.py:359), true residual (:360) ----------
  if (k > 0)
    KRB_TRY(launch_gemv(n, k, R->U, R->ld, h.xc, h.x, -1, d_x_out, st));
  else
    KRB_CHECK_CUDA(cudaMemcpyAsync(d_x_out, h.x, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
  KRB_TRY(spmv_launch(A, d_x_out, h.t, nullptr, st));
  KRB_TRY(launch_phase<PH_TRUE>(h, d, st));
  SolveScalars hs;
  KRB_CHECK_CUDA(cudaMemcpyAsync(&hs, h.S, sizeof(SolveScalars), cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  res->status = hs.status;
  res->hist_len = hs.hist_len;
  res->matvecs = hs.matvecs;
  res->rhs_norm = hs.bnorm;
  res->final_true_resid = hs.final_true_resid;
  res->t_start_ns = hs.t_start;
  res->iterations_run = mode == 2 ? hs.itn : hs.bodies;
  launch_counter() += hs.bodies * per_body;
  res->kernel_launches = launch_counter() - l0;
  return KRB_OK;
}

}  // namespace krb

using namespace krb;

extern "C" {

int krb_rbicgstab(krb_context *ctx, const krb_matrix *A, const double *d_b,
                  const double *d_x_init, const krb_space_view *R,
                  const krb_solve_config *cfg, double *d_x_out,
                  double *d_hist_resid, int64_t *d_hist_matvecs,
                  uint64_t *d_hist_stamp, krb_solve_result *h_result,
                  void *stream) {
  return rbicgstab(ctx, A, d_b, d_x_init, R, cfg, d_x_out, d_hist_resid,
                   d_hist_matvecs, d_hist_stamp, h_result, as_stream(stream));
}

int krb_last_scalars(krb_context *ctx, double *h_out) {
  KRB_REQUIRE(ctx && ctx->S, "krb_last_scalars: no solve yet");
  SolveScalars hs;
  KRB_CHECK_CUDA(cudaMemcpy(&hs, ctx->S, sizeof(hs), cudaMemcpyDeviceToHost));
  h_out[0] = hs.alpha;
  h_out[1] = hs.omega;
  h_out[2] = hs.rho;
  h_out[3] = hs.beta;
  return KRB_OK;
}

}  // extern "C"
