// Deflated two-sided BiCG with Lanczos-direction capture (Algorithm 1 of
// arXiv 1406.2831) on sm_100a: rbicg_solve, reference solvers.py:460-638.
//
// Per iteration: p/pt update; q = A p and qt = A^T pt (the transpose is a
// device CSR built once per matrix); projections against (Chat, C) and
// (Ccheck, Ct); den/alpha; x, xt, r, rt updates with ||r||, ||rt|| and
// (rt, r); then the capture of the normalized direction pair
// v = r/||r||, vt = rt/(v, rt) straight into a device ring of s+2 columns.
// The loop is a CUDA graph with a device WHILE node that pauses (returns to
// the host) only when a cycle of s iterations is complete, so the host-side
// recycle-space update (a tiny generalized eigenproblem) can run, or when the
// solve ends.  Scalar logic follows solvers.py:584-631 in order.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "ctx.cuh"
#include "spmv.cuh"
#include "tdot.cuh"

namespace krb {

namespace cg = cooperative_groups;

enum BiPhase {
  BP_PUPDATE = 0,
  BP_PROJ,      // q -= C zeta, qt -= Ct zetat ; (pt,q), (pt,pt), (q,q)
  BP_XR,        // x, xt, r, rt ; (r,r), (rt,rt), (rt,r)
  BP_CAP1,      // v = r / ||r|| into the ring ; (v, rt)
  BP_CAP2,      // vt = rt / sigma into the ring ; emit / loop control
  BP_INIT,      // (r,r), (rt,rt) -> record 0 ; (v, rt) of the first push
  BP_BNORM,     // (b,b), (bt,bt)
  BP_TRUE,      // true residual
  BP_RINIT,     // r = b - A x_init
  BP_RTINIT,    // rt = bt - A^T xt_init
  BP_DUALCHK,   // (rt0, r0), (rt0, rt0), (r0, r0) for the dual start test
};

struct BiScalars {
  double rho, alpha, beta;
  double den, rnorm, rtnorm, rho_new, sigma;
  double bnorm, btnorm, tol, breakdown_tol;
  double dual_rho, dual_rt2, dual_r2;
  double final_true_resid;
  int64_t itn, max_itn, s;
  int64_t n_matvec, n_rmatvec;
  int64_t hist_len;
  int64_t ncols;        // columns currently in the capture ring
  int64_t npush;        // pushes over the whole solve (rhos entries)
  int64_t nalpha;       // alphas/betas recorded (capture on)
  uint64_t t_start;
  int64_t bodies;
  int32_t status;
  int32_t capture;      // capture still on
  int32_t cap_now;      // push attempt this iteration
  int32_t push_ok;
  int32_t emit;         // pause requested: cycle complete
  int32_t xr_done;
  int32_t pbuf;         // persistent k = 0 path: p / pt live in (p2, pt2) when 1
};

struct BiArgs {
  krb_matrix A, AT;
  int64_t n, nb, ld, ring_ld;
  int k;
  int use_cond;
  cudaGraphConditionalHandle cond;
  const double *C, *Chat, *Ct, *Ccheck;
  double *x, *xt, *r, *rt, *p, *pt, *q, *qt, *b, *bt;
  double *p2, *pt2;        // double buffers of the fused persistent k = 0 path
  double *zeta, *zetat, *zc, *ztc;
  double *V, *Vt;          // capture rings (ring_ld stride per column)
  double *rhos, *alphas, *betas;
  double *part, *part2;   // part2: ping-pong buffer of the persistent kernel
  unsigned int *counters;
  BiScalars *S;
  double *hist_r, *hist_rt;
  int64_t *hist_m;
  uint64_t *hist_t;
};

// S: the scalar block to update (global, or a CTA's shared copy in the
// persistent kernel); only the writer CTA stores history / scalar arrays.
__device__ __forceinline__ void bi_record(const BiArgs &a, BiScalars *S, bool writer) {
  int64_t h = S->hist_len;
  if (writer) {
    a.hist_r[h] = S->rnorm;
    a.hist_rt[h] = S->rtnorm;
    a.hist_m[h] = S->n_matvec + S->n_rmatvec;
    a.hist_t[h] = globaltimer();
  }
  S->hist_len = h + 1;
}

__host__ __device__ constexpr int bi_ndots(int PH) {
  return PH == BP_PROJ ? 3 : PH == BP_XR ? 3 : PH == BP_CAP1 ? 1
       : PH == BP_INIT ? 2 : PH == BP_BNORM ? 2 : PH == BP_TRUE ? 2
       : PH == BP_DUALCHK ? 3 : 0;
}

template <int PH>
__device__ __noinline__ void bi_finalize(const BiArgs &a, BiScalars *S, const double *d,
                                         bool writer = true) {
  const double btol = S->breakdown_tol;
  if (PH == BP_BNORM) {
    S->bnorm = __dsqrt_rn(d[0]);
    S->btnorm = __dsqrt_rn(d[1]);
  } else if (PH == BP_DUALCHK) {
    S->dual_rho = d[0];
    S->dual_rt2 = d[1];
    S->dual_r2 = d[2];
  } else if (PH == BP_INIT) {
    // record entry 0 and decide the initial status (solvers.py:508-579)
    S->rnorm = __dsqrt_rn(d[0]);
    S->rtnorm = __dsqrt_rn(d[1]);
    bi_record(a, S, writer);
    S->rho = S->dual_rho;
    S->beta = 0.0;
    bool conv = S->rnorm <= __dmul_rn(S->tol, S->bnorm) &&
                S->rtnorm <= __dmul_rn(S->tol, S->btnorm);
    if (conv) S->status = KRB_CONVERGED;
    else if (S->max_itn <= 0) S->status = KRB_MAX_ITN;
  } else if (PH == BP_PROJ) {
    S->n_matvec += 1;
    S->n_rmatvec += 1;
    double den = d[0];
    S->den = den;
    double npt = __dsqrt_rn(d[1]), nq = __dsqrt_rn(d[2]);
    if (fabs(den) <= __dmul_rn(__dmul_rn(btol, npt), nq))
      S->status = KRB_BREAKDOWN_SECOND_KIND;
    else
      S->alpha = __ddiv_rn(S->rho, den);
  } else if (PH == BP_XR) {
    S->rnorm = __dsqrt_rn(d[0]);
    S->rtnorm = __dsqrt_rn(d[1]);
    S->rho_new = d[2];
    bi_record(a, S, writer);
    S->itn += 1;
    S->xr_done = 1;
    // capture block (solvers.py:617-622): record alpha/beta, push attempt
    S->emit = 0;
    S->push_ok = 0;
    S->cap_now = 0;
    if (S->capture) {
      if (writer) {
        a.alphas[S->nalpha] = S->alpha;
        a.betas[S->nalpha] = S->beta;
      }
      S->nalpha += 1;
      if (S->rnorm == 0.0) S->capture = 0;
      else S->cap_now = 1;
      if (S->itn % S->s == 0) S->emit = 1;
    }
    // convergence / serious breakdown / beta (solvers.py:623-631)
    bool conv = S->rnorm <= __dmul_rn(S->tol, S->bnorm) &&
                S->rtnorm <= __dmul_rn(S->tol, S->btnorm);
    if (conv) {
      S->status = KRB_CONVERGED;
    } else if (fabs(S->rho_new) <= __dmul_rn(__dmul_rn(btol, S->rtnorm), S->rnorm)) {
      S->status = KRB_BREAKDOWN_SERIOUS;
    } else {
      S->beta = __ddiv_rn(S->rho_new, S->rho);
      S->rho = S->rho_new;
      if (S->itn >= S->max_itn) S->status = KRB_MAX_ITN;
    }
  } else if (PH == BP_CAP1) {
    double sigma = d[0];
    S->sigma = sigma;
    if (fabs(sigma) <= __dmul_rn(btol, S->rtnorm)) {
      S->capture = 0;
    } else {
      if (writer) a.rhos[S->npush] = S->rnorm;
      S->npush += 1;
      S->push_ok = 1;
    }
  } else if (PH == BP_TRUE) {
    double bn = __dsqrt_rn(d[1]);
    S->final_true_resid = __ddiv_rn(__dsqrt_rn(d[0]), bn > 0.0 ? bn : 1.0);
  }
}

template <int kE, int PH>
__global__ void __launch_bounds__(1024) k_bphase(const BiArgs *__restrict__ pa) {
  __shared__ double coef[2][512];
  __shared__ double red[4][32];
  __shared__ int last_flag;
  const BiArgs &a = *pa;
  BiScalars *S = a.S;
  constexpr int ND = bi_ndots(PH);
  if (PH == BP_PUPDATE && blockIdx.x == 0 && threadIdx.x == 0) {
    S->bodies += 1;
    S->xr_done = 0;
  }
  if ((PH == BP_PUPDATE || PH == BP_PROJ || PH == BP_XR) && S->status != KRB_RUNNING)
    return;
  if (PH == BP_CAP1 && !S->cap_now) return;
  if (PH == BP_CAP2) {
    // vt = rt / sigma for an accepted push; then loop control
    if (S->push_ok) {
      const double sg = S->sigma;
      double *vt = a.Vt + S->ncols * a.ring_ld;
      for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
           i += (int64_t)gridDim.x * blockDim.x)
        vt[i] = __ddiv_rn(a.rt[i], sg);
    }
    if (!elect_last_cta(a.counters + 32 + PH, &last_flag)) return;
    if (threadIdx.x == 0) {
      if (S->push_ok) S->ncols += 1;
      S->push_ok = 0;
      S->cap_now = 0;
      if (!S->xr_done) S->emit = 0;
      a.counters[32 + PH] = 0;
      if (a.use_cond)
        cudaGraphSetConditional(a.cond, (S->status == KRB_RUNNING && !S->emit) ? 1u : 0u);
    }
    return;
  }
  const double alpha = S->alpha, beta = S->beta;
  const int k = a.k;
  const int64_t n = a.n, nb = a.nb, ld = a.ld;
  if (PH == BP_PROJ && k > 0) {
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      coef[0][j] = a.zeta[j];
      coef[1][j] = a.zetat[j];
    }
    __syncthreads();
  }
  const double rn = S->rnorm;
  double *vcol = a.V + S->ncols * a.ring_ld;
  for (int64_t blk = blockIdx.x; blk < nb; blk += gridDim.x) {
    const int64_t base = blk * ((int64_t)kLanes * kE) + threadIdx.x;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
#pragma unroll
    for (int e = 0; e < kE; ++e) {
      const int64_t i = base + (int64_t)kLanes * e;
      if (i >= n) continue;
      if (PH == BP_PUPDATE) {
        // p = r + beta p ; pt = rt + conj(beta) pt     (solvers.py:589-590)
        a.p[i] = __dadd_rn(a.r[i], __dmul_rn(beta, a.p[i]));
        a.pt[i] = __dadd_rn(a.rt[i], __dmul_rn(beta, a.pt[i]));
      } else if (PH == BP_PROJ) {
        double qi = a.q[i], qti = a.qt[i];
        if (k > 0) {
          double c1 = 0.0, c2 = 0.0;
          for (int j = 0; j < k; ++j) {
            c1 = __fma_rn(__ldg(a.C + (int64_t)j * ld + i), coef[0][j], c1);
            c2 = __fma_rn(__ldg(a.Ct + (int64_t)j * ld + i), coef[1][j], c2);
          }
          qi = __dsub_rn(qi, c1);     // solvers.py:595
          qti = __dsub_rn(qti, c2);   // solvers.py:597
          a.q[i] = qi;
          a.qt[i] = qti;
        }
        double pti = a.pt[i];
        acc0 = __fma_rn(pti, qi, acc0);     // (pt, q)
        acc1 = __fma_rn(pti, pti, acc1);    // ||pt||^2
        acc2 = __fma_rn(qi, qi, acc2);      // ||q||^2
      } else if (PH == BP_XR) {
        // solvers.py:603-609
        a.x[i] = __dadd_rn(a.x[i], __dmul_rn(alpha, a.p[i]));
        a.xt[i] = __dadd_rn(a.xt[i], __dmul_rn(alpha, a.pt[i]));
        double ri = __dsub_rn(a.r[i], __dmul_rn(alpha, a.q[i]));
        double rti = __dsub_rn(a.rt[i], __dmul_rn(alpha, a.qt[i]));
        a.r[i] = ri;
        a.rt[i] = rti;
        acc0 = __fma_rn(ri, ri, acc0);
        acc1 = __fma_rn(rti, rti, acc1);
        acc2 = __fma_rn(rti, ri, acc2);     // rho_new = (rt, r)
      } else if (PH == BP_CAP1 || PH == BP_INIT) {
        // v = r / ||r|| ; sigma = (v, rt)              (solvers.py:568-569)
        if (PH == BP_INIT) {
          double ri = a.r[i], rti = a.rt[i];
          acc0 = __fma_rn(ri, ri, acc0);
          acc1 = __fma_rn(rti, rti, acc1);
        } else {
          double v = __ddiv_rn(a.r[i], rn);
          vcol[i] = v;
          acc0 = __fma_rn(v, a.rt[i], acc0);
        }
      } else if (PH == BP_BNORM) {
        double bi = a.b[i], bti = a.bt[i];
        acc0 = __fma_rn(bi, bi, acc0);
        acc1 = __fma_rn(bti, bti, acc1);
      } else if (PH == BP_DUALCHK) {
        double ri = a.r[i], rti = a.rt[i];
        acc0 = __fma_rn(rti, ri, acc0);      // rho = (rt0, r0)
        acc1 = __fma_rn(rti, rti, acc1);
        acc2 = __fma_rn(ri, ri, acc2);
      } else if (PH == BP_TRUE) {
        double bi = a.b[i];
        double res = __dsub_rn(bi, a.q[i]);   // A x_out in q
        acc0 = __fma_rn(res, res, acc0);
        acc1 = __fma_rn(bi, bi, acc1);
      } else if (PH == BP_RINIT) {
        a.r[i] = __dsub_rn(a.b[i], a.q[i]);
      } else if (PH == BP_RTINIT) {
        a.rt[i] = __dsub_rn(a.bt[i], a.qt[i]);
      }
    }
    if (ND > 0) {
      double accs[3] = {acc0, acc1, acc2};
      double bp = block_tree_multi<ND == 0 ? 1 : ND>(accs, red);
      const int warp = threadIdx.x >> 5;
      if (warp < ND && (threadIdx.x & 31) == 0) a.part[warp * nb + blk] = bp;
    }
  }
  if (ND == 0) return;
  if (!elect_last_cta(a.counters + 32 + PH, &last_flag)) return;
  __shared__ double dfin[3];
  const int warp = threadIdx.x >> 5;
  if (warp < ND) {
    double v = warp_final_volatile(a.part + warp * nb, nb);
    if ((threadIdx.x & 31) == 0) dfin[warp] = v;
  }
  if (PH == BP_XR) {
    // zc += alpha zeta ; ztc += conj(alpha) zetat     (solvers.py:605-607)
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      a.zc[j] = __dadd_rn(a.zc[j], __dmul_rn(alpha, a.zeta[j]));
      a.ztc[j] = __dadd_rn(a.ztc[j], __dmul_rn(alpha, a.zetat[j]));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bi_finalize<PH>(a, a.S, dfin);
    a.counters[32 + PH] = 0;
  }
}

template <int kE, bool kDual>
__global__ void __launch_bounds__(1024) k_bproj_dot(const BiArgs *__restrict__ pa) {
  const BiArgs &a = *pa;
  if (a.S->status != KRB_RUNNING) return;
  tdot_body<kE, false>(a.n, a.nb, a.k, kDual ? a.Ccheck : a.Chat, a.ld,
                       kDual ? a.qt : a.q, a.part + (kDual ? (int64_t)a.k * a.nb : 0),
                       kDual ? a.zetat : a.zeta,
                       a.counters + (kDual ? 61 : 60));
}

// kF: 0 CSR, 1 SELL-32 / SELL-C-sigma, 2 offset-coded SELL-32 (with the
// values' bulk L2 prefetch pf bytes ahead, as the BiCGSTAB SpMV)
template <int kF, bool kTrans>
__global__ void __launch_bounds__(256, kF == 2 || kF == 5 ? 6 : kF == 4 ? 4 : 1) k_bspmv(const BiArgs *__restrict__ pa,
                                                                int64_t pf) {
  constexpr bool kSell = kF == 1;
  const BiArgs &a = *pa;
  if (a.S->status != KRB_RUNNING) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const krb_matrix &M = kTrans ? a.AT : a.A;
  const double *__restrict__ x = kTrans ? a.pt : a.p;
  double *y = kTrans ? a.qt : a.q;
  if (kF == 2 || kF == 4 || kF == 5) {   // 4 / 5: value-coded (row templates / diagonal form)
    auto xf = [x](int c) { return __ldg(x + c); };
    if (kF == 5)
      y[i] = spmv_row_dia(i, M, x);
    else if (kF == 4)
      y[i] = spmv_row_tmpl(i, M, xf);
    else
      y[i] = spmv_row_dict<0, decltype(xf), 4>(i, M, xf, pf);
  } else {
    y[(kSell && M.perm) ? M.perm[i] : i] = spmv_row<kSell>(i, M, x);
  }
}

__global__ void k_bi_init_scalars(BiScalars *S, double tol, double btol,
                                  int64_t max_itn, int64_t s, int capture) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    BiScalars z = {};
    z.tol = tol;
    z.breakdown_tol = btol;
    z.max_itn = max_itn;
    z.s = s;
    z.capture = capture;
    z.t_start = globaltimer();
    *S = z;
  }
}


template <int PH>
static int bi_launch(const BiArgs &h, const BiArgs *d, cudaStream_t st) {
  if (h.nb == 0) return KRB_OK;
  int grid = grid_for(h.nb);
  KRB_DISPATCH_E(canon_E(h.n), (k_bphase<kE, PH><<<grid, 1024, 0, st>>>(d)));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

static int spmv_kind(const krb_matrix *M) {
  if (M->tent && tuning().value_coding)
    return (M->dia.nd && tuning().value_coding != 2) ? 3 : 2;
  return M->dcode ? 1 : 0;
}

template <bool kTrans>
static int bi_spmv(const BiArgs &h, const BiArgs *d, cudaStream_t st) {
  const krb_matrix &M = kTrans ? h.AT : h.A;
  if (h.n == 0) return KRB_OK;
  if (M.pre)   // split-ILUTP operator / its adjoint (precond.cu)
    return spmv_launch(&M, kTrans ? h.pt : h.p, kTrans ? h.qt : h.q,
                       reinterpret_cast<const int *>(&h.S->status), st);
  unsigned blocks = (unsigned)((h.n + 255) / 256);
  if (spmv_kind(&M) == 3)
    k_bspmv<5, kTrans><<<blocks, 256, 0, st>>>(d, 0);
  else if (spmv_kind(&M) == 2)
    k_bspmv<4, kTrans><<<blocks, 256, 0, st>>>(d, 0);
  else if (M.dcode)
    k_bspmv<2, kTrans><<<blocks, 256, 0, st>>>(d, (int64_t)tuning().spmv_prefetch_mb << 20);
  else if (M.format == 2)
    k_bspmv<1, kTrans><<<blocks, 256, 0, st>>>(d, 0);
  else
    k_bspmv<0, kTrans><<<blocks, 256, 0, st>>>(d, 0);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

template <bool kDual>
static int bi_proj_dot(const BiArgs &h, const BiArgs *d, cudaStream_t st) {
  if (h.k <= 0 || h.nb == 0) return KRB_OK;
  static int per_sm = occupancy_1024(k_bproj_dot<16, kDual>);
  dim3 grid = tdot_grid(h.nb, h.k, per_sm);
  KRB_DISPATCH_E(canon_E(h.n), (k_bproj_dot<kE, kDual><<<grid, 1024, 0, st>>>(d)));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}


// ---------------------------------------------------------------------------
// persistent driver for n <= 606208 (the graph's conditional-node loop costs
// ~16 us per iteration at this size): one cooperative kernel runs iterations
// until a cycle is complete (emit) or the solve stops; phases separated by
// grid barriers, every CTA runs the canonical final stages and the scalar
// logic on its own shared copy of the scalar block (identical inputs, order
// -> identical scalars), CTA 0 writes history, rings' scalars and the block.
// ---------------------------------------------------------------------------
template <int ND>
__device__ __forceinline__ void bi_local_finals(const double *pb, int64_t nb, double *dfin) {
  const int warp = threadIdx.x >> 5;
  if (warp < ND) {
    double v = warp_final_volatile(pb + warp * nb, nb);
    if ((threadIdx.x & 31) == 0) dfin[warp] = v;
  }
  __syncthreads();
}

template <int ND>
__device__ __forceinline__ void bi_block_partials(double *acc, double (*red)[32],
                                                  double *pb, int64_t nb, int64_t blk) {
  double bp = block_tree_multi<ND>(acc, red);
  const int warp = threadIdx.x >> 5;
  if (warp < ND && (threadIdx.x & 31) == 0) pb[warp * nb + blk] = bp;
}

template <bool kSell>
__device__ __forceinline__ double bi_row(int64_t i, const krb_matrix &M, const double *x) {
  return spmv_row<kSell, false>(i, M, x);
}

template <int kE, bool kSell>
__global__ void __launch_bounds__(1024) k_bpersist(const BiArgs *__restrict__ pa) {
  __shared__ double zeta[512], zetat[512];
  __shared__ double red[kTdotCG][32];
  __shared__ double dfin[3];
  __shared__ BiScalars L;
  cg::grid_group grid = cg::this_grid();
  const BiArgs &a = *pa;
  const int64_t G = gridDim.x, me = blockIdx.x;
  const int64_t n = a.n, nb = a.nb, ld = a.ld;
  const int k = a.k;
  const int64_t ncg = (k + kTdotCG - 1) / kTdotCG;
  const bool writer = me == 0;
  const krb_matrix A = a.A, AT = a.AT;
  const bool tsell = AT.format == 2;
  // owner-computes fusion needs unpermuted rows of A, k = 0 and every
  // canonical block owned by one CTA (E <= 2, nb <= 2 G)
  const bool fused = k == 0 && A.perm == nullptr && nb <= 2 * G;
  if (threadIdx.x == 0) L = *a.S;
  __syncthreads();
  double *pb[2] = {a.part, a.part2};
  int cur = 0;
  for (;;) {
    if (L.status != KRB_RUNNING) break;
    // ---- P: p = r + beta p ; pt = rt + conj(beta) pt   (solvers.py:589-590)
    if (threadIdx.x == 0) {
      L.bodies += 1;
      L.xr_done = 0;
    }
    const double beta = L.beta;
    double *pcur = a.p, *ptcur = a.pt;
    if (fused) {
      // k = 0, unpermuted rows: p, pt recomputed on the fly for every
      // gathered column (owners write the new ones into the other buffer),
      // both SpMVs and Q's dots from registers -- P, M and Q in one phase
      const double *po = L.pbuf ? a.p2 : a.p, *pto = L.pbuf ? a.pt2 : a.pt;
      double *pn = L.pbuf ? a.p : a.p2, *ptn = L.pbuf ? a.pt : a.pt2;
      pcur = pn;
      ptcur = ptn;
      const double *__restrict__ r_ = a.r;
      const double *__restrict__ rt_ = a.rt;
      auto pf = [=](int c) { return __dadd_rn(r_[c], __dmul_rn(beta, po[c])); };
      auto ptf = [=](int c) { return __dadd_rn(rt_[c], __dmul_rn(beta, pto[c])); };
      for (int64_t blk = me; blk < nb; blk += G) {
        const int64_t base = blk * ((int64_t)kLanes * kE) + threadIdx.x;
        double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          const int64_t i = base + (int64_t)kLanes * e;
          if (i >= n) continue;
          const double pv = pf((int)i), ptv = ptf((int)i);
          pn[i] = pv;
          ptn[i] = ptv;
          const double qi = spmv_row_f<kSell>(i, A, pf);
          a.q[i] = qi;
          const double qt = tsell ? spmv_row_f<true>(i, AT, ptf) : spmv_row_f<false>(i, AT, ptf);
          a.qt[(tsell && AT.perm) ? AT.perm[i] : i] = qt;
          acc[0] = __fma_rn(ptv, qi, acc[0]);
          acc[1] = __fma_rn(ptv, ptv, acc[1]);
          acc[2] = __fma_rn(qi, qi, acc[2]);
        }
        bi_block_partials<3>(acc, red, pb[cur], nb, blk);
      }
      grid.sync();
    } else {
      for (int64_t i = me * blockDim.x + threadIdx.x; i < n; i += G * blockDim.x) {
        a.p[i] = __dadd_rn(a.r[i], __dmul_rn(beta, a.p[i]));
        a.pt[i] = __dadd_rn(a.rt[i], __dmul_rn(beta, a.pt[i]));
      }
      grid.sync();
      // ---- M: q = A p, qt = A^T pt
      for (int64_t i = me * blockDim.x + threadIdx.x; i < n; i += G * blockDim.x) {
        a.q[(kSell && A.perm) ? A.perm[i] : i] = bi_row<kSell>(i, A, a.p);
        const double qt = tsell ? bi_row<true>(i, AT, a.pt) : bi_row<false>(i, AT, a.pt);
        a.qt[(tsell && AT.perm) ? AT.perm[i] : i] = qt;
      }
      grid.sync();
      // ---- Z: zeta = Chat^T q, zetat = Ccheck^T qt
      if (k > 0) {
        for (int64_t u = me; u < 2 * nb * ncg; u += G) {
          const bool dual = u >= nb * ncg;
          const int64_t v = dual ? u - nb * ncg : u;
          tdot_unit<kE, false>(n, nb, k, dual ? a.Ccheck : a.Chat, ld, dual ? a.qt : a.q,
                               pb[cur] + (dual ? (int64_t)k * nb : 0), v % nb,
                               (int)(v / nb) * kTdotCG, red);
        }
        grid.sync();
        tdot_finals<false>(nb, k, pb[cur], zeta);
        tdot_finals<false>(nb, k, pb[cur] + (int64_t)k * nb, zetat);
        __syncthreads();
        cur ^= 1;
      }
      // ---- Q: q -= C zeta, qt -= Ct zetat ; (pt,q), (pt,pt), (q,q)
      for (int64_t blk = me; blk < nb; blk += G) {
        const int64_t base = blk * ((int64_t)kLanes * kE) + threadIdx.x;
        double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          const int64_t i = base + (int64_t)kLanes * e;
          if (i >= n) continue;
          double qi = a.q[i], qti = a.qt[i];
          if (k > 0) {
            double c1 = 0.0, c2 = 0.0;
            for (int j = 0; j < k; ++j) {
              c1 = __fma_rn(__ldg(a.C + (int64_t)j * ld + i), zeta[j], c1);
              c2 = __fma_rn(__ldg(a.Ct + (int64_t)j * ld + i), zetat[j], c2);
            }
            qi = __dsub_rn(qi, c1);     // solvers.py:595
            qti = __dsub_rn(qti, c2);   // solvers.py:597
            a.q[i] = qi;
            a.qt[i] = qti;
          }
          const double pti = a.pt[i];
          acc[0] = __fma_rn(pti, qi, acc[0]);
          acc[1] = __fma_rn(pti, pti, acc[1]);
          acc[2] = __fma_rn(qi, qi, acc[2]);
        }
        bi_block_partials<3>(acc, red, pb[cur], nb, blk);
      }
      grid.sync();
    }
    bi_local_finals<3>(pb[cur], nb, dfin);
    cur ^= 1;
    if (threadIdx.x == 0) {
      bi_finalize<BP_PROJ>(a, &L, dfin, writer);
      if (fused) L.pbuf ^= 1;
    }
    __syncthreads();
    if (L.status == KRB_RUNNING) {
      // ---- X: x, xt, r, rt ; (r,r), (rt,rt), (rt,r)   (solvers.py:603-609)
      const double alpha = L.alpha;
      for (int64_t blk = me; blk < nb; blk += G) {
        const int64_t base = blk * ((int64_t)kLanes * kE) + threadIdx.x;
        double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          const int64_t i = base + (int64_t)kLanes * e;
          if (i >= n) continue;
          a.x[i] = __dadd_rn(a.x[i], __dmul_rn(alpha, pcur[i]));
          a.xt[i] = __dadd_rn(a.xt[i], __dmul_rn(alpha, ptcur[i]));
          const double ri = __dsub_rn(a.r[i], __dmul_rn(alpha, a.q[i]));
          const double rti = __dsub_rn(a.rt[i], __dmul_rn(alpha, a.qt[i]));
          a.r[i] = ri;
          a.rt[i] = rti;
          acc[0] = __fma_rn(ri, ri, acc[0]);
          acc[1] = __fma_rn(rti, rti, acc[1]);
          acc[2] = __fma_rn(rti, ri, acc[2]);
        }
        bi_block_partials<3>(acc, red, pb[cur], nb, blk);
      }
      if (writer)   // zc += alpha zeta ; ztc += conj(alpha) zetat   (:605-607)
        for (int j = threadIdx.x; j < k; j += blockDim.x) {
          a.zc[j] = __dadd_rn(a.zc[j], __dmul_rn(alpha, zeta[j]));
          a.ztc[j] = __dadd_rn(a.ztc[j], __dmul_rn(alpha, zetat[j]));
        }
      grid.sync();
      bi_local_finals<3>(pb[cur], nb, dfin);
      cur ^= 1;
      if (threadIdx.x == 0) bi_finalize<BP_XR>(a, &L, dfin, writer);
      __syncthreads();
      // ---- capture: v = r / ||r|| into the ring ; sigma = (v, rt)   (:568-569)
      if (L.cap_now) {
        const double rn = L.rnorm;
        double *vcol = a.V + L.ncols * a.ring_ld;
        for (int64_t blk = me; blk < nb; blk += G) {
          const int64_t base = blk * ((int64_t)kLanes * kE) + threadIdx.x;
          double acc[1] = {0.0};
#pragma unroll
          for (int e = 0; e < kE; ++e) {
            const int64_t i = base + (int64_t)kLanes * e;
            if (i >= n) continue;
            const double v = __ddiv_rn(a.r[i], rn);
            vcol[i] = v;
            acc[0] = __fma_rn(v, a.rt[i], acc[0]);
          }
          bi_block_partials<1>(acc, red, pb[cur], nb, blk);
        }
        grid.sync();
        bi_local_finals<1>(pb[cur], nb, dfin);
        cur ^= 1;
        if (threadIdx.x == 0) bi_finalize<BP_CAP1>(a, &L, dfin, writer);
        __syncthreads();
      }
      if (L.push_ok) {   // vt = rt / sigma
        const double sg = L.sigma;
        double *vt = a.Vt + L.ncols * a.ring_ld;
        for (int64_t i = me * blockDim.x + threadIdx.x; i < n; i += G * blockDim.x)
          vt[i] = __ddiv_rn(a.rt[i], sg);
      }
    }
    // loop control (the graph's CAP2 bookkeeping)
    if (threadIdx.x == 0) {
      if (L.push_ok) L.ncols += 1;
      L.push_ok = 0;
      L.cap_now = 0;
      if (!L.xr_done) L.emit = 0;
    }
    __syncthreads();
    if (L.status != KRB_RUNNING || L.emit) break;
  }
  if (writer && threadIdx.x == 0) *a.S = L;
}

template <int kE, bool kSell>
static int bpersist_launch(const BiArgs *d, cudaStream_t st) {
  static int grid = 0;
  if (grid == 0) {
    int per_sm = 0;
    KRB_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, k_bpersist<kE, kSell>, 1024, 0));
    int dev = 0, sms = kNumSMs;
    KRB_CHECK_CUDA(cudaGetDevice(&dev));
    KRB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = (per_sm > 0 ? per_sm : 1) * sms;
  }
  void *args[] = {(void *)&d};
  KRB_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)k_bpersist<kE, kSell>,
                                             dim3(grid), dim3(1024), args, 0, st));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

static int bi_persistent(const BiArgs &h, const BiArgs *d, cudaStream_t st) {
  if (h.n == 0) return KRB_OK;
  const bool sell = h.A.format == 2;
  switch (canon_E(h.n)) {
    case 1: return sell ? bpersist_launch<1, true>(d, st) : bpersist_launch<1, false>(d, st);
    case 2: return sell ? bpersist_launch<2, true>(d, st) : bpersist_launch<2, false>(d, st);
    default:
      set_error("persistent rbicg driver supports n <= %d", 2 * kLanes * kTargetBlocks);
      return KRB_EINVAL;
  }
}

static int bi_iteration(const BiArgs &h, const BiArgs *d, cudaStream_t st) {
  KRB_TRY(bi_launch<BP_PUPDATE>(h, d, st));
  KRB_TRY(bi_spmv<false>(h, d, st));
  KRB_TRY(bi_spmv<true>(h, d, st));
  KRB_TRY(bi_proj_dot<false>(h, d, st));
  KRB_TRY(bi_proj_dot<true>(h, d, st));
  KRB_TRY(bi_launch<BP_PROJ>(h, d, st));
  KRB_TRY(bi_launch<BP_XR>(h, d, st));
  KRB_TRY(bi_launch<BP_CAP1>(h, d, st));
  KRB_TRY(bi_launch<BP_CAP2>(h, d, st));
  return KRB_OK;
}

}  // namespace krb

// ---------------------------------------------------------------------------
// solve handle: the host drives setup / pause-resume / finish
// ---------------------------------------------------------------------------
struct krb_rbicg {
  krb_context *ctx = nullptr;
  krb_matrix *A = nullptr;
  krb::BiArgs h = {};
  krb::BiArgs *d = nullptr;     // descriptor read by the graph (conditional on)
  krb::BiArgs *d_nc = nullptr;  // descriptor for stand-alone launches
  double *bufs = nullptr;      // 10 n-vectors
  double *kb = nullptr;        // zeta, zetat, zc, ztc, y
  double *scal = nullptr;      // rhos, alphas, betas
  double *ring = nullptr;      // V and Vt rings (2 x (s+2) x n)
  double *hist = nullptr;      // resid, resid_dual
  int64_t *hist_m = nullptr;
  uint64_t *hist_t = nullptr;
  krb::BiScalars *S = nullptr;
  // the handle's own block-partial buffers (two ping-pong halves): the
  // context's shared scratch may be reallocated by any kernel a cycle
  // callback launches (update_recycle_space's Grams / norms) while this
  // handle's descriptor still holds the pointer
  double *part = nullptr;
  krb::MatrixSig sig;       // operator whose composite kernels the graph bakes
  int64_t s = 0, max_itn = 0, k = 0;
  krb_space_view R = {};
  bool has_R = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t per_body = 0;
  int64_t l0 = 0;
  int use_graph = 1;
  int fmt = -1, fmt_t = -1;   // storage formats the graph was captured for
  int dict = 0, dict_t = 0;   // SpMV kernels captured: 1 offset-coded, 2 / 3 value-coded
  // host copy of the scalar block as of the last begin / run (the device
  // block only changes inside those calls and in rotate, which keeps this
  // copy current): run and rotate need no extra read-back + synchronisation
  krb::BiScalars hs = {};
  bool hs_valid = false;
};

namespace krb {

static cudaStream_t bi_capture_stream() {
  static thread_local cudaStream_t s = nullptr;
  if (!s) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  return s;
}

static void bi_free(krb_rbicg *H) {
  if (!H) return;
  if (H->exec) cudaGraphExecDestroy(H->exec);
  if (H->graph) cudaGraphDestroy(H->graph);
  cudaFree(H->d);
  cudaFree(H->d_nc);
  cudaFree(H->bufs);
  cudaFree(H->kb);
  cudaFree(H->scal);
  cudaFree(H->ring);
  cudaFree(H->hist);
  cudaFree(H->hist_m);
  cudaFree(H->hist_t);
  cudaFree(H->S);
  cudaFree(H->part);
  delete H;
}

static int bi_build_graph(krb_rbicg *H) {
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
  cudaStream_t cs = bi_capture_stream();
  KRB_CHECK_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeRelaxed));
  const int64_t c0 = launch_counter();
  int rc = bi_iteration(H->h, H->d, cs);
  H->per_body = launch_counter() - c0;
  launch_counter() = c0;
  cudaGraph_t out;
  cudaError_t e = cudaStreamEndCapture(cs, &out);
  if (rc || e != cudaSuccess) {
    cudaGraphDestroy(g);
    if (!rc) set_error("rbicg graph capture: %s", cudaGetErrorString(e));
    return rc ? rc : KRB_ECUDA;
  }
  e = cudaGraphInstantiate(&H->exec, g, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    set_error("rbicg graph instantiate: %s", cudaGetErrorString(e));
    return KRB_ECUDA;
  }
  H->graph = g;
  H->h.cond = hc;
  H->h.use_cond = 1;
  // upload once so every resume after a harvest pause is a plain launch
  KRB_CHECK_CUDA(cudaGraphUpload(H->exec, cs));
  KRB_CHECK_CUDA(cudaStreamSynchronize(cs));
  return KRB_OK;
}

}  // namespace krb

using namespace krb;

extern "C" {

int krb_rbicg_create(krb_rbicg **out, krb_context *ctx, krb_matrix *A,
                     const krb_space_view *R, int64_t s, int64_t max_itn,
                     void *stream) {
  KRB_REQUIRE(out && ctx && A, "krb_rbicg_create: NULL argument");
  KRB_REQUIRE(s >= 0 && max_itn >= 0, "krb_rbicg_create: negative s / max_itn");
  cudaStream_t st = as_stream(stream);
  int rc = ensure_transpose(A, st);
  if (rc) return rc;
  const int64_t n = A->n;
  const int64_t k = (R && R->k > 0) ? R->k : 0;
  if (k > 0 && (R->n != n || R->ld < n)) {
    set_error("recycle space dimension does not match the operator");
    return KRB_EINVAL;
  }
  // reuse the cached handle of the same shape (buffers, descriptors and the
  // instantiated graph, whose kernels read everything per solve from H->d)
  krb_rbicg *H = ctx->bi_cache;
  const bool reuse = H && H->h.n == n && H->k == k && H->s == s && H->max_itn == max_itn &&
                     H->fmt == A->format && H->fmt_t == A->T->format &&
                     H->dict == spmv_kind(A) && H->dict_t == spmv_kind(A->T) &&
                     (!A->pre || same_sig(H->sig, matrix_sig(A)));
  if (H && !reuse) bi_free(H);
  ctx->bi_cache = nullptr;
  if (!reuse) H = new krb_rbicg();
  H->ctx = ctx;
  H->A = A;
  H->s = s;
  H->max_itn = max_itn;
  H->has_R = k > 0;
  if (k > 0) H->R = *R;
  H->k = k;
  H->fmt = A->format;
  H->fmt_t = A->T->format;
  H->dict = spmv_kind(A);
  H->dict_t = spmv_kind(A->T);
  H->sig = matrix_sig(A);
  const int64_t nb = canon_nblocks(n);
  const int64_t ring_cols = (s > 0 ? s : 0) + 3;
  cudaError_t e = cudaSuccess;
  if (reuse) goto fill;
  e = cudaMalloc(&H->d, sizeof(BiArgs));
  if (e == cudaSuccess) e = cudaMalloc(&H->d_nc, sizeof(BiArgs));
  if (e == cudaSuccess) e = cudaMalloc(&H->bufs, sizeof(double) * 12 * (n > 0 ? n : 1));
  if (e == cudaSuccess) e = cudaMalloc(&H->kb, sizeof(double) * 5 * (k > 0 ? k : 1));
  if (e == cudaSuccess) e = cudaMalloc(&H->scal, sizeof(double) * (3 * (max_itn + ring_cols + 2)));
  if (e == cudaSuccess) e = cudaMalloc(&H->ring, sizeof(double) * 2 * ring_cols * (n > 0 ? n : 1));
  if (e == cudaSuccess) e = cudaMalloc(&H->hist, sizeof(double) * 2 * (max_itn + 2));
  if (e == cudaSuccess) e = cudaMalloc(&H->hist_m, sizeof(int64_t) * (max_itn + 2));
  if (e == cudaSuccess) e = cudaMalloc(&H->hist_t, sizeof(uint64_t) * (max_itn + 2));
  if (e == cudaSuccess) e = cudaMalloc(&H->S, sizeof(BiScalars));
  if (e == cudaSuccess)
    e = cudaMalloc(&H->part, sizeof(double) * 2 * ((size_t)((2 * k + 3) * nb) + 64));
  if (e != cudaSuccess) {
    set_error("krb_rbicg_create: %s", cudaGetErrorString(e));
    bi_free(H);
    return KRB_ENOMEM;
  }
fill:
  const size_t part_one = (size_t)((2 * k + 3) * nb) + 64;
  rc = ctx_reserve_counters(ctx, st);
  if (rc) {
    bi_free(H);
    return rc;
  }
  BiArgs &h = H->h;
  h.A = *A;
  h.A.T = nullptr;
  h.AT = *A->T;
  h.AT.T = nullptr;
  h.n = n;
  h.nb = nb;
  h.k = (int)k;
  h.ld = k > 0 ? R->ld : n;
  h.ring_ld = n;
  h.C = k > 0 ? R->C : nullptr;
  h.Chat = k > 0 ? R->Chat : nullptr;
  h.Ct = k > 0 ? R->Ct : nullptr;
  h.Ccheck = k > 0 ? R->Ccheck : nullptr;
  double *B = H->bufs;
  h.x = B; h.xt = B + n; h.r = B + 2 * n; h.rt = B + 3 * n; h.p = B + 4 * n;
  h.pt = B + 5 * n; h.q = B + 6 * n; h.qt = B + 7 * n; h.b = B + 8 * n; h.bt = B + 9 * n;
  h.p2 = B + 10 * n; h.pt2 = B + 11 * n;
  h.zeta = H->kb; h.zetat = H->kb + k; h.zc = H->kb + 2 * k; h.ztc = H->kb + 3 * k;
  h.V = H->ring;
  h.Vt = H->ring + ring_cols * n;
  h.rhos = H->scal;
  h.alphas = H->scal + (max_itn + ring_cols + 2);
  h.betas = H->scal + 2 * (max_itn + ring_cols + 2);
  h.part = H->part;
  h.part2 = H->part + part_one;
  h.counters = ctx->counters;
  h.S = H->S;
  h.hist_r = H->hist;
  h.hist_rt = H->hist + (max_itn + 2);
  h.hist_m = H->hist_m;
  h.hist_t = H->hist_t;
  *out = H;
  return KRB_OK;
}

int krb_rbicg_destroy(krb_rbicg *H) {
  if (!H) return KRB_OK;
  // keep the resources for the next generation solve of the same shape
  if (H->ctx) {
    if (H->ctx->bi_cache && H->ctx->bi_cache != H) bi_free(H->ctx->bi_cache);
    H->ctx->bi_cache = H;
    return KRB_OK;
  }
  bi_free(H);
  return KRB_OK;
}

}  // extern "C"

namespace krb {
void rbicg_cache_free(krb_context *ctx) {
  if (ctx && ctx->bi_cache) {
    bi_free(ctx->bi_cache);
    ctx->bi_cache = nullptr;
  }
}
}  // namespace krb

extern "C" {

/* Setup: b, b_dual, x_init, x_init_dual (device, NULLable except b, bt).
 * Runs project_initial / project_initial_dual and the dual-start test; the
 * three dual-start scalars are returned in h_dual[3] = (rho, ||rt0||^2,
 * ||r0||^2) so the host can re-draw xt exactly as solvers.py:364-375. */
int krb_rbicg_start(krb_rbicg *H, const double *d_b, const double *d_bt,
                    const double *d_x0, const double *d_xt0, double tol,
                    double breakdown_tol, int use_graph, double *h_dual,
                    void *stream) {
  if (H) H->hs_valid = false;
  KRB_REQUIRE(H && d_b && d_bt && h_dual, "krb_rbicg_start: NULL argument");
  cudaStream_t st = as_stream(stream);
  BiArgs &h = H->h;
  const int64_t n = h.n, k = h.k;
  if (H->A->pre && use_graph == 2) use_graph = 1;   // operator products are kernel sequences
  H->use_graph = use_graph;
  H->l0 = launch_counter();
  if (use_graph == 1 && !H->exec) {
    KRB_CHECK_CUDA(cudaStreamSynchronize(st));
    int rc = bi_build_graph(H);
    if (rc) return rc;
  }
  h.use_cond = use_graph == 1 ? 1 : 0;
  KRB_CHECK_CUDA(cudaMemcpyAsync(H->d, &h, sizeof(BiArgs), cudaMemcpyHostToDevice, st));
  BiArgs hnc = h;
  hnc.use_cond = 0;
  KRB_CHECK_CUDA(cudaMemcpyAsync(H->d_nc, &hnc, sizeof(BiArgs), cudaMemcpyHostToDevice, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  k_bi_init_scalars<<<1, 1, 0, st>>>(h.S, tol, breakdown_tol, H->max_itn, H->s > 0 ? H->s : 1,
                                     H->s > 0 ? 1 : 0);
  KRB_CHECK_LAUNCH();
  KRB_CHECK_CUDA(cudaMemcpyAsync(h.b, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  KRB_CHECK_CUDA(cudaMemcpyAsync(h.bt, d_bt, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  KRB_TRY(bi_launch<BP_BNORM>(h, H->d_nc, st));
  double *y = H->kb + 4 * k;
  // primary: project_initial (recycling.py:189-206)
  if (d_x0) {
    KRB_CHECK_CUDA(cudaMemcpyAsync(h.x, d_x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    KRB_TRY(spmv_launch(H->A, h.x, h.q, nullptr, st));
    KRB_TRY(bi_launch<BP_RINIT>(h, H->d_nc, st));
  } else {
    KRB_CHECK_CUDA(cudaMemsetAsync(h.x, 0, sizeof(double) * n, st));
    KRB_CHECK_CUDA(cudaMemcpyAsync(h.r, h.b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
  if (k > 0) {
    KRB_TRY(launch_tdot(H->ctx, n, k, H->R.Chat, H->R.ld, h.r, false, y, nullptr, st));
    KRB_TRY(launch_gemv(n, k, H->R.U, H->R.ld, y, h.x, +1, h.x, st));
    KRB_TRY(launch_gemv(n, k, H->R.C, H->R.ld, y, h.r, -1, h.r, st));
  }
  // dual: project_initial_dual (recycling.py:209-222)
  if (d_xt0) {
    KRB_CHECK_CUDA(cudaMemcpyAsync(h.xt, d_xt0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    KRB_TRY(spmv_launch(H->A->T, h.xt, h.qt, nullptr, st));
    KRB_TRY(bi_launch<BP_RTINIT>(h, H->d_nc, st));
  } else {
    KRB_CHECK_CUDA(cudaMemsetAsync(h.xt, 0, sizeof(double) * n, st));
    KRB_CHECK_CUDA(cudaMemcpyAsync(h.rt, h.bt, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
  if (k > 0) {
    KRB_TRY(launch_tdot(H->ctx, n, k, H->R.Ccheck, H->R.ld, h.rt, false, y, nullptr, st));
    KRB_TRY(launch_gemv(n, k, H->R.Ut, H->R.ld, y, h.xt, +1, h.xt, st));
    KRB_TRY(launch_gemv(n, k, H->R.Ct, H->R.ld, y, h.rt, -1, h.rt, st));
  }
  KRB_TRY(bi_launch<BP_DUALCHK>(h, H->d_nc, st));
  BiScalars hs;
  KRB_CHECK_CUDA(cudaMemcpyAsync(&hs, h.S, sizeof(hs), cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  h_dual[0] = hs.dual_rho;
  h_dual[1] = hs.dual_rt2;
  h_dual[2] = hs.dual_r2;
  return KRB_OK;
}

/* Counted products so far (x_init / xt_init starts): set by the host after a
 * successful dual start (it knows how many re-draw attempts were made). */
int krb_rbicg_set_counts(krb_rbicg *H, int64_t n_matvec, int64_t n_rmatvec,
                         void *stream) {
  KRB_REQUIRE(H, "krb_rbicg_set_counts: NULL handle");
  H->hs_valid = false;
  cudaStream_t st = as_stream(stream);
  KRB_CHECK_CUDA(cudaMemcpyAsync(&H->S->n_matvec, &n_matvec, sizeof(int64_t),
                                 cudaMemcpyHostToDevice, st));
  KRB_CHECK_CUDA(cudaMemcpyAsync(&H->S->n_rmatvec, &n_rmatvec, sizeof(int64_t),
                                 cudaMemcpyHostToDevice, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  return KRB_OK;
}

/* Record entry 0, initial status, zero p/pt/zc/ztc and push the first Lanczos
 * pair (solvers.py:496-582).  Returns the status. */
int krb_rbicg_begin(krb_rbicg *H, int32_t *h_status, void *stream) {
  KRB_REQUIRE(H && h_status, "krb_rbicg_begin: NULL argument");
  cudaStream_t st = as_stream(stream);
  BiArgs &h = H->h;
  const int64_t n = h.n, k = h.k;
  KRB_CHECK_CUDA(cudaMemsetAsync(h.p, 0, sizeof(double) * n, st));
  KRB_CHECK_CUDA(cudaMemsetAsync(h.pt, 0, sizeof(double) * n, st));
  if (k > 0) KRB_CHECK_CUDA(cudaMemsetAsync(h.zc, 0, sizeof(double) * 2 * k, st));
  KRB_TRY(bi_launch<BP_INIT>(h, H->d_nc, st));
  // first push (_push_lanczos before the loop, solvers.py:577)
  BiScalars hs;
  KRB_CHECK_CUDA(cudaMemcpyAsync(&hs, h.S, sizeof(hs), cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  if (hs.capture) {
    int32_t cap_now = hs.rnorm != 0.0 ? 1 : 0;
    int32_t cap = cap_now;
    KRB_CHECK_CUDA(cudaMemcpyAsync(&h.S->cap_now, &cap_now, sizeof(int32_t),
                                   cudaMemcpyHostToDevice, st));
    KRB_CHECK_CUDA(cudaMemcpyAsync(&h.S->capture, &cap, sizeof(int32_t),
                                   cudaMemcpyHostToDevice, st));
    int32_t one = 1;
    KRB_CHECK_CUDA(cudaMemcpyAsync(&h.S->xr_done, &one, sizeof(int32_t),
                                   cudaMemcpyHostToDevice, st));
    KRB_TRY(bi_launch<BP_CAP1>(h, H->d_nc, st));
    KRB_TRY(bi_launch<BP_CAP2>(h, H->d_nc, st));
    int32_t zero = 0;
    KRB_CHECK_CUDA(cudaMemcpyAsync(&h.S->emit, &zero, sizeof(int32_t),
                                   cudaMemcpyHostToDevice, st));
  }
  KRB_CHECK_CUDA(cudaMemcpyAsync(&hs, h.S, sizeof(hs), cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  *h_status = hs.status;
  H->hs = hs;
  H->hs_valid = true;
  return KRB_OK;
}

/* Launch the iterations up to the next completed cycle (or the end of the
 * solve) WITHOUT waiting: graph / persistent drivers only (the host loop
 * needs a read-back per iteration, so there it runs to the pause here).
 * The caller may queue more work on the stream (the harvest of the previous
 * cycle) and then collects the state with krb_rbicg_wait.  *launched = 0
 * when the solve had already stopped (nothing queued). */
int krb_rbicg_launch(krb_rbicg *H, int32_t *launched, void *stream) {
  KRB_REQUIRE(H && launched, "krb_rbicg_launch: NULL argument");
  cudaStream_t st = as_stream(stream);
  *launched = 0;
  BiScalars hs;
  if (H->hs_valid) {
    hs = H->hs;
  } else {
    KRB_CHECK_CUDA(cudaMemcpyAsync(&hs, H->h.S, sizeof(hs), cudaMemcpyDeviceToHost, st));
    KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  }
  if (hs.status != KRB_RUNNING) return KRB_OK;
  KRB_CHECK_CUDA(cudaMemsetAsync(&H->h.S->emit, 0, sizeof(int32_t), st));
  if (H->use_graph == 1) {
    KRB_CHECK_CUDA(cudaGraphLaunch(H->exec, st));
  } else if (H->use_graph == 2) {
    KRB_TRY(bi_persistent(H->h, H->d_nc, st));
  } else {
    for (int64_t it = 0; it <= H->max_itn; ++it) {
      KRB_TRY(bi_iteration(H->h, H->d_nc, st));
      KRB_CHECK_CUDA(cudaMemcpyAsync(&hs, H->h.S, sizeof(hs), cudaMemcpyDeviceToHost, st));
      KRB_CHECK_CUDA(cudaStreamSynchronize(st));
      if (hs.status != KRB_RUNNING || hs.emit) break;
    }
  }
  H->hs_valid = false;   // the device block moves on; krb_rbicg_wait re-reads it
  *launched = 1;
  return KRB_OK;
}

/* Wait for the stream and read the scalar state.
 * h_state[0..6] = status, emit, ncols, itn, nalpha, capture, npush. */
int krb_rbicg_wait(krb_rbicg *H, int64_t *h_state, void *stream) {
  KRB_REQUIRE(H && h_state, "krb_rbicg_wait: NULL argument");
  cudaStream_t st = as_stream(stream);
  BiScalars hs;
  if (H->hs_valid) {
    hs = H->hs;
  } else {
    KRB_CHECK_CUDA(cudaMemcpyAsync(&hs, H->h.S, sizeof(hs), cudaMemcpyDeviceToHost, st));
    KRB_CHECK_CUDA(cudaStreamSynchronize(st));
    H->hs = hs;
    H->hs_valid = true;
  }
  h_state[0] = hs.status;
  h_state[1] = hs.emit;
  h_state[2] = hs.ncols;
  h_state[3] = hs.itn;
  h_state[4] = hs.nalpha;
  h_state[5] = hs.capture;
  h_state[6] = hs.npush;
  return KRB_OK;
}

/* Run iterations until the solve stops or a cycle completes (launch + wait).
 * h_state[0..6] = status, emit, ncols, itn, nalpha, capture, npush. */
int krb_rbicg_run(krb_rbicg *H, int64_t *h_state, void *stream) {
  KRB_REQUIRE(H && h_state, "krb_rbicg_run: NULL argument");
  int32_t launched = 0;
  KRB_TRY(krb_rbicg_launch(H, &launched, stream));
  return krb_rbicg_wait(H, h_state, stream);
}

/* Device pointers of the capture rings and coefficient arrays (read-only
 * views for the host emit logic): V, Vt (ring_ld = n), rhos, alphas, betas. */
int krb_rbicg_views(krb_rbicg *H, double **V, double **Vt, double **rhos,
                    double **alphas, double **betas) {
  KRB_REQUIRE(H, "krb_rbicg_views: NULL handle");
  *V = H->h.V;
  *Vt = H->h.Vt;
  *rhos = H->h.rhos;
  *alphas = H->h.alphas;
  *betas = H->h.betas;
  return KRB_OK;
}

/* After an emit: keep the last `keep` ring columns at the front
 * (solvers.py:555-558) and continue. */
int krb_rbicg_rotate(krb_rbicg *H, int64_t keep, void *stream) {
  KRB_REQUIRE(H, "krb_rbicg_rotate: NULL handle");
  cudaStream_t st = as_stream(stream);
  BiScalars hs;
  if (H->hs_valid) {
    hs = H->hs;
  } else {
    KRB_CHECK_CUDA(cudaMemcpyAsync(&hs, H->h.S, sizeof(hs), cudaMemcpyDeviceToHost, st));
    KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  }
  const int64_t n = H->h.n, nc = hs.ncols;
  KRB_REQUIRE(keep >= 0 && keep <= nc, "krb_rbicg_rotate: keep > ncols");
  KRB_REQUIRE(keep < 256, "krb_rbicg_rotate: keep >= 256");
  for (int64_t c = 0; c < keep; ++c) {
    int64_t src = nc - keep + c;
    if (src == c) continue;
    KRB_CHECK_CUDA(cudaMemcpyAsync(H->h.V + c * n, H->h.V + src * n, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
    KRB_CHECK_CUDA(cudaMemcpyAsync(H->h.Vt + c * n, H->h.Vt + src * n, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
  }
  // ncols = keep without a pageable host->device copy (which may
  // synchronise): zero the int64, then its low byte (little-endian)
  KRB_CHECK_CUDA(cudaMemsetAsync(&H->h.S->ncols, 0, sizeof(int64_t), st));
  if (keep) KRB_CHECK_CUDA(cudaMemsetAsync(&H->h.S->ncols, (int)keep, 1, st));
  if (H->hs_valid) H->hs.ncols = keep;
  return KRB_OK;
}

/* Finish: x_out = x - U zc, xt_out = xt - Ut ztc, true residual; history to
 * the caller's device arrays (length >= max_itn + 2). */
int krb_rbicg_finish(krb_rbicg *H, double *d_x_out, double *d_xt_out,
                     double *d_hist_r, double *d_hist_rt, int64_t *d_hist_m,
                     uint64_t *d_hist_t, krb_solve_result *res,
                     int64_t *h_counts, double *h_btnorm, void *stream) {
  KRB_REQUIRE(H && d_x_out && d_xt_out && res && h_counts && h_btnorm,
              "krb_rbicg_finish: NULL argument");
  cudaStream_t st = as_stream(stream);
  BiArgs &h = H->h;
  const int64_t n = h.n, k = h.k;
  if (k > 0) {
    KRB_TRY(launch_gemv(n, k, H->R.U, H->R.ld, h.zc, h.x, -1, d_x_out, st));
    KRB_TRY(launch_gemv(n, k, H->R.Ut, H->R.ld, h.ztc, h.xt, -1, d_xt_out, st));
  } else {
    KRB_CHECK_CUDA(cudaMemcpyAsync(d_x_out, h.x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    KRB_CHECK_CUDA(cudaMemcpyAsync(d_xt_out, h.xt, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
  KRB_TRY(spmv_launch(H->A, d_x_out, h.q, nullptr, st));
  KRB_TRY(bi_launch<BP_TRUE>(h, H->d_nc, st));
  BiScalars hs;
  KRB_CHECK_CUDA(cudaMemcpyAsync(&hs, h.S, sizeof(hs), cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  const int64_t L = hs.hist_len;
  if (L > 0) {
    KRB_CHECK_CUDA(cudaMemcpyAsync(d_hist_r, h.hist_r, sizeof(double) * L, cudaMemcpyDeviceToDevice, st));
    KRB_CHECK_CUDA(cudaMemcpyAsync(d_hist_rt, h.hist_rt, sizeof(double) * L, cudaMemcpyDeviceToDevice, st));
    KRB_CHECK_CUDA(cudaMemcpyAsync(d_hist_m, h.hist_m, sizeof(int64_t) * L, cudaMemcpyDeviceToDevice, st));
    KRB_CHECK_CUDA(cudaMemcpyAsync(d_hist_t, h.hist_t, sizeof(uint64_t) * L, cudaMemcpyDeviceToDevice, st));
  }
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  res->status = hs.status;
  res->hist_len = L;
  res->matvecs = hs.n_matvec + hs.n_rmatvec;
  res->rhs_norm = hs.bnorm;
  res->final_true_resid = hs.final_true_resid;
  res->t_start_ns = hs.t_start;
  res->iterations_run = hs.bodies;
  if (H->use_graph == 1) launch_counter() += hs.bodies * H->per_body;
  res->kernel_launches = launch_counter() - H->l0;
  res->driver = H->use_graph == 2 ? KRB_DRIVER_PERSISTENT
                : (H->use_graph == 1 ? KRB_DRIVER_GRAPH : KRB_DRIVER_HOST_LOOP);
  h_counts[0] = hs.n_matvec;
  h_counts[1] = hs.n_rmatvec;
  *h_btnorm = hs.btnorm;
  return KRB_OK;
}

}  // extern "C"
