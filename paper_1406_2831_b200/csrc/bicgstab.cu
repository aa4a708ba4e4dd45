// Deflated BiCGSTAB (Algorithm 2 of arXiv 1406.2831) on sm_100a.
//
// Restates rbicgstab_solve (reference solvers.py:245-361; bicgstab_solve
// solvers.py:156-242 is the k = 0 case) as a short chain of fused,
// HBM-streaming phase kernels.  All scalar logic (alpha, omega, beta, rho,
// breakdown and convergence predicates, history records) runs on the device
// in the last CTA of the kernel that produced the reduction it needs, in
// exactly the reference's order, so one iteration needs no host round trip.
// The iteration is captured once into a CUDA graph whose WHILE conditional
// node is re-armed by the device (cudaGraphSetConditional) until the status
// leaves RUNNING: a whole solve is one graph launch plus one final readback.
//
// Per iteration (k > 0; the projection kernels vanish for k = 0):
//   P  p = r + beta (p - omega q)                       stream 3 read, 1 write
//   M  q = A p                                          SpMV
//   Z  zeta = Chat^T q  (block partials + final)        n x k read
//   Q  q -= C zeta ; (rt0,q), (q,q) -> den, alpha        n x k + 3 read, 1 write
//   S  s = r - alpha q ; (s,s) -> half-step exit          2 read, 1 write
//   E  early exit only: x += alpha p, xc += alpha zeta
//   M  t = A s ; Z gamma = Chat^T t
//   T  t -= C gamma ; (t,t), (t,s) -> omega              n x k + 2 read, 1 write
//   X  x = x + alpha p + omega s ; r = s - omega t ;
//      (r,r), (rt0,r) -> record, converge, rho, beta     5 read, 2 write
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace krb {

enum Phase {
  PH_PUPDATE = 0,
  PH_PROJ_Q,
  PH_SUPD,
  PH_EARLY,
  PH_PROJ_T,
  PH_XR,
  PH_BNORM,
  PH_INIT,
  PH_TRUE,
  PH_RINIT,
};

struct IterArgs {
  int64_t n, nb, ld;
  int k;
  const double *C, *Chat, *U;
  double *x, *r, *p, *q, *s, *t, *rt0, *b;
  double *zeta, *gamma, *xc;
  double *part;
  unsigned int *counters;
  SolveScalars *S;
  double *hist_r;
  int64_t *hist_m;
  uint64_t *hist_t;
  cudaGraphConditionalHandle cond;
  int use_cond;
};

__device__ __forceinline__ void record(const IterArgs &a, double rn) {
  SolveScalars *S = a.S;
  int64_t h = S->hist_len;
  a.hist_r[h] = rn;
  a.hist_m[h] = S->matvecs;
  a.hist_t[h] = globaltimer();
  S->hist_len = h + 1;
}

template <int PH>
__host__ __device__ constexpr int ndots_of() {
  switch (PH) {
    case PH_PROJ_Q: return 2;
    case PH_SUPD: return 1;
    case PH_PROJ_T: return 2;
    case PH_XR: return 2;
    case PH_BNORM: return 1;
    case PH_INIT: return 3;
    case PH_TRUE: return 2;
    default: return 0;
  }
}

// Scalar logic of each phase, executed by thread 0 of the last CTA after the
// dot products d[] are final.  Mirrors solvers.py:298-356 line by line.
template <int PH>
__device__ void finalize(const IterArgs &a, const double *d) {
  SolveScalars *S = a.S;
  if (PH == PH_BNORM) {
    S->bnorm = __dsqrt_rn(d[0]);
    S->tol_abs = __dmul_rn(S->tol_abs, S->bnorm);  // tol_abs held tol
  } else if (PH == PH_INIT) {
    double rn = __dsqrt_rn(d[0]);
    record(a, rn);
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
    if (fabs(den) <= __dmul_rn(__dmul_rn(S->breakdown_tol, S->nrt0), nq)) {
      S->status = KRB_BREAKDOWN_SERIOUS;
      S->itn += 1;
    } else {
      S->alpha = __ddiv_rn(S->rho, den);
    }
  } else if (PH == PH_SUPD) {
    double sn = __dsqrt_rn(d[0]);
    S->snorm = sn;
    if (sn <= S->tol_abs) {
      record(a, sn);
      S->early = 1;
      S->status = KRB_CONVERGED;
      S->itn += 1;
    }
  } else if (PH == PH_PROJ_T) {
    S->matvecs += 1;
    double tt = d[0];
    S->tt = tt;
    S->ts = d[1];
    if (tt == 0.0) {
      S->status = KRB_BREAKDOWN_OMEGA;
      S->itn += 1;
    } else {
      double om = __ddiv_rn(d[1], tt);
      if (om == 0.0) {
        S->status = KRB_BREAKDOWN_OMEGA;
        S->itn += 1;
      } else {
        S->omega = om;
      }
    }
  } else if (PH == PH_XR) {
    double rn = __dsqrt_rn(d[0]);
    S->rnorm = rn;
    record(a, rn);
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

template <int kE, int PH>
__global__ void __launch_bounds__(256) k_phase(IterArgs a) {
  __shared__ double coef[512];
  __shared__ double red[3][8];
  __shared__ int last_flag;
  SolveScalars *S = a.S;
  constexpr int ND = ndots_of<PH>();
  const bool gated = (PH != PH_BNORM && PH != PH_INIT && PH != PH_TRUE &&
                      PH != PH_RINIT);
  if (PH == PH_XR && blockIdx.x == 0 && threadIdx.x == 0) S->bodies += 1;
  if (PH == PH_EARLY) {
    if (S->early != 1) return;
  } else if (gated && S->status != KRB_RUNNING) {
    if (PH == PH_XR && blockIdx.x == 0 && threadIdx.x == 0) {
      if (S->early == 1) S->early = 2;  // half-step exit consumed
      if (a.use_cond) cudaGraphSetConditional(a.cond, 0);
    }
    return;
  }
  const double alpha = S->alpha, omega = S->omega, beta = S->beta;
  const int k = a.k;
  if (PH == PH_PROJ_Q || PH == PH_PROJ_T) {
    const double *src = PH == PH_PROJ_Q ? a.zeta : a.gamma;
    for (int j = threadIdx.x; j < k; j += blockDim.x) coef[j] = src[j];
    __syncthreads();
  }
  const int64_t n = a.n;
  for (int64_t blk = blockIdx.x; blk < a.nb; blk += gridDim.x) {
    const int64_t base = blk * (256 * kE) + threadIdx.x;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
#pragma unroll
    for (int e = 0; e < kE; ++e) {
      const int64_t i = base + 256 * e;
      if (i >= n) continue;
      if (PH == PH_PUPDATE) {
        // p = r + beta * (p - omega * q)          (solvers.py:303)
        double pv = __dsub_rn(a.p[i], __dmul_rn(omega, a.q[i]));
        a.p[i] = __dadd_rn(a.r[i], __dmul_rn(beta, pv));
      } else if (PH == PH_PROJ_Q || PH == PH_PROJ_T) {
        double *v = PH == PH_PROJ_Q ? a.q : a.t;
        double vi = v[i];
        if (k > 0) {
          double cz = 0.0;
          for (int j = 0; j < k; ++j)
            cz = __fma_rn(__ldg(a.C + (int64_t)j * a.ld + i), coef[j], cz);
          vi = __dsub_rn(vi, cz);   // q - C @ zeta   (solvers.py:307,329)
          v[i] = vi;
        }
        if (PH == PH_PROJ_Q) {
          acc0 = __fma_rn(a.rt0[i], vi, acc0);   // (rt0, q)
          acc1 = __fma_rn(vi, vi, acc1);         // (q, q)
        } else {
          acc0 = __fma_rn(vi, vi, acc0);         // (t, t)
          acc1 = __fma_rn(vi, a.s[i], acc1);     // (t, s)
        }
      } else if (PH == PH_SUPD) {
        // s = r - alpha * q                       (solvers.py:313)
        double sv = __dsub_rn(a.r[i], __dmul_rn(alpha, a.q[i]));
        a.s[i] = sv;
        acc0 = __fma_rn(sv, sv, acc0);
      } else if (PH == PH_EARLY) {
        // x = x + alpha * p                       (solvers.py:316)
        a.x[i] = __dadd_rn(a.x[i], __dmul_rn(alpha, a.p[i]));
      } else if (PH == PH_XR) {
        // x = x + alpha*p + omega*s ; r = s - omega*t   (solvers.py:338,341)
        double sv = a.s[i];
        double xv = __dadd_rn(__dadd_rn(a.x[i], __dmul_rn(alpha, a.p[i])),
                              __dmul_rn(omega, sv));
        a.x[i] = xv;
        double rv = __dsub_rn(sv, __dmul_rn(omega, a.t[i]));
        a.r[i] = rv;
        acc0 = __fma_rn(rv, rv, acc0);
        acc1 = __fma_rn(a.rt0[i], rv, acc1);
      } else if (PH == PH_BNORM) {
        double bv = a.b[i];
        acc0 = __fma_rn(bv, bv, acc0);
      } else if (PH == PH_INIT) {
        double rv = a.r[i], tv = a.rt0[i];
        acc0 = __fma_rn(rv, rv, acc0);
        acc1 = __fma_rn(tv, rv, acc1);
        acc2 = __fma_rn(tv, tv, acc2);
      } else if (PH == PH_TRUE) {
        // true residual b - A x_out   (solvers.py:147-153); A x_out in t
        double bv = a.b[i];
        double res = __dsub_rn(bv, a.t[i]);
        acc0 = __fma_rn(res, res, acc0);
        acc1 = __fma_rn(bv, bv, acc1);
      } else if (PH == PH_RINIT) {
        // r = b - A x_init            (recycling.py:200); A x_init in t
        a.r[i] = __dsub_rn(a.b[i], a.t[i]);
      }
    }
    if (ND > 0) {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      double w0 = warp_tree(acc0);
      double w1 = ND > 1 ? warp_tree(acc1) : 0.0;
      double w2 = ND > 2 ? warp_tree(acc2) : 0.0;
      if (lane == 0) {
        red[0][warp] = w0;
        if (ND > 1) red[1][warp] = w1;
        if (ND > 2) red[2][warp] = w2;
      }
      __syncthreads();
      if (threadIdx.x < ND) {
        double v8[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) v8[t] = red[threadIdx.x][t];
#pragma unroll
        for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
          for (int t = 0; t < off; ++t) v8[t] = __dadd_rn(v8[t], v8[t + off]);
        a.part[threadIdx.x * a.nb + blk] = v8[0];
      }
      __syncthreads();
    }
  }
  // xc updates of the k-vector ride on block 0 (no reduction needed)
  if (PH == PH_EARLY && blockIdx.x == 0) {
    for (int j = threadIdx.x; j < k; j += blockDim.x)
      a.xc[j] = __dadd_rn(a.xc[j], __dmul_rn(alpha, a.zeta[j]));
  }
  if (ND == 0) return;
  if (!elect_last_cta(a.counters + PH, &last_flag)) return;
  __shared__ double dfin[3];
  const int warp = threadIdx.x >> 5;
  if (warp < ND) {
    double v = warp_final_volatile(a.part + warp * a.nb, a.nb);
    if ((threadIdx.x & 31) == 0) dfin[warp] = v;
  }
  if (PH == PH_XR) {
    // xc = xc + alpha*zeta + omega*gamma     (solvers.py:340)
    for (int j = threadIdx.x; j < k; j += blockDim.x)
      a.xc[j] = __dadd_rn(__dadd_rn(a.xc[j], __dmul_rn(alpha, a.zeta[j])),
                          __dmul_rn(omega, a.gamma[j]));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    finalize<PH>(a, dfin);
    a.counters[PH] = 0;
    if (PH == PH_XR && a.use_cond)
      cudaGraphSetConditional(a.cond, S->status == KRB_RUNNING ? 1u : 0u);
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

template <int PH>
static int launch_phase(const IterArgs &a, cudaStream_t st) {
  if (a.nb == 0) return KRB_OK;
  int grid = grid_for(a.nb);
  switch (canon_E(a.n)) {
    case 1: k_phase<1, PH><<<grid, 256, 0, st>>>(a); break;
    case 2: k_phase<2, PH><<<grid, 256, 0, st>>>(a); break;
    case 4: k_phase<4, PH><<<grid, 256, 0, st>>>(a); break;
    case 8: k_phase<8, PH><<<grid, 256, 0, st>>>(a); break;
    default: k_phase<16, PH><<<grid, 256, 0, st>>>(a); break;
  }
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

#define KRB_TRY(x)          \
  do {                      \
    int rc_ = (x);          \
    if (rc_) return rc_;    \
  } while (0)

// one iteration (the graph body)
static int launch_iteration(krb_context *ctx, const krb_matrix *A,
                            const IterArgs &a, cudaStream_t st) {
  const int *status = &a.S->status;
  KRB_TRY(launch_phase<PH_PUPDATE>(a, st));
  KRB_TRY(spmv_launch(A, a.p, a.q, status, st));
  if (a.k > 0)
    KRB_TRY(launch_tdot(ctx, a.n, a.k, a.Chat, a.ld, a.q, false, a.zeta, status, st));
  KRB_TRY(launch_phase<PH_PROJ_Q>(a, st));
  KRB_TRY(launch_phase<PH_SUPD>(a, st));
  KRB_TRY(launch_phase<PH_EARLY>(a, st));
  KRB_TRY(spmv_launch(A, a.s, a.t, status, st));
  if (a.k > 0)
    KRB_TRY(launch_tdot(ctx, a.n, a.k, a.Chat, a.ld, a.t, false, a.gamma, status, st));
  KRB_TRY(launch_phase<PH_PROJ_T>(a, st));
  KRB_TRY(launch_phase<PH_XR>(a, st));
  return KRB_OK;
}

int ctx_reserve_vectors(krb_context *ctx, int64_t n, int64_t k) {
  if (n <= ctx->vec_n && k <= ctx->vec_k) return KRB_OK;
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
  ctx->vec_n = nn;
  ctx->vec_k = kk;
  ctx->graph.reset();
  return KRB_OK;
}

static int build_graph(krb_context *ctx, const krb_matrix *A, IterArgs a,
                       cudaStream_t capture) {
  GraphCache &G = ctx->graph;
  G.reset();
  cudaGraph_t g;
  KRB_CHECK_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  KRB_CHECK_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  KRB_CHECK_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  a.cond = h;
  a.use_cond = 1;
  KRB_CHECK_CUDA(cudaStreamBeginCaptureToGraph(capture, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeRelaxed));
  const int64_t c0 = launch_counter();
  int rc = launch_iteration(ctx, A, a, capture);
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
  const int64_t l0 = launch_counter();
  int64_t per_body = 0;
  const int64_t nb = canon_nblocks(n);
  KRB_TRY(ctx_reserve_part(ctx, (size_t)(3 * nb > k * nb ? 3 * nb : k * nb) + 64));
  if (!ctx->S) {
    KRB_CHECK_CUDA(cudaMalloc(&ctx->S, sizeof(SolveScalars)));
    KRB_CHECK_CUDA(cudaMalloc(&ctx->counters, sizeof(unsigned int) * 32));
    KRB_CHECK_CUDA(cudaMemsetAsync(ctx->counters, 0, sizeof(unsigned int) * 32, st));
  }
  IterArgs a = {};
  a.n = n;
  a.nb = nb;
  a.k = (int)k;
  a.ld = k > 0 ? R->ld : n;
  a.C = k > 0 ? R->C : nullptr;
  a.Chat = k > 0 ? R->Chat : nullptr;
  a.U = k > 0 ? R->U : nullptr;
  a.x = ctx->x; a.r = ctx->r; a.p = ctx->p; a.q = ctx->q; a.s = ctx->s;
  a.t = ctx->t; a.rt0 = ctx->rt0; a.b = ctx->b;
  a.zeta = ctx->kbuf;
  a.gamma = ctx->kbuf + ctx->vec_k;
  a.xc = ctx->kbuf + 2 * ctx->vec_k;
  double *ybuf = ctx->kbuf + 3 * ctx->vec_k;
  a.part = ctx->part;
  a.counters = ctx->counters;
  a.S = ctx->S;
  a.hist_r = hist_r;
  a.hist_m = hist_m;
  a.hist_t = hist_t;

  // ---- setup (solvers.py:257-296) -------------------------------------
  KRB_CHECK_CUDA(cudaMemcpyAsync(a.b, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  k_init_scalars<<<1, 1, 0, st>>>(a.S, cfg->tol, cfg->breakdown_tol, cfg->max_itn,
                                  (int)k, d_x_init ? 1 : 0);
  KRB_CHECK_LAUNCH();
  KRB_TRY(launch_phase<PH_BNORM>(a, st));
  // shadow residual rt_{-1} (solvers.py:268-269)
  if (cfg->d_shadow)
    KRB_CHECK_CUDA(cudaMemcpyAsync(ctx->w, cfg->d_shadow, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
  else
    KRB_TRY(krb_uniform_pcg64(n, cfg->pcg_state_hi, cfg->pcg_state_lo, cfg->pcg_inc_hi,
                              cfg->pcg_inc_lo, -1.0, 1.0, ctx->w, st));
  // x0, r0 (project_initial, recycling.py:189-206)
  if (d_x_init) {
    KRB_CHECK_CUDA(cudaMemcpyAsync(a.x, d_x_init, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
    KRB_TRY(spmv_launch(A, a.x, a.t, nullptr, st));
    KRB_TRY(launch_phase<PH_RINIT>(a, st));
  } else {
    KRB_CHECK_CUDA(cudaMemsetAsync(a.x, 0, sizeof(double) * n, st));
    KRB_CHECK_CUDA(cudaMemcpyAsync(a.r, a.b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
  if (k > 0) {
    KRB_TRY(launch_tdot(ctx, n, k, R->Chat, R->ld, a.r, false, ybuf, nullptr, st));
    KRB_TRY(launch_gemv(n, k, R->U, R->ld, ybuf, a.x, +1, a.x, st));
    KRB_TRY(launch_gemv(n, k, R->C, R->ld, ybuf, a.r, -1, a.r, st));
    // rt0 = rt_{-1} - Ct (Ccheck^H rt_{-1})   (solvers.py:273)
    KRB_TRY(launch_tdot(ctx, n, k, R->Ccheck, R->ld, ctx->w, false, ybuf, nullptr, st));
    KRB_TRY(launch_gemv(n, k, R->Ct, R->ld, ybuf, ctx->w, -1, a.rt0, st));
    KRB_CHECK_CUDA(cudaMemsetAsync(a.xc, 0, sizeof(double) * k, st));
  } else {
    KRB_CHECK_CUDA(cudaMemcpyAsync(a.rt0, ctx->w, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
  }
  KRB_CHECK_CUDA(cudaMemsetAsync(a.p, 0, sizeof(double) * n, st));
  KRB_CHECK_CUDA(cudaMemsetAsync(a.q, 0, sizeof(double) * n, st));
  KRB_TRY(launch_phase<PH_INIT>(a, st));

  // ---- iterations (solvers.py:298-356) --------------------------------
  if (cfg->use_graph == 1) {
    GraphCache &G = ctx->graph;
    bool hit = G.exec && G.A == A && G.n == n && G.k == k && G.ld == a.ld &&
               G.C == a.C && G.Chat == a.Chat && G.hist_r == hist_r &&
               G.hist_m == hist_m && G.hist_t == hist_t;
    if (!hit) {
      KRB_TRY(build_graph(ctx, A, a, capture_stream()));
      G.A = A; G.n = n; G.k = k; G.ld = a.ld; G.C = a.C; G.Chat = a.Chat;
      G.hist_r = hist_r; G.hist_m = hist_m; G.hist_t = hist_t;
    }
    KRB_CHECK_CUDA(cudaGraphLaunch(G.exec, st));
    per_body = G.kernels_per_body;
  } else {
    // host-driven loop, status polled every 8 iterations (kernels no-op once
    // the status leaves RUNNING, so the overshoot is harmless)
    int32_t status = 0;
    for (int64_t it = 0; it < cfg->max_itn + 1; ++it) {
      KRB_TRY(launch_iteration(ctx, A, a, st));
      if ((it & 7) == 7 || it == cfg->max_itn) {
        KRB_CHECK_CUDA(cudaMemcpyAsync(&status, &a.S->status, sizeof(int32_t),
                                       cudaMemcpyDeviceToHost, st));
        KRB_CHECK_CUDA(cudaStreamSynchronize(st));
        if (status != KRB_RUNNING) break;
      }
    }
  }

  // ---- x_out = x - U xc (solvers.py:359), true residual (:360) ----------
  if (k > 0)
    KRB_TRY(launch_gemv(n, k, R->U, R->ld, a.xc, a.x, -1, d_x_out, st));
  else
    KRB_CHECK_CUDA(cudaMemcpyAsync(d_x_out, a.x, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
  KRB_TRY(spmv_launch(A, d_x_out, a.t, nullptr, st));
  KRB_TRY(launch_phase<PH_TRUE>(a, st));
  SolveScalars hs;
  KRB_CHECK_CUDA(cudaMemcpyAsync(&hs, a.S, sizeof(SolveScalars), cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  res->status = hs.status;
  res->hist_len = hs.hist_len;
  res->matvecs = hs.matvecs;
  res->rhs_norm = hs.bnorm;
  res->final_true_resid = hs.final_true_resid;
  res->t_start_ns = hs.t_start;
  res->iterations_run = hs.bodies;
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
