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

#include <cstdlib>

#include "iter.cuh"
#include "spmv.cuh"
#include "tdot.cuh"

namespace krb {

// ---------------------------------------------------------------------------
// graph / host-loop driver: one kernel per phase, last CTA finalizes
// ---------------------------------------------------------------------------
// Register budget and element unroll per phase (kV = tuning "phase_variant"
// 0, measured on C5, same box, A/B): the projection updates Q / T keep up to
// 64 registers (one 1024-thread CTA per SM) and 4 elements in flight
// (702 us vs 739 at 32 registers); P, S and X run two CTAs per SM (at most 32
// registers): P with 4 elements unrolled (86 vs 104 us at 64 registers), S
// with 2 (73 vs 97), X with 1 (191 us; 205 with 2, 253 at 64 registers x 4).  kV = 1: every phase at 64
// registers / 4 elements (the round-1 kernels, kept for A/B); kV = 2: the
// record_iterates kernels (INIT / X with the snapshot stores); kV = 3: as 0
// with S / X unrolled once (A/B).  Same arithmetic, same bits.
__host__ __device__ constexpr int phase_minb(int PH, int kV) {
  return (kV == 1 || kV == 2) ? 1 : ((PH == PH_PROJ_Q || PH == PH_PROJ_T) ? 1 : 2);
}
__host__ __device__ constexpr int phase_unroll(int PH, int kV) {
  return (kV == 1 || kV == 2) ? 4
       : PH == PH_XR ? 1 : PH == PH_SUPD ? (kV == 3 ? 1 : 2) : 4;
}

template <int kE, int PH, int kV>
__global__ void __launch_bounds__(1024, phase_minb(PH, kV)) k_phase(const IterArgs *__restrict__ pa) {
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
  constexpr int kSlot = ktime_slot_of(PH);
  ktime_start(a, kSlot);
  if (PH == PH_PROJ_Q || PH == PH_PROJ_T) {
    const double *src = PH == PH_PROJ_Q ? a.zeta : a.gamma;
    for (int j = threadIdx.x; j < a.k; j += blockDim.x) coef[j] = src[j];
    __syncthreads();
  }
  phase_blocks<kE, PH, phase_unroll(PH, kV), kV == 2, true>(a, sc, red, coef, blockIdx.x, gridDim.x,
                                                      a.part);
  if (ND == 0) {
    ktime_finish(a, kSlot);
    return;
  }
  if (!elect_last_cta(a.counters + PH, &last_flag)) return;
  phase_leader<PH>(a, sc);
  if (PH == PH_XR && a.ktime && threadIdx.x < 32) ktime_fold_spmv(a);
  if (threadIdx.x == 0) {
    ktime_add(a, kSlot);
    a.counters[PH] = 0;
    if (PH == PH_XR && a.use_cond)
      cudaGraphSetConditional(a.cond, S->status == KRB_RUNNING ? 1u : 0u);
  }
}

// projection dots inside the iteration: Chat^T v -> zeta / gamma
// kV (tuning "tdot_variant"): 0 = up to 64 registers, 4 elements unrolled;
// 1 = at most 32 registers (two 1024-thread CTAs per SM), 2 elements;
// 3 = as 0 in groups of 4 columns over a 1-D grid of balanced unit ranges
// (automatic below kTdotSmallNb blocks: C3 256 blocks, 102 -> see DESIGN).
// (Measured dead end, C5: guard-free full blocks with the next element's
// loads issued before the current fmas over balanced 1-D unit ranges,
// 669 vs 632 us.)
template <int kE, bool kGamma, int kV>
__global__ void __launch_bounds__(1024, kV == 1 ? 2 : 1) k_proj_dot(const IterArgs *__restrict__ pa) {
  const IterArgs &a = *pa;
  if (a.S->status != KRB_RUNNING) return;
  ktime_start(a, kGamma ? 6 : 2);
  tdot_body<kE, false, false, kV == 1 ? 2 : 4, kV == 3 ? 4 : kTdotCG>(
      a.n, a.nb, a.k, a.Chat, a.ld, kGamma ? a.t : a.q, a.part, kGamma ? a.gamma : a.zeta,
      a.counters + kCounterTdotGraph, a.l2keep != 0);
  ktime_finish(a, kGamma ? 6 : 2);
}

constexpr int64_t kTdotSmallNb = 4 * kNumSMs;

// SpMV inside the iteration: one row per thread, the matrix, x, y and the
// status word as kernel parameters (constant bank operands, as the
// standalone k_spmv), so no thread chases the descriptor before its first
// matrix load.  The graph bakes these parameters; rbicgstab re-captures it
// when the matrix (or the kernel-timing buffer) differs from the captured
// one.  (Reading them through the descriptor: 1025 us per C5 launch vs
// 898 us for the same rows with parameters; broadcasting them through shared
// memory costs 48 registers; a grid-stride variant with 6 x 148 CTAs:
// 1258 us.)
// kF: 0 CSR, 1 SELL-32 / SELL-C-sigma, 2 offset-coded SELL-32 (uniform
// slices: offsets by warp shuffle), 3 its first version (tuning spmv_variant=1),
// 4 value-coded (constant diagonals from the row templates), 5 value-coded in
// diagonal form (table in the matrix argument).
template <int kF, int kSlot, int kMinB = 1, int kBU = 4>
__global__ void __launch_bounds__(256, kMinB) k_iter_spmv(krb_matrix A, const double *__restrict__ x,
                                                   double *__restrict__ y,
                                                   const int *__restrict__ status,
                                                   uint64_t *__restrict__ kt, int64_t pf) {
  constexpr bool kSell = kF == 1;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (kF >= 2) {
    // the status word is consumed only at the store (no dependent round
    // trip before the first matrix load of every CTA); after a half-step
    // exit (status set by S) the product of a finished solve is discarded
    const int run = __ldg(status);
    if (kt && blockIdx.x == 0 && threadIdx.x == 0 && run == KRB_RUNNING)
      *(volatile uint64_t *)&kt[4 * kSlot] = globaltimer();
    if (i < A.n) {
      auto xf = [x](int c) { return __ldg(x + c); };
      double yi;
      if (kF == 5)
        yi = spmv_row_dia(i, A, x);
      else if (kF == 4)
        yi = spmv_row_tmpl(i, A, xf);
      else
        yi = spmv_row_dict<kF == 3 ? 1 : 0, decltype(xf), kBU>(i, A, xf, pf);
      if (run == KRB_RUNNING) y[i] = yi;
    }
    if (run != KRB_RUNNING) return;
  } else {
    if (*status != KRB_RUNNING) return;
    if (kt && blockIdx.x == 0 && threadIdx.x == 0)
      *(volatile uint64_t *)&kt[4 * kSlot] = globaltimer();
    if (i < A.n) y[(kSell && A.perm) ? A.perm[i] : i] = spmv_row<kSell>(i, A, x);
  }
  if (kt && blockIdx.x + 4096u >= gridDim.x) {
    // per-SM end stamp (iter.cuh ktime_end_spmv), from the CTAs of the last
    // ~4 waves only (the kernel's end is among them; an atomic from every
    // one of 65536 CTAs cost ~2 % of the iteration)
    __syncthreads();
    if (threadIdx.x == 0)
      atomicMax((unsigned long long *)&kt[kKtSpmvBase + kKtSmSlots * (kSlot == 5 ? 1 : 0) + smid()],
                (unsigned long long)globaltimer());
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
static int launch_phase(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  if (h.nb == 0) return KRB_OK;
  // 2 x 148 CTAs even where only one fits per SM: the second wave balances
  // the blocks dynamically (one wave of 148: Q / T 702 -> 776 us on C5)
  int grid = grid_for(h.nb);
  if (h.rec_x && (PH == PH_INIT || PH == PH_XR)) {   // record_iterates snapshots
    KRB_DISPATCH_E(canon_E(h.n), (k_phase<kE, PH, 2><<<grid, 1024, 0, st>>>(d)));
  } else if (tuning().phase_variant == 1) {
    KRB_DISPATCH_E(canon_E(h.n), (k_phase<kE, PH, 1><<<grid, 1024, 0, st>>>(d)));
  } else if (tuning().phase_variant == 3) {
    KRB_DISPATCH_E(canon_E(h.n), (k_phase<kE, PH, 3><<<grid, 1024, 0, st>>>(d)));
  } else {
    KRB_DISPATCH_E(canon_E(h.n), (k_phase<kE, PH, 0><<<grid, 1024, 0, st>>>(d)));
  }
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

template <bool kGamma>
static int launch_proj_dot(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  if (h.k <= 0 || h.nb == 0) return KRB_OK;
  const int tv = tuning().tdot_variant;
  if (tv == 3 || (tv == 0 && h.nb < kTdotSmallNb)) {
    static int per_sm3 = occupancy_1024(k_proj_dot<16, kGamma, 3>);
    const int64_t units = h.nb * ((h.k + 3) / 4);
    const int64_t g = (int64_t)kNumSMs * per_sm3 < units ? (int64_t)kNumSMs * per_sm3 : units;
    KRB_DISPATCH_E(canon_E(h.n), (k_proj_dot<kE, kGamma, 3><<<dim3((unsigned)g, 1), 1024, 0, st>>>(d)));
  } else if (tv == 1) {
    static int per_sm1 = occupancy_1024(k_proj_dot<16, kGamma, 1>);
    dim3 grid = tdot_grid(h.nb, h.k, per_sm1);
    KRB_DISPATCH_E(canon_E(h.n), (k_proj_dot<kE, kGamma, 1><<<grid, 1024, 0, st>>>(d)));
  } else {
    static int per_sm0 = occupancy_1024(k_proj_dot<16, kGamma, 0>);
    dim3 grid = tdot_grid(h.nb, h.k, per_sm0);
    KRB_DISPATCH_E(canon_E(h.n), (k_proj_dot<kE, kGamma, 0><<<grid, 1024, 0, st>>>(d)));
  }
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

template <bool kSecond>
static int launch_iter_spmv(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  if (h.n == 0) return KRB_OK;
  if (h.A.pre)   // split-ILUTP operator: the composite kernels (precond.cu)
    return spmv_launch(&h.A, kSecond ? h.s : h.p, kSecond ? h.t : h.q,
                       reinterpret_cast<const int *>(&h.S->status), st);
  unsigned blocks = (unsigned)((h.n + 255) / 256);
  const int *status = reinterpret_cast<const int *>(&h.S->status);
  const double *x = kSecond ? h.s : h.p;
  double *y = kSecond ? h.t : h.q;
  const int64_t pf = (int64_t)tuning().spmv_prefetch_mb << 20;
  // offset-coded: at most 40 registers (6 CTAs / SM; 47 unbounded, 5 CTAs:
  // 776 vs 746 us live on C5; 32 registers spill: 776).  In-process A/B of
  // the iteration (profiles/r02_spmv_variants_ab2.jsonl): 4 entries per
  // batch at 40 registers 4666 us, at 48: 4743; 8 entries at 48 / 60
  // registers: 4706 / 4969; the int4-offset version: 4666 (median 4783).
  if (h.A.tent && tuning().value_coding && h.A.dia.nd && tuning().value_coding != 2)
    k_iter_spmv<5, kSecond ? 5 : 1, 6><<<blocks, 256, 0, st>>>(h.A, x, y, status, h.ktime, 0);
  else if (h.A.tent && tuning().value_coding)
    k_iter_spmv<4, kSecond ? 5 : 1, 4><<<blocks, 256, 0, st>>>(h.A, x, y, status, h.ktime, 0);
  else if (h.A.dcode && tuning().spmv_variant == 1)
    k_iter_spmv<3, kSecond ? 5 : 1, 6><<<blocks, 256, 0, st>>>(h.A, x, y, status, h.ktime, pf);
  else if (h.A.dcode)
    k_iter_spmv<2, kSecond ? 5 : 1, 6><<<blocks, 256, 0, st>>>(h.A, x, y, status, h.ktime, pf);
  else if (h.A.format == 2)
    k_iter_spmv<1, kSecond ? 5 : 1><<<blocks, 256, 0, st>>>(h.A, x, y, status, h.ktime, 0);
  else
    k_iter_spmv<0, kSecond ? 5 : 1><<<blocks, 256, 0, st>>>(h.A, x, y, status, h.ktime, 0);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

// one iteration (the graph body).  (Programmatic dependent launches of
// kernels 2..9 -- CTAs starting in the previous kernel's tail, waiting on
// griddepcontrol -- measured no faster on C5: 4484-4518 vs 4468-4494 us.)
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

int launch_persistent(const IterArgs &h, const IterArgs *d, cudaStream_t st, int *driver);


int ctx_reserve_vectors(krb_context *ctx, int64_t n, int64_t k) {
  if (n <= ctx->vec_n && k <= ctx->vec_k && ctx->desc) return KRB_OK;
  double **vecs[] = {&ctx->x, &ctx->r, &ctx->p, &ctx->q, &ctx->s,
                     &ctx->t, &ctx->rt0, &ctx->b, &ctx->w, &ctx->p2, &ctx->q2};
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
  KRB_CHECK_CUDA(cudaGraphUpload(exec, capture));
  KRB_CHECK_CUDA(cudaStreamSynchronize(capture));
  return KRB_OK;
}

// Per-solve setup (solvers.py:257-296) for the solve described by h / d (the
// device descriptor must already hold h): scalars, ||b||, shadow residual,
// x0 / r0 (project_initial), rt0 projection, INIT.  w: n-vector scratch for
// the shadow residual, ybuf: k-vector scratch.  Stream-ordered, no sync.
int solve_setup(krb_context *ctx, const krb_matrix *A, const double *d_b,
                const double *d_x_init, const krb_space_view *R,
                const krb_solve_config *cfg, const IterArgs &h, const IterArgs *d,
                double *w, double *ybuf, cudaStream_t st) {
  const int64_t n = h.n, k = h.k;
  KRB_CHECK_CUDA(cudaMemcpyAsync(h.b, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  k_init_scalars<<<1, 1, 0, st>>>(h.S, cfg->tol, cfg->breakdown_tol, cfg->max_itn,
                                  (int)k, d_x_init ? 1 : 0);
  KRB_CHECK_LAUNCH();
  KRB_TRY(launch_phase<PH_BNORM>(h, d, st));
  // shadow residual rt_{-1} (solvers.py:268-269)
  if (cfg->d_shadow)
    KRB_CHECK_CUDA(cudaMemcpyAsync(w, cfg->d_shadow, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
  else
    KRB_TRY(krb_uniform_pcg64(n, cfg->pcg_state_hi, cfg->pcg_state_lo, cfg->pcg_inc_hi,
                              cfg->pcg_inc_lo, -1.0, 1.0, w, st));
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
    KRB_TRY(launch_tdot(ctx, n, k, R->Ccheck, R->ld, w, false, ybuf, nullptr, st));
    KRB_TRY(launch_gemv(n, k, R->Ct, R->ld, ybuf, w, -1, h.rt0, st));
    KRB_CHECK_CUDA(cudaMemsetAsync(h.xc, 0, sizeof(double) * k, st));
  } else {
    KRB_CHECK_CUDA(cudaMemcpyAsync(h.rt0, w, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
  }
  KRB_CHECK_CUDA(cudaMemsetAsync(h.p, 0, sizeof(double) * n, st));
  KRB_CHECK_CUDA(cudaMemsetAsync(h.q, 0, sizeof(double) * n, st));
  KRB_TRY(launch_phase<PH_INIT>(h, d, st));

  return KRB_OK;
}

// x_out = x - U xc (solvers.py:359) and the final true residual (:360);
// stream-ordered, no sync.
int solve_tail(const krb_matrix *A, const krb_space_view *R, const IterArgs &h,
               const IterArgs *d, double *d_x_out, cudaStream_t st) {
  const int64_t n = h.n, k = h.k;
  if (k > 0)
    KRB_TRY(launch_gemv(n, k, R->U, R->ld, h.xc, h.x, -1, d_x_out, st));
  else
    KRB_CHECK_CUDA(cudaMemcpyAsync(d_x_out, h.x, sizeof(double) * n,
                                   cudaMemcpyDeviceToDevice, st));
  KRB_TRY(spmv_launch(A, d_x_out, h.t, nullptr, st));
  KRB_TRY(launch_phase<PH_TRUE>(h, d, st));
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
  const size_t part_one = (size_t)((k + 3) * nb) + 64;
  KRB_TRY(ctx_reserve_part(ctx, 2 * part_one + 16 * 160));   // + per-CTA flags (<= 160 CTAs)
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
  h.p2 = ctx->p2; h.q2 = ctx->q2;
  h.zeta = ctx->kbuf;
  h.gamma = ctx->kbuf + ctx->vec_k;
  h.xc = ctx->kbuf + 2 * ctx->vec_k;
  double *ybuf = ctx->kbuf + 3 * ctx->vec_k;
  h.part = ctx->part;
  h.part2 = ctx->part + part_one;
  h.flags = reinterpret_cast<unsigned int *>(ctx->part + 2 * part_one);
  h.counters = ctx->counters;
  h.S = ctx->S;
  h.hist_r = hist_r;
  h.hist_m = hist_m;
  h.hist_t = hist_t;
  h.prof = cfg->d_phase_stamps;
  h.prof_cap = cfg->d_phase_stamps ? cfg->phase_stamps_cap : 0;
  h.ktime = cfg->d_kernel_times;
  if (cfg->d_rec_x) {
    KRB_REQUIRE(cfg->use_graph == 0, "record_iterates needs the host-loop driver");
    KRB_REQUIRE(cfg->d_rec_r && cfg->d_rec_s && cfg->d_rec_t && cfg->d_rec_omega &&
                    (k == 0 || cfg->d_rec_xc),
                "record_iterates: NULL snapshot buffer");
    h.rec_x = cfg->d_rec_x; h.rec_r = cfg->d_rec_r; h.rec_xc = cfg->d_rec_xc;
    h.rec_s = cfg->d_rec_s; h.rec_t = cfg->d_rec_t; h.rec_omega = cfg->d_rec_omega;
  }
  // 0 host loop, 1 graph, 2 persistent; a preconditioned operator runs the
  // graph (its products are kernel sequences the fused kernels do not have)
  const int mode = (A->pre && cfg->use_graph == 2) ? 1 : cfg->use_graph;
  const bool graph = mode == 1;
  GraphCache &G = ctx->graph;
  const MatrixSig sig = matrix_sig(A);
  const bool hit = graph && G.exec && G.n == n && G.k == k && same_sig(G.sig, sig) &&
                   G.ktime == cfg->d_kernel_times &&
                   G.variant == tuning().phase_variant + 16 * tuning().tdot_variant +
                                    256 * tuning().spmv_variant +
                                    4096 * tuning().spmv_prefetch_mb +
                                    (1 << 24) * tuning().value_coding;
  h.use_cond = graph ? 1 : 0;
  {
    // evict_last for the recycle blocks (and evict_first for the matrix
    // entries in the fused kernel) when C and Chat fit in about 3/4 of the
    // L2 (tuning "l2keep" = 0 / 1 overrides)
    const int e = tuning().l2keep;
    h.l2keep = e >= 0 ? e : (2.0 * 8.0 * (double)n * (double)k <= 100e6 ? 1 : 0);
    h.pf_rows = tuning().phase_pf_rows;
  }
  h.cond = hit ? G.cond : 0;
  IterArgs *d = reinterpret_cast<IterArgs *>(ctx->desc);

  // ---- setup (solvers.py:257-296) -------------------------------------
  if (graph && !hit) {
    KRB_CHECK_CUDA(cudaStreamSynchronize(st));
    KRB_TRY(build_graph(ctx, h, d, capture_stream()));
    G.n = n; G.k = k; G.format = A->format; G.sig = sig;
    G.ktime = cfg->d_kernel_times;
    G.variant = tuning().phase_variant + 16 * tuning().tdot_variant +
                256 * tuning().spmv_variant + 4096 * tuning().spmv_prefetch_mb +
                (1 << 24) * tuning().value_coding;
    h.cond = G.cond;
  }
  // the descriptor is written in stream order (the previous solve on this
  // stream has finished reading it)
  KRB_CHECK_CUDA(cudaMemcpyAsync(d, &h, sizeof(IterArgs), cudaMemcpyHostToDevice, st));
  KRB_TRY(solve_setup(ctx, A, d_b, d_x_init, R, cfg, h, d, ctx->w, ybuf, st));

  // ---- iterations (solvers.py:298-356) --------------------------------
  int driver = mode == 1 ? KRB_DRIVER_GRAPH : KRB_DRIVER_HOST_LOOP;
  if (mode == 2) {
    KRB_TRY(launch_persistent(h, d, st, &driver));
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

  KRB_TRY(solve_tail(A, R, h, d, d_x_out, st));
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
  res->driver = driver;
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
