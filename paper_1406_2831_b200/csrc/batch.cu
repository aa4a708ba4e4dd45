// Multi-right-hand-side RBiCGSTAB: up to kMaxB
// independent solves with the SAME matrix and the SAME recycle space advance
// in lockstep, so each iteration reads the matrix and the n x k blocks C /
// Chat once for all of them instead of once per right-hand side (C3: four
// right-hand sides per matrix).
//
// Every right-hand side keeps its own vectors, scalars, status, shadow
// residual and history, and its arithmetic is exactly that of the single
// solve (same canonical blocks, same per-element order, same scalar logic):
// the results are bit-identical to kMaxB separate krb_rbicgstab calls.
// A right-hand side that stops (converged / breakdown / max_itn) drops out
// of the batch; the CUDA graph's WHILE node runs until none is left.
//
// Iteration body (graph kernels, reading per-RHS descriptors):
//   P   p_b = r_b + beta_b (p_b - omega_b q_b)          (no dots)
//   M   q_b = A p_b            one pass over the matrix rows, B gathers
//   Z   zeta_b = Chat^T q_b    one pass over Chat, B x 4-column units
//   Q   q_b -= C zeta_b; (rt0_b, q_b), (q_b, q_b)      one pass over C
//   S   s_b = r_b - alpha_b q_b; (s_b, s_b)
//   M   t_b = A s_b ;  Z gamma_b = Chat^T t_b
//   T   t_b -= C gamma_b; (t_b, t_b), (t_b, s_b)
//   X   x_b, r_b; (r_b, r_b), (rt0_b, r_b)
#include <cuda_runtime.h>

#include "iter.cuh"
#include "spmv.cuh"
#include "tdot.cuh"

namespace krb {

constexpr int kMaxB = 4;
constexpr int kBatMaxK = 128;   // recycle dimension limit of the batched path
constexpr int kBatCG = 4;       // projection columns per unit (x B rhs values)
constexpr int kBatCounter = 32; // election counters: kBatCounter + PH, +9 proj

struct BatArgs {
  IterArgs *a;        // [nrhs] device descriptors
  int nrhs;
  int use_cond;
  cudaGraphConditionalHandle cond;
  unsigned int *counters;
};

// ---- per-RHS status snapshot (shared memory) ------------------------------
struct BatState {
  int run[kMaxB];
  int half[kMaxB];
  PhaseScal sc[kMaxB];
  int any;
};

__device__ __forceinline__ void load_state(const BatArgs &B, BatState &st) {
  if (threadIdx.x < kMaxB) {
    const int b = threadIdx.x;
    int run = 0, half = 0;
    PhaseScal sc = {0.0, 0.0, 0.0};
    if (b < B.nrhs) {
      const SolveScalars *S = B.a[b].S;
      run = S->status == KRB_RUNNING;
      half = (!run && S->early == 1);
      sc = load_scal(S);
    }
    st.run[b] = run;
    st.half[b] = half;
    st.sc[b] = sc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int any = 0;
    for (int b = 0; b < kMaxB; ++b) any |= st.run[b];
    st.any = any;
  }
  __syncthreads();
}

// canonical block stage for up to 8 values (rhs b, dot d) -> part_b rows
template <int ND>
__device__ __forceinline__ void bat_block_stage(const BatArgs &B, double (&acc)[kMaxB][2],
                                                double (*red)[32], int64_t blk) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = 0.0;
#pragma unroll
  for (int b = 0; b < kMaxB; ++b)
#pragma unroll
    for (int d = 0; d < ND; ++d) v[b * ND + d] = acc[b][d];
  int col;
  double w = warp_tree_multi<8>(v, col);
  if ((lane & 3) == 0) red[col][warp] = w;
  __syncthreads();
  if (warp < B.nrhs * ND) {
    const int b = warp / ND, d = warp - b * ND;
    double r = warp_tree(red[warp][lane]);
    if (lane == 0) B.a[b].part[d * B.a[b].nb + blk] = r;
  }
  __syncthreads();
}

template <int kE, int PH>
__global__ void __launch_bounds__(1024) k_bat_phase(const BatArgs *__restrict__ pb) {
  constexpr int ND = ndots_of(PH);
  constexpr bool kProj = PH == PH_PROJ_Q || PH == PH_PROJ_T;
  __shared__ double coef[kMaxB][kBatMaxK];
  __shared__ double red[8][32];
  __shared__ double dfin[kMaxB][3];
  __shared__ int last_flag;
  __shared__ BatState st;
  const BatArgs &B = *pb;
  const IterArgs &a0 = B.a[0];
  const int64_t n = a0.n, nb = a0.nb, ld = a0.ld;
  const int k = a0.k;
  if (PH == PH_XR && blockIdx.x == 0 && threadIdx.x < B.nrhs) B.a[threadIdx.x].S->bodies += 1;
  load_state(B, st);
  if (PH == PH_PUPDATE && blockIdx.x == 0 && threadIdx.x < B.nrhs) {
    // a half-step exit applied by the previous X phase: mark it consumed
    SolveScalars *S = B.a[threadIdx.x].S;
    if (S->status != KRB_RUNNING && S->early == 1) S->early = 2;
  }
  int anyhalf = 0;
#pragma unroll
  for (int b = 0; b < kMaxB; ++b) anyhalf |= st.half[b];
  if (!st.any) {
    if (PH == PH_XR) {
      for (int b = 0; b < B.nrhs; ++b)
        if (st.half[b]) half_exit_update(B.a[b], st.sc[b].alpha, blockIdx.x, gridDim.x);
      if (blockIdx.x == 0 && threadIdx.x == 0 && B.use_cond) cudaGraphSetConditional(B.cond, 0);
    }
    return;
  }
  if (kProj) {
    for (int b = 0; b < B.nrhs; ++b) {
      const double *src = PH == PH_PROJ_Q ? B.a[b].zeta : B.a[b].gamma;
      for (int j = threadIdx.x; j < k; j += blockDim.x) coef[b][j] = st.run[b] ? src[j] : 0.0;
    }
    __syncthreads();
  }
  const double *__restrict__ Cm = a0.C;
  for (int64_t blk = blockIdx.x; blk < nb; blk += gridDim.x) {
    const int64_t base = blk * ((int64_t)kLanes * kE) + threadIdx.x;
    double acc[kMaxB][2];
#pragma unroll
    for (int b = 0; b < kMaxB; ++b) acc[b][0] = acc[b][1] = 0.0;
#pragma unroll(kE < 4 ? kE : 4)
    for (int e = 0; e < kE; ++e) {
      const int64_t i = base + (int64_t)kLanes * e;
      if (i >= n) continue;
      double cz[kMaxB] = {0.0, 0.0, 0.0, 0.0};
      if (kProj && k > 0) {
        // C read once for every rhs: sequential fma over the columns
        int j = 0;
        for (; j + 4 <= k; j += 4) {
          const double c0 = __ldg(Cm + (int64_t)j * ld + i);
          const double c1 = __ldg(Cm + (int64_t)(j + 1) * ld + i);
          const double c2 = __ldg(Cm + (int64_t)(j + 2) * ld + i);
          const double c3 = __ldg(Cm + (int64_t)(j + 3) * ld + i);
#pragma unroll
          for (int b = 0; b < kMaxB; ++b) {
            cz[b] = __fma_rn(c0, coef[b][j], cz[b]);
            cz[b] = __fma_rn(c1, coef[b][j + 1], cz[b]);
            cz[b] = __fma_rn(c2, coef[b][j + 2], cz[b]);
            cz[b] = __fma_rn(c3, coef[b][j + 3], cz[b]);
          }
        }
        for (; j < k; ++j) {
          const double c = __ldg(Cm + (int64_t)j * ld + i);
#pragma unroll
          for (int b = 0; b < kMaxB; ++b) cz[b] = __fma_rn(c, coef[b][j], cz[b]);
        }
      }
#pragma unroll
      for (int b = 0; b < kMaxB; ++b) {
        if (b >= B.nrhs || !st.run[b]) continue;
        const IterArgs &a = B.a[b];
        const PhaseScal sc = st.sc[b];
        if (PH == PH_PUPDATE) {
          double pv = __dsub_rn(a.p[i], __dmul_rn(sc.omega, a.q[i]));   // solvers.py:303
          a.p[i] = __dadd_rn(a.r[i], __dmul_rn(sc.beta, pv));
        } else if (kProj) {
          double *v = PH == PH_PROJ_Q ? a.q : a.t;
          double vi = v[i];
          if (k > 0) {
            vi = __dsub_rn(vi, cz[b]);   // q - C @ zeta   (solvers.py:307,329)
            v[i] = vi;
          }
          if (PH == PH_PROJ_Q) {
            acc[b][0] = __fma_rn(a.rt0[i], vi, acc[b][0]);   // (rt0, q)
            acc[b][1] = __fma_rn(vi, vi, acc[b][1]);         // (q, q)
          } else {
            acc[b][0] = __fma_rn(vi, vi, acc[b][0]);         // (t, t)
            acc[b][1] = __fma_rn(vi, a.s[i], acc[b][1]);     // (t, s)
          }
        } else if (PH == PH_SUPD) {
          const double sv = __dsub_rn(a.r[i], __dmul_rn(sc.alpha, a.q[i]));   // :313
          a.s[i] = sv;
          acc[b][0] = __fma_rn(sv, sv, acc[b][0]);
        } else if (PH == PH_XR) {
          const double sv = a.s[i];
          a.x[i] = __dadd_rn(__dadd_rn(a.x[i], __dmul_rn(sc.alpha, a.p[i])),
                             __dmul_rn(sc.omega, sv));                        // :338
          const double rv = __dsub_rn(sv, __dmul_rn(sc.omega, a.t[i]));      // :341
          a.r[i] = rv;
          acc[b][0] = __fma_rn(rv, rv, acc[b][0]);
          acc[b][1] = __fma_rn(a.rt0[i], rv, acc[b][1]);
        }
      }
    }
    if (ND > 0) bat_block_stage<ND == 0 ? 1 : ND>(B, acc, red, blk);
  }
  if (PH == PH_XR && anyhalf) {
    for (int b = 0; b < B.nrhs; ++b)
      if (st.half[b]) half_exit_update(B.a[b], st.sc[b].alpha, blockIdx.x, gridDim.x);
  }
  if (ND == 0) return;
  if (!elect_last_cta(B.counters + PH, &last_flag)) return;
  // final stages of every running rhs's dots, then its scalar logic
  {
    constexpr int NDd = ND > 0 ? ND : 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < B.nrhs * ND) {
      const int b = warp / NDd, d = warp - b * NDd;
      if (st.run[b]) {
        double v = warp_final_volatile(B.a[b].part + d * nb, nb);
        if (lane == 0) dfin[b][d] = v;
      }
    }
    if (PH == PH_XR) {
      for (int b = 0; b < B.nrhs; ++b) {
        if (!st.run[b]) continue;
        const IterArgs &a = B.a[b];
        for (int j = threadIdx.x; j < k; j += blockDim.x)   // solvers.py:340
          a.xc[j] = __dadd_rn(__dadd_rn(a.xc[j], __dmul_rn(st.sc[b].alpha, a.zeta[j])),
                              __dmul_rn(st.sc[b].omega, a.gamma[j]));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int anyrun = 0;
      for (int b = 0; b < B.nrhs; ++b) {
        if (st.run[b]) finalize<PH>(B.a[b], B.a[b].S, dfin[b]);
        anyrun |= B.a[b].S->status == KRB_RUNNING;
      }
      B.counters[PH] = 0;
      if (PH == PH_XR && B.use_cond) cudaGraphSetConditional(B.cond, anyrun ? 1u : 0u);
    }
  }
}

// q_b = A p_b (kSecond: t_b = A s_b) for every running rhs: the row's
// entries are read once, the B sums stay sequential in CSR order
template <bool kSell, bool kSecond>
__global__ void __launch_bounds__(256) k_bat_spmv(const BatArgs *__restrict__ pb) {
  __shared__ BatState st;
  const BatArgs &B = *pb;
  load_state(B, st);
  if (!st.any) return;
  const krb_matrix &A = B.a[0].A;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  const double *xs[kMaxB];
#pragma unroll
  for (int b = 0; b < kMaxB; ++b)
    xs[b] = (b < B.nrhs && st.run[b]) ? (kSecond ? B.a[b].s : B.a[b].p) : nullptr;
  const int32_t *__restrict__ cp;
  const double *__restrict__ vp;
  int len, stride;
  if (kSell) {
    len = __ldg(A.rlen + i);
    const int64_t base = __ldg(A.sl_ptr + (i >> 5)) + (i & 31);
    cp = A.s_col + base;
    vp = A.s_val + base;
    stride = 32;
  } else {
    const int64_t b0 = __ldg(A.rp + i);
    len = (int)(__ldg(A.rp + i + 1) - b0);
    cp = A.ci + b0;
    vp = A.val + b0;
    stride = 1;
  }
  double sum[kMaxB] = {0.0, 0.0, 0.0, 0.0};
  for (int j = 0; j < len; j += 4) {
    int c[4];
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = j + u < len;
      c[u] = ok ? __ldg(cp + (int64_t)stride * (j + u)) : 0;
      v[u] = ok ? __ldg(vp + (int64_t)stride * (j + u)) : 0.0;
    }
#pragma unroll
    for (int b = 0; b < kMaxB; ++b) {
      if (!xs[b]) continue;
      double xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = j + u < len ? xs[b][c[u]] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j + u < len) sum[b] = __dadd_rn(sum[b], __dmul_rn(v[u], xv[u]));
    }
  }
  const int64_t row = (kSell && A.perm) ? A.perm[i] : i;
#pragma unroll
  for (int b = 0; b < kMaxB; ++b)
    if (xs[b]) (kSecond ? B.a[b].t : B.a[b].q)[row] = sum[b];
}

// zeta_b = Chat^T q_b (kGamma: gamma_b = Chat^T t_b): unit = (canonical
// block, kBatCG columns), Chat read once for every rhs; per (rhs, column)
// canonical trees; the last CTA runs every final stage.
template <int kE, bool kGamma>
__global__ void __launch_bounds__(1024) k_bat_proj(const BatArgs *__restrict__ pb) {
  __shared__ double red[16][32];
  __shared__ int last_flag;
  __shared__ BatState st;
  const BatArgs &B = *pb;
  load_state(B, st);
  if (!st.any) return;
  const IterArgs &a0 = B.a[0];
  const int64_t n = a0.n, nb = a0.nb, ld = a0.ld;
  const int k = a0.k;
  const double *__restrict__ M = a0.Chat;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = blockIdx.y * kBatCG;
  const int nj = min(kBatCG, k - j0);
  const double *vs[kMaxB];
#pragma unroll
  for (int b = 0; b < kMaxB; ++b)
    vs[b] = (b < B.nrhs && st.run[b]) ? (kGamma ? B.a[b].t : B.a[b].q) : nullptr;
  for (int64_t blk = blockIdx.x; blk < nb; blk += gridDim.x) {
    double acc[kMaxB][kBatCG];
#pragma unroll
    for (int b = 0; b < kMaxB; ++b)
#pragma unroll
      for (int c = 0; c < kBatCG; ++c) acc[b][c] = 0.0;
    const int64_t base = blk * ((int64_t)kLanes * kE) + threadIdx.x;
#pragma unroll(kE < 4 ? kE : 4)
    for (int e = 0; e < kE; ++e) {
      const int64_t i = base + (int64_t)kLanes * e;
      if (i >= n) continue;
      double m[kBatCG];
#pragma unroll
      for (int c = 0; c < kBatCG; ++c) m[c] = c < nj ? __ldg(M + (int64_t)(j0 + c) * ld + i) : 0.0;
#pragma unroll
      for (int b = 0; b < kMaxB; ++b) {
        if (!vs[b]) continue;
        const double vi = vs[b][i];
#pragma unroll
        for (int c = 0; c < kBatCG; ++c) acc[b][c] = __fma_rn(m[c], vi, acc[b][c]);
      }
    }
    // 16 values (rhs b, column c) -> two transposed 8-value warp trees
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = acc[2 * h + (u >> 2)][u & 3];
      int col;
      double w = warp_tree_multi<8>(v, col);
      if ((lane & 3) == 0) red[8 * h + col][warp] = w;
    }
    __syncthreads();
    if (warp < 16) {
      const int b = warp >> 2, c = warp & 3;
      if (vs[b] && c < nj) {
        double r = warp_tree(red[warp][lane]);
        if (lane == 0) B.a[b].part[(int64_t)(j0 + c) * nb + blk] = r;
      }
    }
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(B.counters + 9, 1u);
    last_flag = (prev == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!last_flag) return;
  __threadfence();
  for (int u = warp; u < B.nrhs * k; u += 32) {
    const int b = u / k, j = u - b * k;
    if (!vs[b]) continue;
    double r = warp_final_volatile(B.a[b].part + (int64_t)j * nb, nb);
    if (lane == 0) (kGamma ? B.a[b].gamma : B.a[b].zeta)[j] = r;
  }
  if (threadIdx.x == 0) B.counters[9] = 0;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
template <int PH>
static int bat_launch_phase(int64_t n, int64_t nb, const BatArgs *d, cudaStream_t st) {
  if (nb == 0) return KRB_OK;
  KRB_DISPATCH_E(canon_E(n), (k_bat_phase<kE, PH><<<grid_for(nb), 1024, 0, st>>>(d)));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

template <bool kSecond>
static int bat_launch_spmv(int64_t n, int fmt, const BatArgs *d, cudaStream_t st) {
  if (n == 0) return KRB_OK;
  unsigned blocks = (unsigned)((n + 255) / 256);
  if (fmt == 2)
    k_bat_spmv<true, kSecond><<<blocks, 256, 0, st>>>(d);
  else
    k_bat_spmv<false, kSecond><<<blocks, 256, 0, st>>>(d);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

template <bool kGamma>
static int bat_launch_proj(int64_t n, int64_t nb, int64_t k, const BatArgs *d,
                           cudaStream_t st) {
  if (k <= 0 || nb == 0) return KRB_OK;
  const int64_t groups = (k + kBatCG - 1) / kBatCG;
  int64_t gx = (int64_t)kNumSMs * 2 / groups;
  if (gx < 1) gx = 1;
  if (gx > nb) gx = nb;
  dim3 grid((unsigned)gx, (unsigned)groups);
  KRB_DISPATCH_E(canon_E(n), (k_bat_proj<kE, kGamma><<<grid, 1024, 0, st>>>(d)));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

static int bat_iteration(int64_t n, int64_t nb, int64_t k, int fmt, const BatArgs *d,
                         cudaStream_t st) {
  KRB_TRY(bat_launch_phase<PH_PUPDATE>(n, nb, d, st));
  KRB_TRY(bat_launch_spmv<false>(n, fmt, d, st));
  KRB_TRY(bat_launch_proj<false>(n, nb, k, d, st));
  KRB_TRY(bat_launch_phase<PH_PROJ_Q>(n, nb, d, st));
  KRB_TRY(bat_launch_phase<PH_SUPD>(n, nb, d, st));
  KRB_TRY(bat_launch_spmv<true>(n, fmt, d, st));
  KRB_TRY(bat_launch_proj<true>(n, nb, k, d, st));
  KRB_TRY(bat_launch_phase<PH_PROJ_T>(n, nb, d, st));
  KRB_TRY(bat_launch_phase<PH_XR>(n, nb, d, st));
  return KRB_OK;
}

// per-context batch resources (vectors of every rhs, descriptors, graph)
struct BatchPool {
  int64_t n = 0, k = 0;
  double *vec = nullptr;       // kMaxB x 10 n-vectors
  double *kbuf = nullptr;      // kMaxB x 4 k-vectors
  double *part = nullptr;      // kMaxB x part_one
  size_t part_one = 0;
  SolveScalars *S = nullptr;   // kMaxB
  IterArgs *desc = nullptr;    // kMaxB
  BatArgs *bdesc = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond = 0;
  int gn = -1, gfmt = -1;
  int64_t gnn = -1, gk = -1;
  int64_t per_body = 0;
  void reset_graph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    gn = gfmt = -1;
    gnn = gk = -1;
  }
  void release() {
    reset_graph();
    cudaFree(vec);
    cudaFree(kbuf);
    cudaFree(part);
    cudaFree(S);
    cudaFree(desc);
    cudaFree(bdesc);
    vec = kbuf = part = nullptr;
    S = nullptr;
    desc = nullptr;
    bdesc = nullptr;
    n = k = 0;
  }
};

static BatchPool &pool_of(krb_context *ctx) {
  // one pool per context, owned through ctx->batch
  if (!ctx->batch) ctx->batch = new BatchPool();
  return *reinterpret_cast<BatchPool *>(ctx->batch);
}

void batch_pool_free(krb_context *ctx) {
  if (ctx && ctx->batch) {
    BatchPool *P = reinterpret_cast<BatchPool *>(ctx->batch);
    P->release();
    delete P;
    ctx->batch = nullptr;
  }
}

static int pool_reserve(BatchPool &P, int64_t n, int64_t k) {
  if (P.vec && n <= P.n && k <= P.k) return KRB_OK;
  P.release();
  const int64_t nn = n > 0 ? n : 1, kk = k > 0 ? k : 1;
  const int64_t nb = canon_nblocks(n);
  P.part_one = (size_t)((kk + 3) * (nb > 0 ? nb : 1)) + 64;
  KRB_CHECK_CUDA(cudaMalloc(&P.vec, sizeof(double) * kMaxB * 10 * nn));
  KRB_CHECK_CUDA(cudaMalloc(&P.kbuf, sizeof(double) * kMaxB * 4 * kk));
  KRB_CHECK_CUDA(cudaMalloc(&P.part, sizeof(double) * kMaxB * P.part_one));
  KRB_CHECK_CUDA(cudaMalloc(&P.S, sizeof(SolveScalars) * kMaxB));
  KRB_CHECK_CUDA(cudaMalloc(&P.desc, sizeof(IterArgs) * kMaxB));
  KRB_CHECK_CUDA(cudaMalloc(&P.bdesc, sizeof(BatArgs)));
  P.n = nn;
  P.k = kk;
  return KRB_OK;
}

static cudaStream_t bat_capture_stream() {
  static thread_local cudaStream_t s = nullptr;
  if (!s) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  return s;
}

static int bat_build_graph(BatchPool &P, int64_t n, int64_t nb, int64_t k, int fmt) {
  P.reset_graph();
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
  cudaStream_t cs = bat_capture_stream();
  KRB_CHECK_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeRelaxed));
  const int64_t c0 = launch_counter();
  int rc = bat_iteration(n, nb, k, fmt, P.bdesc, cs);
  P.per_body = launch_counter() - c0;
  launch_counter() = c0;
  cudaGraph_t out;
  cudaError_t e = cudaStreamEndCapture(cs, &out);
  if (rc || e != cudaSuccess) {
    cudaGraphDestroy(g);
    if (!rc) set_error("batch graph capture: %s", cudaGetErrorString(e));
    return rc ? rc : KRB_ECUDA;
  }
  e = cudaGraphInstantiate(&P.exec, g, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    set_error("batch graph instantiate: %s", cudaGetErrorString(e));
    return KRB_ECUDA;
  }
  P.graph = g;
  P.cond = hc;
  KRB_CHECK_CUDA(cudaGraphUpload(P.exec, cs));
  KRB_CHECK_CUDA(cudaStreamSynchronize(cs));
  P.gnn = n;
  P.gk = k;
  P.gfmt = fmt;
  return KRB_OK;
}

int rbicgstab_batch(krb_context *ctx, const krb_matrix *A, int64_t nrhs,
                    const double *const *d_b, const double *const *d_x_init,
                    const krb_space_view *R, const krb_solve_config *cfgs,
                    double *const *d_x_out, double *const *hist_r,
                    int64_t *const *hist_m, uint64_t *const *hist_t,
                    krb_solve_result *res, cudaStream_t st) {
  KRB_REQUIRE(ctx && A && d_b && cfgs && d_x_out && hist_r && hist_m && hist_t && res,
              "krb_rbicgstab_batch: NULL argument");
  KRB_REQUIRE(nrhs >= 1 && nrhs <= kMaxB, "krb_rbicgstab_batch: 1 <= nrhs <= 4");
  KRB_REQUIRE(!A->pre, "krb_rbicgstab_batch: preconditioned operators run one solve at a time");
  const int64_t n = A->n;
  const int64_t k = (R && R->k > 0) ? R->k : 0;
  if (k > 0) {
    KRB_REQUIRE(R->n == n, "recycle space dimension does not match the operator");
    KRB_REQUIRE(R->ld >= n, "recycle space leading dimension < n");
    KRB_REQUIRE(R->U && R->C && R->Ct && R->Chat && R->Ccheck,
                "recycle space view has NULL blocks");
    KRB_REQUIRE(k <= kBatMaxK, "krb_rbicgstab_batch: recycle dimension > 128");
  }
  const int mode = cfgs[0].use_graph == 0 ? 0 : 1;   // host loop or graph
  for (int64_t b = 0; b < nrhs; ++b)
    KRB_REQUIRE(d_b[b] && d_x_out[b] && hist_r[b] && hist_m[b] && hist_t[b],
                "krb_rbicgstab_batch: NULL per-rhs argument");
  BatchPool &P = pool_of(ctx);
  KRB_TRY(pool_reserve(P, n, k));
  KRB_TRY(ctx_reserve_vectors(ctx, n, k));   // shadow scratch (ctx->w)
  KRB_TRY(ctx_reserve_counters(ctx, st));
  const int64_t l0 = launch_counter();
  const int64_t nb = canon_nblocks(n);
  IterArgs h[kMaxB];
  for (int64_t b = 0; b < nrhs; ++b) {
    IterArgs &x = h[b];
    x = IterArgs{};
    x.A = *A;
    x.A.T = nullptr;
    x.n = n;
    x.nb = nb;
    x.k = (int)k;
    x.ld = k > 0 ? R->ld : n;
    x.C = k > 0 ? R->C : nullptr;
    x.Chat = k > 0 ? R->Chat : nullptr;
    x.U = k > 0 ? R->U : nullptr;
    double *V = P.vec + (size_t)b * 10 * P.n;
    x.x = V; x.r = V + P.n; x.p = V + 2 * P.n; x.q = V + 3 * P.n; x.s = V + 4 * P.n;
    x.t = V + 5 * P.n; x.rt0 = V + 6 * P.n; x.b = V + 7 * P.n;
    x.p2 = V + 8 * P.n; x.q2 = V + 9 * P.n;
    double *K = P.kbuf + (size_t)b * 4 * P.k;
    x.zeta = K; x.gamma = K + P.k; x.xc = K + 2 * P.k;
    x.part = P.part + (size_t)b * P.part_one;
    x.part2 = x.part;
    x.counters = ctx->counters;
    x.S = P.S + b;
    x.hist_r = hist_r[b];
    x.hist_m = hist_m[b];
    x.hist_t = hist_t[b];
    x.l2keep = 0;
  }
  const bool hit = mode == 1 && P.exec && P.gnn == n && P.gk == k && P.gfmt == A->format;
  if (mode == 1 && !hit) {
    KRB_CHECK_CUDA(cudaStreamSynchronize(st));
    KRB_TRY(bat_build_graph(P, n, nb, k, A->format));
  }
  BatArgs bh;
  bh.a = P.desc;
  bh.nrhs = (int)nrhs;
  bh.use_cond = mode == 1 ? 1 : 0;
  bh.cond = mode == 1 ? P.cond : 0;
  bh.counters = ctx->counters + kBatCounter;
  KRB_CHECK_CUDA(cudaMemcpyAsync(P.desc, h, sizeof(IterArgs) * nrhs, cudaMemcpyHostToDevice, st));
  KRB_CHECK_CUDA(cudaMemcpyAsync(P.bdesc, &bh, sizeof(BatArgs), cudaMemcpyHostToDevice, st));
  // per-rhs setup, exactly the single solve's (solvers.py:257-296)
  for (int64_t b = 0; b < nrhs; ++b) {
    double *ybuf = P.kbuf + (size_t)b * 4 * P.k + 3 * P.k;
    KRB_TRY(solve_setup(ctx, A, d_b[b], d_x_init ? d_x_init[b] : nullptr, R, &cfgs[b], h[b],
                        P.desc + b, ctx->w, ybuf, st));
  }
  int64_t per_body = 0;
  if (mode == 1) {
    KRB_CHECK_CUDA(cudaGraphLaunch(P.exec, st));
    per_body = P.per_body;
  } else {
    int64_t max_itn = 0;
    for (int64_t b = 0; b < nrhs; ++b) max_itn = cfgs[b].max_itn > max_itn ? cfgs[b].max_itn : max_itn;
    for (int64_t it = 0; it < max_itn + 1; ++it) {
      KRB_TRY(bat_iteration(n, nb, k, A->format, P.bdesc, st));
      if ((it & 7) == 7 || it == max_itn) {
        SolveScalars hs[kMaxB];
        KRB_CHECK_CUDA(cudaMemcpyAsync(hs, P.S, sizeof(SolveScalars) * nrhs,
                                       cudaMemcpyDeviceToHost, st));
        KRB_CHECK_CUDA(cudaStreamSynchronize(st));
        bool any = false;
        for (int64_t b = 0; b < nrhs; ++b) any |= hs[b].status == KRB_RUNNING;
        if (!any) break;
      }
    }
  }
  for (int64_t b = 0; b < nrhs; ++b)
    KRB_TRY(solve_tail(A, R, h[b], P.desc + b, d_x_out[b], st));
  SolveScalars hs[kMaxB];
  KRB_CHECK_CUDA(cudaMemcpyAsync(hs, P.S, sizeof(SolveScalars) * nrhs, cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  int64_t bodies = 0;
  for (int64_t b = 0; b < nrhs; ++b) bodies = hs[b].bodies > bodies ? hs[b].bodies : bodies;
  launch_counter() += bodies * per_body;
  for (int64_t b = 0; b < nrhs; ++b) {
    res[b].status = hs[b].status;
    res[b].hist_len = hs[b].hist_len;
    res[b].matvecs = hs[b].matvecs;
    res[b].rhs_norm = hs[b].bnorm;
    res[b].final_true_resid = hs[b].final_true_resid;
    res[b].t_start_ns = hs[b].t_start;
    res[b].iterations_run = hs[b].bodies;
    res[b].kernel_launches = launch_counter() - l0;
    res[b].driver = mode == 1 ? KRB_DRIVER_BATCH_GRAPH : KRB_DRIVER_HOST_LOOP;
  }
  return KRB_OK;
}

}  // namespace krb

using namespace krb;

extern "C" {

int krb_rbicgstab_batch(krb_context *ctx, const krb_matrix *A, int64_t nrhs,
                        const double *const *d_b, const double *const *d_x_init,
                        const krb_space_view *R, const krb_solve_config *cfgs,
                        double *const *d_x_out, double *const *d_hist_resid,
                        int64_t *const *d_hist_matvecs, uint64_t *const *d_hist_stamp,
                        krb_solve_result *h_results, void *stream) {
  return rbicgstab_batch(ctx, A, nrhs, d_b, d_x_init, R, cfgs, d_x_out, d_hist_resid,
                         d_hist_matvecs, d_hist_stamp, h_results, as_stream(stream));
}

}  // extern "C"
