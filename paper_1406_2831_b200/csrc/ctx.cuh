// krb_context: scratch owned by the library (partials, solver vectors,
// device scalar block, solve descriptor, CUDA-graph cache).
#pragma once

#include "krb_internal.cuh"

namespace krb {

// Device-resident solver scalars (one block per context).
struct SolveScalars {
  double rho, alpha, omega, beta;
  double den, qnorm, snorm, tt, ts, rnorm;
  double bnorm, tol_abs, nrt0, breakdown_tol;
  double final_true_resid, bb, rr_true;
  int64_t itn;       // completed iterations
  int64_t max_itn;
  int64_t matvecs;   // counted products
  int64_t hist_len;  // recorded history entries
  uint64_t t_start;
  int64_t bodies;    // graph-body (iteration) executions, incl. no-op tails
  int32_t status;
  int32_t early;     // converged at the half step this iteration
  int32_t k;
  int32_t pad;
};

// One instantiated solve graph; valid for every solve of the same shape
// (all per-solve pointers live in the device descriptor).
struct GraphCache {
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphConditionalHandle cond = 0;
  int64_t n = -1, k = -1;
  MatrixSig sig;                 // matrix (operator) / kernel-timing buffer baked
  const void *ktime = nullptr;   // into the SpMV node parameters
  int variant = -1;              // phase kernel variant (tuning) captured
  int format = -1;
  int64_t kernels_per_body = 0;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    cond = 0;
    n = k = -1;
    format = -1;
    kernels_per_body = 0;
  }
};

}  // namespace krb

struct krb_rbicg;

struct krb_context {
  // generic partial buffer for canonical reductions
  double *part = nullptr;
  size_t part_cap = 0;  // doubles
  unsigned int *counters = nullptr;  // last-CTA election counters
  // solver state
  krb::SolveScalars *S = nullptr;
  void *desc = nullptr;   // device copy of the solve descriptor (IterArgs)
  int64_t vec_n = 0, vec_k = 0;
  double *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *s = nullptr,
         *t = nullptr, *rt0 = nullptr, *b = nullptr, *w = nullptr;
  double *p2 = nullptr, *q2 = nullptr;   // double buffers (persistent v2)
  double *kbuf = nullptr;  // zeta, gamma, xc, y  (4 x k)
  krb::GraphCache graph;
  // buffers + instantiated graph of the last destroyed RBiCG handle, reused
  // by the next krb_rbicg_create of the same shape (no cudaMalloc / graph
  // instantiation / device-synchronising cudaFree per generation solve)
  krb_rbicg *bi_cache = nullptr;
  void *batch = nullptr;   // multi-rhs pool (batch.cu)
};

namespace krb {
// election-counter slots (ctx->counters)
constexpr int kNumCounters = 64;
constexpr int kCounterTdotStandalone = 20;
constexpr int kCounterTdotGraph = 21;
constexpr int kCounterGridSync = 48;   // 2 words: persistent-kernel grid barrier

// Process-wide driver / kernel-variant knobs (krb_set_tuning).  Every
// variant computes the same bits; the knobs exist so tests can force each
// driver and profiling tools can stamp phases.  -1 = automatic.
struct Tuning {
  int persist0 = 1;       // k = 0 fused kernel with the operator on chip
  int p0_grid_half = 0;   // persist0: one CTA per two canonical blocks
  int p0_onchip = 1;      // persist0: 0 = gather from global memory
  int p0_prof_cta = 0;    // persist0: CTA whose phase stamps are recorded
  int cluster = 1;        // single-cluster kernel for tiny systems
  int persist_v1 = 0;     // force the nine-barrier persistent kernel
  int gemm_mode = -1;     // krb_gemm: 0 row kernel, 8 / 12 / 24 / 122 tiled
  int l2keep = -1;        // evict_last policy on the recycle blocks
  int phase_variant = 0;  // graph phase kernels: 0 tuned per phase, 1 uniform (round 1)
  int tdot_variant = 0;   // graph projection dots: 0 <= 64 regs, 1 <= 32 regs
  int spmv_prefetch_mb = 6;  // offset-coded SpMV: bulk L2 prefetch distance ahead (MB, 0 = off)
  int spmm_variant = 1;      // offset-coded SpMM: 0 generic kernel, 1 k_spmm_dict (L2 prefetch)
  int phase_pf_rows = 1;     // graph P / S / X: L2 prefetch distance (1024-element rows)
  int spmv_variant = 0;   // offset-coded SpMV: 0 = uniform offsets by warp shuffle, 1 = int4 loads
  int value_coding = 1;   // value tables of constant diagonals: 0 = neither built nor used
};
Tuning &tuning();

int ctx_reserve_part(krb_context *ctx, size_t doubles);
int ctx_reserve_counters(krb_context *ctx, cudaStream_t st);
dim3 tdot_grid(int64_t nb, int64_t k, int per_sm);
// resident 1024-thread CTAs per SM of a kernel (>= 1)
template <class K>
int occupancy_1024(K kernel) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, 1024, 0) != cudaSuccess) {
    cudaGetLastError();
    b = 1;
  }
  return b > 0 ? b : 1;
}
int ctx_reserve_vectors(krb_context *ctx, int64_t n, int64_t k);
void rbicg_cache_free(krb_context *ctx);
void batch_pool_free(krb_context *ctx);

// canonical primitives used across translation units (stream-ordered)
int launch_dot_partials(int64_t n, const double *x, const double *y,
                        double *part, cudaStream_t st);
int launch_final(int ndots, int64_t nb, const double *part, double *out,
                 cudaStream_t st);
int launch_tdot(krb_context *ctx, int64_t n, int64_t k, const double *M,
                int64_t ldm, const double *v, bool self, double *out,
                const int *status, cudaStream_t st, bool self_sqrt = true);
int launch_gemv(int64_t n, int64_t k, const double *M, int64_t ldm,
                const double *y, const double *base, int sign, double *out,
                cudaStream_t st);
int spmv_launch(const krb_matrix *A, const double *x, double *y,
                const int *d_status, cudaStream_t st);
int ensure_transpose(krb_matrix *A, cudaStream_t st);
}  // namespace krb
