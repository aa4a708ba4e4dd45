// Split ILUTP preconditioned operator on the device (reference ilutp.py:
// apply_left / apply_left_h / apply_right / apply_right_h at :76-97 and
// SplitPreconditionedOperator at :106-128):
//
//   op x   = L^{-1} A P U^{-1} x      t1 = U^{-1} x ; t2[perm] = t1 ;
//                                     t3 = A t2 ; y = L^{-1} t3
//   op^H x = U^{-H} P^T A^H L^{-H} x  t1 = L^{-H} x ; t2 = A^H t1 ;
//                                     t3 = t2[perm] ; y = U^{-H} t3
//
// The operator is a krb_matrix "view" of A carrying a krb_precond: every
// libkrb entry that applies A (krb_spmv / krb_spmv_t / krb_spmm, the
// solvers' setup / true residual, the graph iteration kernels of the
// BiCGSTAB and RBiCG drivers) goes through spmv_launch, which runs the
// composite above; the persistent drivers are not used for it.
//
// Triangular solves: ONE 512-thread CTA (16 warps) walks the level schedule (rows of a
// level depend only on earlier levels; __syncthreads between levels).  Row
// r of a level goes to warp r mod 16; each warp keeps its next 4 rows' data
// (off-diagonal entries, b, diagonal) in flight in registers, so a level
// costs a barrier + shared-memory gathers + one warp tree, not an L2 round
// trip.  x lives in shared memory when it fits (n <= 25600: C1).
//
// Canonical order of one row (oracle canon_trsv): lane l accumulates
// fma(v_e, x_{c_e}, acc) over the row's off-diagonal entries e = l, l + 32,
// ... in column order; the canonical 32-lane tree (offsets 16..1) gives S;
// x_i = b_i - S, divided by u_ii for U (unit L: no division).
#include <cuda_runtime.h>

#include <climits>
#include <vector>

#include "ctx.cuh"

namespace krb {

constexpr int kTriSmemN = 25600;       // x in shared memory up to this n
constexpr int kTriWarps = 16;          // warps of the solve CTA (krb_tri_host.warp_ptr)
static int64_t g_precond_serial = 0;

struct TriDev {
  int64_t n = 0;
  int32_t nlev = 0;
  const int64_t *rp = nullptr;     // off-diagonal CSR
  const int32_t *ci = nullptr;
  const double *val = nullptr;
  const double *diag = nullptr;    // nullptr: unit diagonal
  const int32_t *warp_ptr = nullptr;   // kTriWarps + 1: task range of each warp
  const int32_t *t_row = nullptr, *t_lev = nullptr, *t_len = nullptr;
  const int64_t *t_start = nullptr;
};

}  // namespace krb

struct krb_precond {
  krb::TriDev L, Lt, U, Ut;
  int64_t *perm = nullptr;
  double *t1 = nullptr, *t2 = nullptr, *t3 = nullptr;
  std::vector<void *> owned;
  int64_t serial = 0;
  int64_t n = 0;
};

namespace krb {

struct TriSlot {
  int row, lev, len;
  int64_t start;
  int c0, c1;
  double v0, v1, bv, dv;
};

template <bool kUnit>
__device__ __forceinline__ void tri_load(TriSlot &s, const TriDev &T, const double *b,
                                         int j, int je, int lane) {
  if (j >= je) {
    s.lev = INT_MAX;
    return;
  }
  s.row = __ldg(T.t_row + j);
  s.lev = __ldg(T.t_lev + j);
  s.len = __ldg(T.t_len + j);
  s.start = __ldg(T.t_start + j);
  s.c0 = lane < s.len ? __ldg(T.ci + s.start + lane) : 0;
  s.v0 = lane < s.len ? __ldg(T.val + s.start + lane) : 0.0;
  s.c1 = lane + 32 < s.len ? __ldg(T.ci + s.start + lane + 32) : 0;
  s.v1 = lane + 32 < s.len ? __ldg(T.val + s.start + lane + 32) : 0.0;
  s.bv = b[s.row];
  s.dv = kUnit ? 1.0 : __ldg(T.diag + s.row);
}

template <bool kSmem>
__device__ __forceinline__ double tri_x(const double *xs, const double *x, int c) {
  return kSmem ? xs[c] : __ldcg(x + c);
}

template <bool kUnit, bool kSmem>
__device__ __forceinline__ void tri_row(const TriSlot &s, const TriDev &T, double *xs,
                                        double *x, int lane) {
  double acc = 0.0;
  if (lane < s.len) acc = __fma_rn(s.v0, tri_x<kSmem>(xs, x, s.c0), acc);
  if (lane + 32 < s.len) acc = __fma_rn(s.v1, tri_x<kSmem>(xs, x, s.c1), acc);
  for (int e = lane + 64; e < s.len; e += 32)      // long rows: the rest on demand
    acc = __fma_rn(__ldg(T.val + s.start + e), tri_x<kSmem>(xs, x, __ldg(T.ci + s.start + e)),
                   acc);
  acc = warp_tree(acc);
  if (lane == 0) {
    double v = __dsub_rn(s.bv, acc);
    if (!kUnit) v = __ddiv_rn(v, s.dv);
    if (kSmem)
      xs[s.row] = v;
    else
      x[s.row] = v;
  }
}

// x = T^{-1} b; gated on *status != 0 (a finished solve's graph tail)
template <bool kUnit, bool kSmem>
__global__ void __launch_bounds__(kTriWarps * 32, 1) k_trsv(TriDev T, const double *__restrict__ b,
                                                  double *__restrict__ x,
                                                  const int *__restrict__ status) {
  extern __shared__ double xs[];
  if (status && *status) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int j = T.warp_ptr[warp];
  const int je = T.warp_ptr[warp + 1];
  TriSlot s0, s1, s2, s3;
  tri_load<kUnit>(s0, T, b, j, je, lane);
  tri_load<kUnit>(s1, T, b, j + 1, je, lane);
  tri_load<kUnit>(s2, T, b, j + 2, je, lane);
  tri_load<kUnit>(s3, T, b, j + 3, je, lane);
  int ph = 0;   // ring slot holding the warp's next task
#define KRB_TRI_STEP(S, NEXT)                                 \
  if (S.lev != lev) goto level_done;                          \
  tri_row<kUnit, kSmem>(S, T, xs, x, lane);                   \
  tri_load<kUnit>(S, T, b, j + 4, je, lane);                  \
  ++j;                                                        \
  ph = NEXT;
  for (int lev = 0; lev < T.nlev; ++lev) {
    for (;;) {
      switch (ph) {
        case 0: KRB_TRI_STEP(s0, 1) [[fallthrough]];
        case 1: KRB_TRI_STEP(s1, 2) [[fallthrough]];
        case 2: KRB_TRI_STEP(s2, 3) [[fallthrough]];
        default: KRB_TRI_STEP(s3, 0)
      }
    }
  level_done:
    __syncthreads();
  }
#undef KRB_TRI_STEP
  if (kSmem)
    for (int64_t i = threadIdx.x; i < T.n; i += blockDim.x) x[i] = xs[i];
}

__global__ void k_perm_scatter(int64_t n, const int64_t *__restrict__ perm,
                               const double *__restrict__ in, double *__restrict__ out,
                               const int *__restrict__ status) {
  if (status && *status) return;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[perm[j]] = in[j];       // x[perm] = t  (ilutp.py:89-90)
}

__global__ void k_perm_gather(int64_t n, const int64_t *__restrict__ perm,
                              const double *__restrict__ in, double *__restrict__ out,
                              const int *__restrict__ status) {
  if (status && *status) return;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[j] = in[perm[j]];       // z = x[perm]  (ilutp.py:96)
}

static int tri_launch(const TriDev &T, bool unit, const double *b, double *x,
                      const int *status, cudaStream_t st) {
  if (T.n == 0) return KRB_OK;
  const bool smem = T.n <= kTriSmemN;
  const size_t bytes = smem ? sizeof(double) * (size_t)T.n : 0;
  static bool attr = false;
  if (!attr) {
    const int mx = (int)(sizeof(double) * kTriSmemN);
    KRB_CHECK_CUDA(cudaFuncSetAttribute(k_trsv<true, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    KRB_CHECK_CUDA(cudaFuncSetAttribute(k_trsv<false, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    attr = true;
  }
  constexpr int kT = kTriWarps * 32;
  if (unit && smem) k_trsv<true, true><<<1, kT, bytes, st>>>(T, b, x, status);
  else if (unit) k_trsv<true, false><<<1, kT, 0, st>>>(T, b, x, status);
  else if (smem) k_trsv<false, true><<<1, kT, bytes, st>>>(T, b, x, status);
  else k_trsv<false, false><<<1, kT, 0, st>>>(T, b, x, status);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

// composite operator apply (called by spmv_launch for a view with `pre`)
int precond_apply_op(const krb_matrix *A, const double *x, double *y, const int *status,
                     cudaStream_t st) {
  const krb_precond *P = A->pre;
  const int64_t n = A->n;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (!A->pre_adj) {
    KRB_TRY(tri_launch(P->U, false, x, P->t1, status, st));
    k_perm_scatter<<<blocks, 256, 0, st>>>(n, P->perm, P->t1, P->t2, status);
    KRB_CHECK_LAUNCH();
    KRB_TRY(spmv_launch(A->base, P->t2, P->t3, status, st));
    KRB_TRY(tri_launch(P->L, true, P->t3, y, status, st));
  } else {
    KRB_TRY(tri_launch(P->Lt, true, x, P->t1, status, st));
    KRB_TRY(spmv_launch(A->base, P->t1, P->t2, status, st));
    k_perm_gather<<<blocks, 256, 0, st>>>(n, P->perm, P->t2, P->t3, status);
    KRB_CHECK_LAUNCH();
    KRB_TRY(tri_launch(P->Ut, false, P->t3, y, status, st));
  }
  return KRB_OK;
}

void precond_free(krb_precond *P) {
  if (!P) return;
  for (void *p : P->owned) dev_free(p, nullptr);
  delete P;
}

int64_t precond_serial(const krb_precond *P) { return P ? P->serial : 0; }

static int upload(krb_precond *P, const void *h, size_t bytes, void **d, cudaStream_t st) {
  *d = nullptr;
  if (!h || bytes == 0) return KRB_OK;
  KRB_CHECK_CUDA(dev_alloc(d, bytes, st));
  P->owned.push_back(*d);
  KRB_CHECK_CUDA(cudaMemcpyAsync(*d, h, bytes, cudaMemcpyHostToDevice, st));
  return KRB_OK;
}

static int upload_tri(krb_precond *P, const krb_tri_host *H, TriDev *T, cudaStream_t st) {
  KRB_REQUIRE(H != nullptr, "krb_precond_create: NULL factor");
  T->n = H->n;
  T->nlev = H->nlev;
  void *d;
  KRB_TRY(upload(P, H->rp, sizeof(int64_t) * (H->n + 1), &d, st)); T->rp = (const int64_t *)d;
  KRB_TRY(upload(P, H->ci, sizeof(int32_t) * H->nnz_off, &d, st)); T->ci = (const int32_t *)d;
  KRB_TRY(upload(P, H->val, sizeof(double) * H->nnz_off, &d, st)); T->val = (const double *)d;
  KRB_TRY(upload(P, H->diag, sizeof(double) * H->n, &d, st)); T->diag = (const double *)d;
  KRB_TRY(upload(P, H->warp_ptr, sizeof(int32_t) * (kTriWarps + 1), &d, st)); T->warp_ptr = (const int32_t *)d;
  KRB_TRY(upload(P, H->t_row, sizeof(int32_t) * H->ntasks, &d, st)); T->t_row = (const int32_t *)d;
  KRB_TRY(upload(P, H->t_lev, sizeof(int32_t) * H->ntasks, &d, st)); T->t_lev = (const int32_t *)d;
  KRB_TRY(upload(P, H->t_len, sizeof(int32_t) * H->ntasks, &d, st)); T->t_len = (const int32_t *)d;
  KRB_TRY(upload(P, H->t_start, sizeof(int64_t) * H->ntasks, &d, st)); T->t_start = (const int64_t *)d;
  return KRB_OK;
}

}  // namespace krb

using namespace krb;

extern "C" {

int krb_tri_levels(int64_t n, const int64_t *rp, const int32_t *ci, int lower,
                   int32_t *lev_out, int32_t *nlev_out) {
  KRB_REQUIRE(n >= 0 && (n == 0 || (rp && ci && lev_out)) && nlev_out,
              "krb_tri_levels: NULL argument");
  int32_t nlev = 0;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t i = lower ? t : n - 1 - t;
    int32_t lv = 0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const int64_t c = ci[e];
      if (lower ? c < i : c > i) {
        if (lev_out[c] + 1 > lv) lv = lev_out[c] + 1;
      } else if (c != i) {
        set_error("krb_tri_levels: entry (%lld, %lld) outside the %s triangle",
                  (long long)i, (long long)c, lower ? "lower" : "upper");
        return KRB_EINVAL;
      }
    }
    lev_out[i] = lv;
    if (lv + 1 > nlev) nlev = lv + 1;
  }
  *nlev_out = nlev;
  return KRB_OK;
}

int krb_precond_create(const krb_tri_host *L, const krb_tri_host *Lt, const krb_tri_host *U,
                       const krb_tri_host *Ut, const int64_t *h_perm, krb_precond **out,
                       void *stream) {
  KRB_REQUIRE(L && Lt && U && Ut && h_perm && out, "krb_precond_create: NULL argument");
  cudaStream_t st = as_stream(stream);
  const int64_t n = L->n;
  for (const krb_tri_host *T : {Lt, U, Ut})
    KRB_REQUIRE(T->n == n, "krb_precond_create: factor dimensions differ");
  krb_precond *P = new krb_precond();
  P->serial = ++g_precond_serial;
  int rc = upload_tri(P, L, &P->L, st);
  if (!rc) rc = upload_tri(P, Lt, &P->Lt, st);
  if (!rc) rc = upload_tri(P, U, &P->U, st);
  if (!rc) rc = upload_tri(P, Ut, &P->Ut, st);
  void *d = nullptr;
  if (!rc) rc = upload(P, h_perm, sizeof(int64_t) * n, &d, st);
  P->perm = (int64_t *)d;
  for (double **t : {&P->t1, &P->t2, &P->t3}) {
    if (rc) break;
    void *p = nullptr;
    if (dev_alloc(&p, sizeof(double) * (n > 0 ? n : 1), st) != cudaSuccess) {
      set_error("krb_precond_create: out of memory");
      rc = KRB_ENOMEM;
      break;
    }
    P->owned.push_back(p);
    *t = (double *)p;
  }
  if (!rc && cudaStreamSynchronize(st) != cudaSuccess) {
    set_error("krb_precond_create: upload failed");
    rc = KRB_ECUDA;
  }
  if (rc) {
    precond_free(P);
    return rc;
  }
  P->n = n;
  *out = P;
  return KRB_OK;
}

int krb_precond_destroy(krb_precond *P) {
  precond_free(P);
  return KRB_OK;
}

int krb_operator_create(krb_matrix *A, const krb_precond *P, krb_matrix **op_out) {
  KRB_REQUIRE(A && P && op_out, "krb_operator_create: NULL argument");
  KRB_REQUIRE(!A->pre, "krb_operator_create: A is already preconditioned");
  KRB_REQUIRE(A->n == P->n, "operator and factor dimensions disagree");
  krb_matrix *op = new krb_matrix(*A);
  op->T = nullptr;
  op->base = A;
  op->borrowed = true;
  op->pre = const_cast<krb_precond *>(P);
  op->pre_adj = false;
  *op_out = op;
  return KRB_OK;
}

int krb_precond_apply(const krb_precond *P, int which, const double *d_in, double *d_out,
                      void *stream) {
  KRB_REQUIRE(P && d_in && d_out, "krb_precond_apply: NULL argument");
  cudaStream_t st = as_stream(stream);
  switch (which) {
    case 0: return tri_launch(P->L, true, d_in, d_out, nullptr, st);     // L^{-1}
    case 1: return tri_launch(P->Lt, true, d_in, d_out, nullptr, st);    // L^{-H}
    case 2: return tri_launch(P->U, false, d_in, d_out, nullptr, st);    // U^{-1}
    case 3: return tri_launch(P->Ut, false, d_in, d_out, nullptr, st);   // U^{-H}
    default: break;
  }
  set_error("krb_precond_apply: which must be 0..3");
  return KRB_EINVAL;
}

}  // extern "C"
