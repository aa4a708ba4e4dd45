// Device sparse matrices and SpMV for sm_100a.
//
// Replaces SparseMatrix.matvec / rmatvec (reference sparse.py:117-130), i.e.
// scipy's csr_matvec: y_i = ((0 + a_i0 x_c0) + a_i1 x_c1) + ... in CSR order,
// every product rounded before the add.  To stay bit-identical the GPU keeps
// ONE thread per row walking its row in CSR order (no segmented or
// warp-split sums, which would re-associate), and the library is compiled
// with -fmad=false so the multiply and add are never contracted.
//
// Formats (chosen per matrix, krb_matrix_create(format=0)):
//   SELL-32   32 consecutive rows form a slice stored column-major
//             (element j of lane l at slice_ptr[s] + 32 j + l), so the 32
//             threads of a warp read 32 consecutive doubles / int32 per step:
//             fully coalesced 256 B + 128 B transactions.  Per-row lengths
//             stop every thread at its own row end (padding is never summed).
//   CSR       fallback when SELL padding would exceed 20% of nnz (power-law
//             rows); same per-row order, loads served through L1.
// The transpose (A^T, for rmatvec / two-sided RBiCG) is built on the device
// once by a stable radix sort of the column indices, which reproduces
// scipy's .transpose().tocsr() order (ascending original row within each
// column), and gets its own format choice.
#include <cub/cub.cuh>
#include <cstring>
#include <mutex>
#include <atomic>
#include <vector>

#include "krb_internal.cuh"
#include "spmv.cuh"
#include "ctx.cuh"


namespace krb {

__global__ void k_row_len(int64_t n, const int64_t *__restrict__ rp,
                          int32_t *__restrict__ rlen) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rlen[i] = (int32_t)(rp[i + 1] - rp[i]);
}

// width of each 32-row slice = max row length (warp max)
__global__ void k_slice_width(int64_t n, const int32_t *__restrict__ rlen,
                              int64_t *__restrict__ width) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int v = i < n ? rlen[i] : 0;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
    v = max(v, __shfl_xor_sync(0xffffffffu, v, off));
  if ((threadIdx.x & 31) == 0 && (i >> 5) < (n + 31) / 32)
    width[i >> 5] = 32 * (int64_t)v;
}

__global__ void k_sell_fill(int64_t n, const int64_t *__restrict__ rp,
                            const int32_t *__restrict__ ci,
                            const double *__restrict__ val,
                            const int64_t *__restrict__ sl_ptr,
                            int32_t *__restrict__ s_col,
                            double *__restrict__ s_val) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t base = sl_ptr[i >> 5] + (i & 31);
  int64_t b = rp[i], e = rp[i + 1];
  for (int64_t jj = b; jj < e; ++jj) {
    s_col[base + 32 * (jj - b)] = ci[jj];
    s_val[base + 32 * (jj - b)] = val[jj];
  }
}

__global__ void k_pad_fill(int64_t total, int32_t *s_col, double *s_val) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) {
    s_col[i] = 0;
    s_val[i] = 0.0;
  }
}

template <bool kSell>
__global__ void __launch_bounds__(256) k_spmv(krb_matrix A,
                                              const double *__restrict__ x,
                                              double *__restrict__ y,
                                              const int *__restrict__ status) {
  if (status && *status) return;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  y[(kSell && A.perm) ? A.perm[i] : i] = spmv_row<kSell>(i, A, x);
}

static int64_t next_uid() {
  static std::atomic<int64_t> c{0};
  return ++c;
}

MatrixSig matrix_sig(const krb_matrix *A) {
  MatrixSig g;
  memset(g.p, 0, sizeof(g.p));
  if (!A) return g;
  const krb_matrix *B = A->base ? A->base : A;
  const void *ptrs[] = {A->rp, A->ci, A->val, A->sl_ptr, A->rlen, A->s_col, A->s_val,
                        A->perm, B->rp, B->ci, B->val, B->sl_ptr, B->rlen, B->s_col,
                        B->s_val, B->perm, A->dcode, A->dptr, A->dict, B->dcode, B->dptr,
                        B->dict, A->vtab, A->tent, A->tid, B->vtab, B->tent, B->tid};
  static_assert(sizeof(ptrs) == sizeof(g.p), "MatrixSig size");
  for (int i = 0; i < 28; ++i) g.p[i] = ptrs[i];
  g.n = A->n;
  g.format = A->format;
  g.serial = precond_serial(A->pre);
  // the diagonal table is baked into a captured graph's kernel parameters BY
  // VALUE: another matrix at the same addresses (freed and re-allocated
  // arrays) with other constants must not reuse that graph
  g.uid = B->dia.nd ? B->uid : 0;
  return g;
}

bool same_sig(const MatrixSig &a, const MatrixSig &b) {
  return a.n == b.n && a.format == b.format && a.serial == b.serial && a.uid == b.uid &&
         memcmp(a.p, b.p, sizeof(a.p)) == 0;
}

// offset-coded SELL-32 (identity row order)
template <int kV, int kVC = 0>   // kVC: 1 value-coded by row templates, 2 in diagonal form
__global__ void __launch_bounds__(256, kVC == 1 ? 4 : 6) k_spmv_dict(krb_matrix A, const double *__restrict__ x,
                                                   double *__restrict__ y,
                                                   const int *__restrict__ status, int64_t pf) {
  if (status && *status) return;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  auto xf = [x](int c) { return __ldg(x + c); };
  if (kVC == 2)
    y[i] = spmv_row_dia(i, A, x);
  else if (kVC == 1)
    y[i] = spmv_row_tmpl(i, A, xf);
  else
    y[i] = spmv_row_dict<kV, decltype(xf), 4>(i, A, xf, pf);
}

int spmv_launch(const krb_matrix *A, const double *x, double *y,
                const int *d_status, cudaStream_t st) {
  if (A->n == 0) return KRB_OK;
  if (A->pre) return precond_apply_op(A, x, y, d_status, st);
  int64_t blocks = (A->n + 255) / 256;
  const int64_t pf = (int64_t)tuning().spmv_prefetch_mb << 20;
  if (A->tent && tuning().value_coding && A->dia.nd && tuning().value_coding != 2)
    k_spmv_dict<0, 2><<<(unsigned)blocks, 256, 0, st>>>(*A, x, y, d_status, 0);
  else if (A->tent && tuning().value_coding)
    k_spmv_dict<0, 1><<<(unsigned)blocks, 256, 0, st>>>(*A, x, y, d_status, 0);
  else if (A->dcode && tuning().spmv_variant == 1)
    k_spmv_dict<1><<<(unsigned)blocks, 256, 0, st>>>(*A, x, y, d_status, pf);
  else if (A->dcode)
    k_spmv_dict<0><<<(unsigned)blocks, 256, 0, st>>>(*A, x, y, d_status, pf);
  else if (A->format == 2)
    k_spmv<true><<<(unsigned)blocks, 256, 0, st>>>(*A, x, y, d_status);
  else
    k_spmv<false><<<(unsigned)blocks, 256, 0, st>>>(*A, x, y, d_status);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}


// ---- SpMM: Y[:,c] = A X[:,c] for a group of kNC columns per pass --------
// Each thread owns one row and walks it ONCE in CSR order, keeping kNC
// independent sequential sums (multiply then add, from 0.0) -- so every
// column is bit-identical to its own SpMV, while the matrix is read once per
// group of kNC columns instead of once per column.
template <int kF, int kNC>
__global__ void __launch_bounds__(256) k_spmm(krb_matrix A, int ncols,
                                              const double *__restrict__ X,
                                              int64_t ldx, double *__restrict__ Y,
                                              int64_t ldy) {
  constexpr bool kSell = kF == 1;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  const int c0 = blockIdx.y * kNC;
  const int nc = min(kNC, ncols - c0);
  const double *Xc = X + (int64_t)c0 * ldx;
  double sum[kNC];
#pragma unroll
  for (int c = 0; c < kNC; ++c) sum[c] = 0.0;
  int64_t row = i;
  if (kF == 2) {
    const int64_t s = i >> 5;
    const int l = (int)(i & 31);
    const int len = __ldg(A.rlen + i);
    const int64_t base = __ldg(A.sl_ptr + s) + l;
    const int64_t dp = __ldg(A.dptr + s);
    const bool uni = dp & 1;
    const uint8_t *cp = A.dcode + (dp >> 1) + (uni ? 0 : l);
    for (int j = 0; j < len; ++j) {
      const int col = (int)i + (uni ? __ldg(reinterpret_cast<const int32_t *>(cp) + j)
                                    : __ldg(A.dict + __ldg(cp + 32 * j)));
      const double v = __ldg(A.s_val + base + 32 * j);
#pragma unroll
      for (int c = 0; c < kNC; ++c)
        if (c < nc) sum[c] = __dadd_rn(sum[c], __dmul_rn(v, __ldg(Xc + (int64_t)c * ldx + col)));
    }
  } else if (kSell) {
    if (A.perm) row = A.perm[i];
    const int len = __ldg(A.rlen + i);
    const int64_t base = __ldg(A.sl_ptr + (i >> 5)) + (i & 31);
    for (int j = 0; j < len; ++j) {
      const int col = __ldg(A.s_col + base + 32 * j);
      const double v = __ldg(A.s_val + base + 32 * j);
#pragma unroll
      for (int c = 0; c < kNC; ++c)
        if (c < nc) sum[c] = __dadd_rn(sum[c], __dmul_rn(v, __ldg(Xc + (int64_t)c * ldx + col)));
    }
  } else {
    const int64_t b = __ldg(A.rp + i), e = __ldg(A.rp + i + 1);
    for (int64_t jj = b; jj < e; ++jj) {
      const int col = __ldg(A.ci + jj);
      const double v = __ldg(A.val + jj);
#pragma unroll
      for (int c = 0; c < kNC; ++c)
        if (c < nc) sum[c] = __dadd_rn(sum[c], __dmul_rn(v, __ldg(Xc + (int64_t)c * ldx + col)));
    }
  }
  double *Yc = Y + (int64_t)c0 * ldy;
#pragma unroll
  for (int c = 0; c < kNC; ++c)
    if (c < nc) Yc[(int64_t)c * ldy + row] = sum[c];
}

// Offset-coded SpMM with kB entries of the row in flight per step (their
// kB x kNC gathers issued together), the value stream bulk-prefetched into
// L2 as in the SpMV; per column the same sequential mul-then-add sum.
// C5, 30 columns (A/B): <8, 1> 11.5 ms, <8, 2> 12.9 ms (80 registers),
// <4, 4> 27.6 ms (84 registers, twice the matrix passes), the generic
// k_spmm<2, 8> 15.9 ms.
template <int kNC, int kB, bool kVC = false>
__global__ void __launch_bounds__(256) k_spmm_dict(krb_matrix A, int ncols,
                                                   const double *__restrict__ X, int64_t ldx,
                                                   double *__restrict__ Y, int64_t ldy,
                                                   int64_t pf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  const int c0 = blockIdx.y * kNC;
  const int nc = min(kNC, ncols - c0);
  const double *__restrict__ Xc = X + (int64_t)c0 * ldx;
  double sum[kNC];
#pragma unroll
  for (int c = 0; c < kNC; ++c) sum[c] = 0.0;
  const int64_t s = i >> 5;
  const int l = (int)(i & 31);
  const int64_t vbase = __ldg(A.sl_ptr + s);
  const double *__restrict__ vp = A.s_val + vbase + l;
  const int row = (int)i;
  if (kVC) {
    // value-coded: the row's template (spmv_row_tmpl) supplies offsets and
    // the values of the constant diagonals
    const int t = __ldg(A.tid + i);
    const int len = __ldg(A.tlen + t);
    const int4 *__restrict__ te = reinterpret_cast<const int4 *>(A.tent) + (int64_t)t * A.tstride;
    for (int j = 0; j < len; j += kB) {
      int col[kB];
      double v[kB], g[kB][kNC];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const bool ok = j + u < len;
        const int4 e = ok ? __ldg(te + j + u) : make_int4(0, 1, 0, 0);
        col[u] = row + e.x;
        v[u] = e.y ? __hiloint2double(e.w, e.z) : __ldg(vp + 32 * (j + u));
      }
#pragma unroll
      for (int u = 0; u < kB; ++u)
#pragma unroll
        for (int c = 0; c < kNC; ++c)
          g[u][c] = (j + u < len && c < nc) ? __ldg(Xc + (int64_t)c * ldx + col[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < kB; ++u)
        if (j + u < len) {
#pragma unroll
          for (int c = 0; c < kNC; ++c) sum[c] = __dadd_rn(sum[c], __dmul_rn(v[u], g[u][c]));
        }
    }
  } else {
    const int len = __ldg(A.rlen + i);
    if (pf > 0 && l == 0) {
      const int64_t at = vbase + pf / 8, nbytes = 256 * (int64_t)len;
      if (at + nbytes / 8 <= A.sell_elems && nbytes > 0) prefetch_l2_bulk(A.s_val + at, (uint32_t)nbytes);
    }
    const int64_t dp = __ldg(A.dptr + s);
    const bool uni = dp & 1;
    const uint8_t *__restrict__ cp = A.dcode + (dp >> 1) + (uni ? 0 : l);
    for (int j = 0; j < len; j += kB) {
      int col[kB];
      double v[kB], g[kB][kNC];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const bool ok = j + u < len;
        col[u] = ok ? row + (uni ? __ldg(reinterpret_cast<const int32_t *>(cp) + j + u)
                                 : __ldg(A.dict + __ldg(cp + 32 * (j + u))))
                    : row;
        v[u] = ok ? __ldg(vp + 32 * (j + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kB; ++u)
#pragma unroll
        for (int c = 0; c < kNC; ++c)
          g[u][c] = (j + u < len && c < nc) ? __ldg(Xc + (int64_t)c * ldx + col[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < kB; ++u)
        if (j + u < len) {
#pragma unroll
          for (int c = 0; c < kNC; ++c) sum[c] = __dadd_rn(sum[c], __dmul_rn(v[u], g[u][c]));
        }
    }
  }
  double *Yc = Y + (int64_t)c0 * ldy;
#pragma unroll
  for (int c = 0; c < kNC; ++c)
    if (c < nc) Yc[(int64_t)c * ldy + i] = sum[c];
}

int spmm_launch(const krb_matrix *M, int64_t ncols, const double *X, int64_t ldx,
                double *Y, int64_t ldy, cudaStream_t st) {
  constexpr int kNC = 8;
  const int sv = tuning().spmm_variant;
  if (M->dcode && !M->pre && M->n > 0 && ncols > 0 && sv > 0) {
    const int64_t pf = (int64_t)tuning().spmv_prefetch_mb << 20;
    const unsigned gx = (unsigned)((M->n + 255) / 256);
    dim3 grid(gx, (unsigned)((ncols + 7) / 8));
    if (M->tent && tuning().value_coding)
      k_spmm_dict<8, 1, true><<<grid, 256, 0, st>>>(*M, (int)ncols, X, ldx, Y, ldy, 0);
    else
      k_spmm_dict<8, 1><<<grid, 256, 0, st>>>(*M, (int)ncols, X, ldx, Y, ldy, pf);
    KRB_CHECK_LAUNCH();
    return KRB_OK;
  }
  if (M->n == 0 || ncols == 0) return KRB_OK;
  if (M->pre) {   // preconditioned operator: one composite application per column
    for (int64_t c = 0; c < ncols; ++c)
      KRB_TRY(spmv_launch(M, X + c * ldx, Y + c * ldy, nullptr, st));
    return KRB_OK;
  }
  dim3 grid((unsigned)((M->n + 255) / 256), (unsigned)((ncols + kNC - 1) / kNC));
  if (M->dcode)
    k_spmm<2, kNC><<<grid, 256, 0, st>>>(*M, (int)ncols, X, ldx, Y, ldy);
  else if (M->format == 2)
    k_spmm<1, kNC><<<grid, 256, 0, st>>>(*M, (int)ncols, X, ldx, Y, ldy);
  else
    k_spmm<0, kNC><<<grid, 256, 0, st>>>(*M, (int)ncols, X, ldx, Y, ldy);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

// ---- build ---------------------------------------------------------------
__global__ void k_i64_to_i32(int64_t m, const int64_t *src, int32_t *dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) dst[i] = (int32_t)src[i];
}

__global__ void k_iota(int64_t m, int32_t *p) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) p[i] = (int32_t)i;
}

__global__ void k_sell_fill_perm(int64_t n, const int64_t *__restrict__ rp,
                                 const int32_t *__restrict__ ci,
                                 const double *__restrict__ val,
                                 const int64_t *__restrict__ sl_ptr,
                                 const int32_t *__restrict__ perm,
                                 int32_t *__restrict__ s_col,
                                 double *__restrict__ s_val) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t row = perm[p];
  int64_t base = sl_ptr[p >> 5] + (p & 31);
  int64_t b = rp[row], e = rp[row + 1];
  for (int64_t jj = b; jj < e; ++jj) {
    s_col[base + 32 * (jj - b)] = ci[jj];
    s_val[base + 32 * (jj - b)] = val[jj];
  }
}

__global__ void k_window_offsets(int64_t nseg, int64_t n, int64_t sigma, int *off) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= nseg) off[i] = (int)(i * sigma < n ? i * sigma : n);
}

// slice widths + exclusive scan -> sl_ptr; returns the padded element count
static int sell_layout(krb_matrix *A, const int32_t *rlen_pos, int64_t *total,
                       cudaStream_t st) {
  const int64_t n = A->n;
  int64_t *width = nullptr;
  KRB_CHECK_CUDA(dev_alloc((void **)&width, sizeof(int64_t) * (A->nslices + 1), st));
  if (n > 0) {
    unsigned wblocks = (unsigned)((A->nslices * 32 + 255) / 256);
    k_slice_width<<<wblocks, 256, 0, st>>>(n, rlen_pos, width);
    KRB_CHECK_LAUNCH();
  }
  KRB_CHECK_CUDA(cudaMemsetAsync(width + A->nslices, 0, sizeof(int64_t), st));
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, width, A->sl_ptr, A->nslices + 1, st);
  KRB_CHECK_CUDA(dev_alloc((void **)&tmp, tmp_bytes, st));
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, width, A->sl_ptr, A->nslices + 1, st);
  KRB_CHECK_CUDA(cudaGetLastError());
  KRB_CHECK_CUDA(cudaMemcpyAsync(total, A->sl_ptr + A->nslices, sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  dev_free(tmp, st);
  dev_free(width, st);
  return KRB_OK;
}

// SELL-C-sigma: sort rows by length (descending, stable) inside windows of
// kSigma rows so every 32-row slice holds rows of similar length; the
// permutation only moves whole rows, each row is still summed in CSR order.
constexpr int64_t kSigma = 4096;

static int sigma_sort(krb_matrix *A, cudaStream_t st) {
  const int64_t n = A->n;
  const int64_t nseg = (n + kSigma - 1) / kSigma;
  int32_t *keys_out = nullptr, *iota = nullptr;
  int *off = nullptr;
  KRB_CHECK_CUDA(dev_alloc((void **)&keys_out, sizeof(int32_t) * n, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&iota, sizeof(int32_t) * n, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&A->perm, sizeof(int32_t) * n, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&off, sizeof(int) * (nseg + 1), st));
  k_iota<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, iota);
  KRB_CHECK_LAUNCH();
  k_window_offsets<<<(unsigned)((nseg + 256) / 256), 256, 0, st>>>(nseg, n, kSigma, off);
  KRB_CHECK_LAUNCH();
  void *tmp = nullptr;
  size_t tb = 0;
  cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, tb, A->rlen, keys_out, iota,
                                                     A->perm, (int)n, (int)nseg, off, off + 1,
                                                     0, 32, st);
  KRB_CHECK_CUDA(dev_alloc((void **)&tmp, tb, st));
  cub::DeviceSegmentedRadixSort::SortPairsDescending(tmp, tb, A->rlen, keys_out, iota,
                                                     A->perm, (int)n, (int)nseg, off, off + 1,
                                                     0, 32, st);
  KRB_CHECK_CUDA(cudaGetLastError());
  dev_free(tmp, st);
  dev_free(off, st);
  dev_free(iota, st);
  dev_free(A->rlen, st);
  A->rlen = keys_out;   // lengths now indexed by slice position
  return KRB_OK;
}

static int build_sell(krb_matrix *A, int format, cudaStream_t st) {
  const int64_t n = A->n;
  A->nslices = (n + 31) / 32;
  KRB_CHECK_CUDA(dev_alloc((void **)&A->rlen, sizeof(int32_t) * (n > 0 ? n : 1), st));
  KRB_CHECK_CUDA(dev_alloc((void **)&A->sl_ptr, sizeof(int64_t) * (A->nslices + 1), st));
  unsigned blocks = (unsigned)((n + 255) / 256);
  if (n > 0) {
    k_row_len<<<blocks, 256, 0, st>>>(n, A->rp, A->rlen);
    KRB_CHECK_LAUNCH();
  }
  int64_t total = 0;
  int rc = sell_layout(A, A->rlen, &total, st);
  if (rc) return rc;
  const int64_t budget = A->nnz + A->nnz / 5;   // <= 20 % padding
  bool use_sell = format == 2 || (format == 0 && total <= budget);
  if (!use_sell && (format == 0 || format == 3) && n > 0) {
    rc = sigma_sort(A, st);
    if (rc) return rc;
    rc = sell_layout(A, A->rlen, &total, st);
    if (rc) return rc;
    use_sell = format == 3 || total <= budget;
    if (!use_sell) {
      dev_free(A->perm, st);
      A->perm = nullptr;
    }
  }
  A->sell_elems = total;
  if (!use_sell) {
    dev_free(A->sl_ptr, st);
    A->sl_ptr = nullptr;
    dev_free(A->rlen, st);
    A->rlen = nullptr;
    A->format = 1;
    return KRB_OK;
  }
  KRB_CHECK_CUDA(dev_alloc((void **)&A->s_col, sizeof(int32_t) * (total > 0 ? total : 1), st));
  KRB_CHECK_CUDA(dev_alloc((void **)&A->s_val, sizeof(double) * (total > 0 ? total : 1), st));
  if (total > A->nnz) {
    k_pad_fill<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(total, A->s_col, A->s_val);
    KRB_CHECK_LAUNCH();
  }
  if (n > 0) {
    if (A->perm)
      k_sell_fill_perm<<<blocks, 256, 0, st>>>(n, A->rp, A->ci, A->val, A->sl_ptr, A->perm,
                                               A->s_col, A->s_val);
    else
      k_sell_fill<<<blocks, 256, 0, st>>>(n, A->rp, A->ci, A->val, A->sl_ptr,
                                          A->s_col, A->s_val);
    KRB_CHECK_LAUNCH();
  }
  A->format = 2;
  A->bytes += total * 12 + (A->nslices + 1) * 8 + n * 4 + (A->perm ? n * 4 : 0);
  return KRB_OK;
}

// ---- offset-coded SELL-32 (krb_internal.cuh) ------------------------------
__global__ void k_row_offsets(int64_t n, const int64_t *__restrict__ rp,
                              const int32_t *__restrict__ ci, int32_t *__restrict__ off) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t jj = rp[i]; jj < rp[i + 1]; ++jj) off[jj] = ci[jj] - (int32_t)i;
}

__device__ __forceinline__ int dict_code(const int32_t *sd, int nd, int32_t off) {
  int lo = 0, hi = nd - 1;   // sd sorted ascending, off present
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sd[mid] < off) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// one warp per slice: uniform (all 32 rows present, equal lengths, equal
// offset sequences) -> one int32 offset row (4 len bytes rounded up to 32),
// else one code byte per element (32 x width)
__global__ void k_dict_classify(int64_t n, int64_t nslices, const int64_t *__restrict__ sl_ptr,
                                const int32_t *__restrict__ rlen,
                                const int32_t *__restrict__ s_col, int64_t *__restrict__ bytes,
                                uint8_t *__restrict__ uni, unsigned long long *__restrict__ nuni) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int l = threadIdx.x & 31;
  if (s >= nslices) return;
  const int64_t row = s * 32 + l;
  const int len = row < n ? rlen[row] : -1;
  const int64_t base = sl_ptr[s];
  const int width = (int)((sl_ptr[s + 1] - base) / 32);
  bool ok = __all_sync(0xffffffffu, len == __shfl_sync(0xffffffffu, len, 0));
  for (int j = 0; ok && j < len; ++j) {
    const int32_t off = s_col[base + 32 * j + l] - (int32_t)row;
    ok = __all_sync(0xffffffffu, off == __shfl_sync(0xffffffffu, off, 0));
  }
  if (l == 0) {
    uni[s] = ok ? 1 : 0;
    if (ok) atomicAdd(nuni, 1ull);
    bytes[s] = ok ? (int64_t)((len + 7) / 8) * 32 : (int64_t)32 * width;
  }
}

__global__ void k_dict_fill(int64_t n, int64_t nslices, const int64_t *__restrict__ sl_ptr,
                            const int32_t *__restrict__ rlen, const int32_t *__restrict__ s_col,
                            const int32_t *__restrict__ dict, int nd,
                            const int64_t *__restrict__ cptr, const uint8_t *__restrict__ uni,
                            uint8_t *__restrict__ code, int64_t *__restrict__ dptr) {
  __shared__ int32_t sd[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) sd[t] = dict[t];
  __syncthreads();
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int l = threadIdx.x & 31;
  if (s >= nslices) return;
  const int64_t base = sl_ptr[s], cb = cptr[s];
  const int width = (int)((sl_ptr[s + 1] - base) / 32);
  const int64_t row = s * 32 + l;
  if (uni[s]) {
    const int len = rlen[s * 32];
    int32_t *orow = reinterpret_cast<int32_t *>(code + cb);
    for (int j = l; j < (len + 7) / 8 * 8; j += 32)
      orow[j] = j < len ? s_col[base + 32 * j] - (int32_t)(s * 32) : 0;
  } else {
    const int len = row < n ? rlen[row] : 0;
    for (int j = 0; j < width; ++j)
      code[cb + 32 * j + l] =
          j < len ? (uint8_t)dict_code(sd, nd, s_col[base + 32 * j + l] - (int32_t)row) : 0;
  }
  if (l == 0) dptr[s] = (cb << 1) | (uni[s] ? 1 : 0);
}

// one CSR entry index per offset code (any entry of that diagonal; the race
// between writers is benign)
__global__ void __launch_bounds__(256) k_dict_rep(int64_t n, const int64_t *__restrict__ rp,
                                                  const int32_t *__restrict__ ci,
                                                  const int32_t *__restrict__ dict, int nd,
                                                  int32_t *__restrict__ rep) {
  __shared__ int32_t sd[256];
  __shared__ int sf[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) {
    sd[t] = dict[t];
    sf[t] = -1;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    for (int64_t jj = rp[i]; jj < rp[i + 1]; ++jj) {
      const int code = dict_code(sd, nd, ci[jj] - (int32_t)i);
      if (sf[code] < 0) sf[code] = (int)jj;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nd; t += blockDim.x)
    if (sf[t] >= 0 && rep[t] < 0) rep[t] = sf[t];
}

// Build the offset-coded stream beside an identity-order SELL-32 matrix when
// its entries use at most 255 distinct offsets col - row.  Leaves the matrix
// untouched (dcode == NULL) otherwise.
static int build_dict(krb_matrix *A, cudaStream_t st) {
  const int64_t n = A->n, nnz = A->nnz;
  if (A->format != 2 || A->perm || n == 0 || nnz == 0) return KRB_OK;
  int32_t *off = nullptr, *sorted = nullptr, *uniq = nullptr;
  int *d_num = nullptr;
  KRB_CHECK_CUDA(dev_alloc((void **)&off, sizeof(int32_t) * nnz, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&sorted, sizeof(int32_t) * nnz, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&uniq, sizeof(int32_t) * nnz, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&d_num, sizeof(int), st));
  k_row_offsets<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, A->rp, A->ci, off);
  KRB_CHECK_LAUNCH();
  void *tmp = nullptr;
  size_t tb1 = 0, tb2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb1, off, sorted, (int)nnz, 0, 32, st);
  cub::DeviceSelect::Unique(nullptr, tb2, sorted, uniq, d_num, (int)nnz, st);
  KRB_CHECK_CUDA(dev_alloc(&tmp, tb1 > tb2 ? tb1 : tb2, st));
  cub::DeviceRadixSort::SortKeys(tmp, tb1, off, sorted, (int)nnz, 0, 32, st);
  cub::DeviceSelect::Unique(tmp, tb2, sorted, uniq, d_num, (int)nnz, st);
  KRB_CHECK_CUDA(cudaGetLastError());
  int num = 0;
  KRB_CHECK_CUDA(cudaMemcpyAsync(&num, d_num, sizeof(int), cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  dev_free(tmp, st);
  dev_free(off, st);
  dev_free(sorted, st);
  dev_free(d_num, st);
  if (num < 1 || num > 255) {
    dev_free(uniq, st);
    return KRB_OK;
  }
  KRB_CHECK_CUDA(dev_alloc((void **)&A->dict, sizeof(int32_t) * 256, st));
  KRB_CHECK_CUDA(cudaMemsetAsync(A->dict, 0, sizeof(int32_t) * 256, st));
  KRB_CHECK_CUDA(cudaMemcpyAsync(A->dict, uniq, sizeof(int32_t) * num,
                                 cudaMemcpyDeviceToDevice, st));
  A->ndict = num;
  const int64_t ns = A->nslices;
  int64_t *bytes = nullptr, *cptr = nullptr;
  uint8_t *uni = nullptr;
  KRB_CHECK_CUDA(dev_alloc((void **)&bytes, sizeof(int64_t) * (ns + 1), st));
  KRB_CHECK_CUDA(dev_alloc((void **)&cptr, sizeof(int64_t) * (ns + 1), st));
  unsigned long long *nuni = nullptr;
  KRB_CHECK_CUDA(dev_alloc((void **)&uni, ns, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&nuni, sizeof(unsigned long long), st));
  KRB_CHECK_CUDA(cudaMemsetAsync(bytes + ns, 0, sizeof(int64_t), st));
  KRB_CHECK_CUDA(cudaMemsetAsync(nuni, 0, sizeof(unsigned long long), st));
  const unsigned wb = (unsigned)((ns * 32 + 255) / 256);
  k_dict_classify<<<wb, 256, 0, st>>>(n, ns, A->sl_ptr, A->rlen, A->s_col, bytes, uni, nuni);
  KRB_CHECK_LAUNCH();
  tb1 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb1, bytes, cptr, ns + 1, st);
  KRB_CHECK_CUDA(dev_alloc(&tmp, tb1, st));
  cub::DeviceScan::ExclusiveSum(tmp, tb1, bytes, cptr, ns + 1, st);
  KRB_CHECK_CUDA(cudaGetLastError());
  int64_t total = 0;
  KRB_CHECK_CUDA(cudaMemcpyAsync(&total, cptr + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaMemcpyAsync(&A->uniform_slices, nuni, sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  dev_free(tmp, st);
  KRB_CHECK_CUDA(dev_alloc((void **)&A->dcode, total > 0 ? total : 1, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&A->dptr, sizeof(int64_t) * ns, st));
  k_dict_fill<<<wb, 256, 0, st>>>(n, ns, A->sl_ptr, A->rlen, A->s_col, A->dict, num, cptr, uni,
                                  A->dcode, A->dptr);
  KRB_CHECK_LAUNCH();
  // one CSR entry per offset code (where the value tables take their values)
  KRB_CHECK_CUDA(dev_alloc((void **)&A->rep, sizeof(int32_t) * 256, st));
  KRB_CHECK_CUDA(cudaMemsetAsync(A->rep, 0xff, sizeof(int32_t) * 256, st));
  k_dict_rep<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, A->rp, A->ci, A->dict, num, A->rep);
  KRB_CHECK_LAUNCH();
  dev_free(bytes, st);
  dev_free(cptr, st);
  dev_free(uni, st);
  dev_free(nuni, st);
  dev_free(uniq, st);
  A->dcode_bytes = total;
  A->bytes += total + ns * 8 + 256 * 8;
  return KRB_OK;
}
static int build_templates(krb_matrix *A, cudaStream_t st);

// ---- value tables of a value-coded matrix (krb_internal.cuh) --------------
// flag[d] = 1 where some entry of diagonal d differs (bitwise) from vtab[d]
__global__ void __launch_bounds__(256) k_vc_check(int64_t n, const int64_t *__restrict__ rp,
                                                  const int32_t *__restrict__ ci,
                                                  const double *__restrict__ val,
                                                  const int32_t *__restrict__ dict, int nd,
                                                  const double *__restrict__ vtab,
                                                  int *__restrict__ varies) {
  __shared__ int32_t sd[256];
  __shared__ unsigned long long sv[256];
  __shared__ int sf[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) {
    sd[t] = dict[t];
    sv[t] = (unsigned long long)__double_as_longlong(vtab[t]);
    sf[t] = 0;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    for (int64_t jj = rp[i]; jj < rp[i + 1]; ++jj) {
      const int code = dict_code(sd, nd, ci[jj] - (int32_t)i);
      // (a non-finite value counts as varying: the diagonal-form kernel
      // multiplies table values by zero for absent entries)
      const double v = val[jj];
      if (((unsigned long long)__double_as_longlong(v) != sv[code] || !isfinite(v)) && !sf[code])
        sf[code] = 1;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nd; t += blockDim.x)
    if (sf[t] && !varies[t]) varies[t] = 1;
}

__global__ void k_vc_pick(int nd, const int32_t *__restrict__ rep, const double *__restrict__ val,
                          double *__restrict__ vtab) {
  const int t = threadIdx.x;
  if (t < 256) vtab[t] = (t < nd && rep[t] >= 0) ? val[rep[t]] : 0.0;
}

// flag bytes behind the table; values of the varying diagonals zeroed
__global__ void k_vc_flags(int nd, const int *__restrict__ varies, double *__restrict__ vtab) {
  const int t = threadIdx.x;
  uint8_t *fl = reinterpret_cast<uint8_t *>(vtab + 256);
  if (t < 256) fl[t] = (t < nd && !varies[t]) ? 1 : 0;
}

// ---- row templates (pattern level) ----------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  return h ^ (h >> 33);
}

// hash of row i's offset sequence (length included)
__global__ void k_row_hash(int64_t n, const int64_t *__restrict__ rp,
                           const int32_t *__restrict__ ci, uint64_t *__restrict__ hash,
                           int *__restrict__ maxlen) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t b = rp[i], e = rp[i + 1];
  uint64_t h = mix64(0x243f6a8885a308d3ull, (uint64_t)(e - b));
  for (int64_t jj = b; jj < e; ++jj) h = mix64(h, (uint64_t)(uint32_t)(ci[jj] - (int32_t)i));
  hash[i] = h;
  if (e - b > 64) atomicMax(maxlen, (int)(e - b > 1 << 30 ? 1 << 30 : e - b));
}

// template of row i = position of its hash among the sorted distinct hashes;
// rep_row[t] = some row of template t (the race between writers is benign)
__global__ void k_row_tid(int64_t n, const uint64_t *__restrict__ hash,
                          const uint64_t *__restrict__ uniq, int nt, int32_t *__restrict__ tid,
                          int32_t *__restrict__ rep_row) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t h = hash[i];
  int lo = 0, hi = nt - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (uniq[mid] < h) lo = mid + 1; else hi = mid;
  }
  tid[i] = lo;
  if (rep_row[lo] < 0) rep_row[lo] = (int32_t)i;
}

// template t <- the codes of its representative row
__global__ void k_tmpl_fill(int nt, const int32_t *__restrict__ rep_row,
                            const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                            const int32_t *__restrict__ dict, int nd, int32_t *__restrict__ tlen,
                            uint8_t *__restrict__ tcode) {
  __shared__ int32_t sd[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) sd[t] = dict[t];
  __syncthreads();
  const int t = blockIdx.x, j = threadIdx.x;
  const int64_t r = rep_row[t];
  const int64_t b = rp[r];
  const int len = (int)(rp[r + 1] - b);
  if (j == 0) tlen[t] = len;
  if (j < 64) tcode[64 * t + j] = j < len ? (uint8_t)dict_code(sd, nd, ci[b + j] - (int32_t)r) : 0;
}

// every row against its template (a hash collision clears *ok); rows per template
__global__ void __launch_bounds__(256) k_tmpl_verify(int64_t n, const int64_t *__restrict__ rp,
                                                     const int32_t *__restrict__ ci,
                                                     const int32_t *__restrict__ dict,
                                                     const int32_t *__restrict__ tid,
                                                     const int32_t *__restrict__ tlen,
                                                     const uint8_t *__restrict__ tcode,
                                                     unsigned long long *__restrict__ rows_of,
                                                     int *__restrict__ ok) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < n;
  const int t = valid ? tid[i] : -1;
  if (valid) {
    const int64_t b = rp[i];
    const int len = (int)(rp[i + 1] - b);
    bool same = len == tlen[t];
    for (int j = 0; same && j < len; ++j)
      same = ci[b + j] - (int32_t)i == dict[tcode[64 * t + j]];
    if (!same) *ok = 0;
  }
  // one atomic per group of lanes with the same template
  const unsigned grp = __match_any_sync(0xffffffffu, t);
  if (valid && (threadIdx.x & 31) == __ffs(grp) - 1)
    atomicAdd(rows_of + t, (unsigned long long)__popc(grp));
}

// Row templates of an offset-coded pattern: rows with the same offset
// sequence share template tid[i] (C5: the 27 boundary combinations of the
// 27-point stencil).  Left unbuilt (tid == NULL) when a row is longer than 64
// or there are more than 1024 distinct sequences.
constexpr int kMaxTemplates = 1024;
static int build_templates(krb_matrix *A, cudaStream_t st) {
  const int64_t n = A->n;
  if (!A->dcode || n == 0 || A->nnz == 0) return KRB_OK;
  uint64_t *hash = nullptr, *sorted = nullptr, *uniq = nullptr;
  int *d_num = nullptr;
  KRB_CHECK_CUDA(dev_alloc((void **)&hash, sizeof(uint64_t) * n, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&sorted, sizeof(uint64_t) * n, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&uniq, sizeof(uint64_t) * n, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&d_num, 2 * sizeof(int), st));
  KRB_CHECK_CUDA(cudaMemsetAsync(d_num, 0, 2 * sizeof(int), st));
  const unsigned rb = (unsigned)((n + 255) / 256);
  k_row_hash<<<rb, 256, 0, st>>>(n, A->rp, A->ci, hash, d_num + 1);
  KRB_CHECK_LAUNCH();
  void *tmp = nullptr;
  size_t tb1 = 0, tb2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb1, hash, sorted, (int)n, 0, 64, st);
  cub::DeviceSelect::Unique(nullptr, tb2, sorted, uniq, d_num, (int)n, st);
  KRB_CHECK_CUDA(dev_alloc(&tmp, tb1 > tb2 ? tb1 : tb2, st));
  cub::DeviceRadixSort::SortKeys(tmp, tb1, hash, sorted, (int)n, 0, 64, st);
  cub::DeviceSelect::Unique(tmp, tb2, sorted, uniq, d_num, (int)n, st);
  KRB_CHECK_CUDA(cudaGetLastError());
  int h_num[2] = {0, 0};
  KRB_CHECK_CUDA(cudaMemcpyAsync(h_num, d_num, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  dev_free(tmp, st);
  dev_free(sorted, st);
  const int nt = h_num[0];
  int rc = KRB_OK;
  int32_t *rep_row = nullptr;
  unsigned long long *rows_of = nullptr;
  int *ok = nullptr;
  if (nt >= 1 && nt <= kMaxTemplates && h_num[1] <= 64) {
    auto chk = [&](cudaError_t e) {
      if (e != cudaSuccess && rc == KRB_OK) {
        set_error("build_templates: %s", cudaGetErrorString(e));
        rc = KRB_ECUDA;
      }
    };
    chk(dev_alloc((void **)&A->tid, sizeof(int32_t) * n, st));
    chk(dev_alloc((void **)&A->tlen, sizeof(int32_t) * nt, st));
    chk(dev_alloc((void **)&A->tcode, 64 * (size_t)nt, st));
    chk(dev_alloc((void **)&rep_row, sizeof(int32_t) * nt, st));
    chk(dev_alloc((void **)&rows_of, sizeof(unsigned long long) * nt, st));
    chk(dev_alloc((void **)&ok, sizeof(int), st));
    if (rc == KRB_OK) {
      chk(cudaMemsetAsync(rep_row, 0xff, sizeof(int32_t) * nt, st));
      chk(cudaMemsetAsync(rows_of, 0, sizeof(unsigned long long) * nt, st));
      const int one = 1;
      chk(cudaMemcpyAsync(ok, &one, sizeof(int), cudaMemcpyHostToDevice, st));
      k_row_tid<<<rb, 256, 0, st>>>(n, hash, uniq, nt, A->tid, rep_row);
      k_tmpl_fill<<<nt, 64, 0, st>>>(nt, rep_row, A->rp, A->ci, A->dict, A->ndict, A->tlen,
                                     A->tcode);
      k_tmpl_verify<<<rb, 256, 0, st>>>(n, A->rp, A->ci, A->dict, A->tid, A->tlen, A->tcode,
                                        rows_of, ok);
      launch_counter() += 3;
      chk(cudaGetLastError());
      std::vector<int32_t> h_len(nt);
      std::vector<uint8_t> h_code(64 * (size_t)nt);
      std::vector<unsigned long long> h_rows(nt);
      int h_ok = 0;
      chk(cudaMemcpyAsync(h_len.data(), A->tlen, sizeof(int32_t) * nt, cudaMemcpyDeviceToHost,
                          st));
      chk(cudaMemcpyAsync(h_code.data(), A->tcode, 64 * (size_t)nt, cudaMemcpyDeviceToHost, st));
      chk(cudaMemcpyAsync(h_rows.data(), rows_of, sizeof(unsigned long long) * nt,
                          cudaMemcpyDeviceToHost, st));
      chk(cudaMemcpyAsync(&h_ok, ok, sizeof(int), cudaMemcpyDeviceToHost, st));
      chk(cudaStreamSynchronize(st));
      if (rc == KRB_OK && h_ok) {
        A->ntmpl = nt;
        int mx = 1;
        A->code_count = new int64_t[512]();
        std::vector<uint64_t> h_mask(nt, 0);
        bool sorted_rows = A->ndict <= 32;
        for (int t = 0; t < nt; ++t) {
          if (h_len[t] > mx) mx = h_len[t];
          for (int j = 0; j < h_len[t]; ++j) {
            const int code = h_code[64 * (size_t)t + j];
            A->code_count[code] += (int64_t)h_rows[t];
            // (strictly ascending codes <=> the row is sorted by column)
            if (j > 0 && code <= h_code[64 * (size_t)t + j - 1]) sorted_rows = false;
            if (code < 64) h_mask[t] |= 1ull << code;
          }
        }
        A->tstride = (mx + 3) / 4 * 4;
        A->bytes += 4 * n + 68 * (int64_t)nt;
        {   // the offsets on the host (diagonal tables are assembled there)
          int32_t h_dict[256];
          chk(cudaMemcpyAsync(h_dict, A->dict, sizeof(h_dict), cudaMemcpyDeviceToHost, st));
          chk(cudaStreamSynchronize(st));
          for (int d = 0; d < 256; ++d) A->code_count[256 + d] = h_dict[d];
        }
        // diagonal form: rows sorted by column, <= 32 diagonals, at least
        // half of the n x ndict positions filled
        if (rc == KRB_OK && sorted_rows && 2 * A->nnz >= n * (int64_t)A->ndict) {
          chk(dev_alloc((void **)&A->tmask, sizeof(uint64_t) * nt, st));
          if (rc == KRB_OK)
            chk(cudaMemcpyAsync(A->tmask, h_mask.data(), sizeof(uint64_t) * nt,
                                cudaMemcpyHostToDevice, st));
          chk(cudaStreamSynchronize(st));
          A->bytes += 8 * (int64_t)nt;
        }
      }
    }
    if (rc != KRB_OK || !A->ntmpl) {   // no templates (hash collision: practically never)
      for (void *p : {(void *)A->tid, (void *)A->tlen, (void *)A->tcode, (void *)A->tmask})
        if (p) dev_free(p, st);
      A->tid = nullptr; A->tlen = nullptr; A->tcode = nullptr; A->tmask = nullptr;
      A->ntmpl = 0;
    }
  }
  for (void *p : {(void *)hash, (void *)uniq, (void *)d_num, (void *)rep_row, (void *)rows_of,
                  (void *)ok})
    if (p) dev_free(p, st);
  return rc;
}

// tent[tstride t + j] = {offset, constant?, value} of entry j of template t
__global__ void k_tent_fill(int ntmpl, int tstride, const int32_t *__restrict__ tlen,
                            const uint8_t *__restrict__ tcode, const int32_t *__restrict__ dict,
                            const double *__restrict__ vtab, krb_tentry *__restrict__ tent) {
  const int t = blockIdx.x, j = threadIdx.x;
  if (t >= ntmpl || j >= tstride) return;
  const uint8_t *fl = reinterpret_cast<const uint8_t *>(vtab + 256);
  krb_tentry e = {0, 1, 0.0};
  if (j < tlen[t]) {
    const int code = tcode[64 * t + j];
    e.off = dict[code];
    e.cst = fl[code] ? 1 : 0;
    e.val = fl[code] ? vtab[code] : 0.0;
  }
  tent[(int64_t)tstride * t + j] = e;
}

static int64_t vcode_bytes(const krb_matrix *A) {
  return A->tent ? 256 * 8 + 256 + (int64_t)A->ntmpl * A->tstride * 16 : 0;
}

static void free_vcode(krb_matrix *A, cudaStream_t st) {
  for (void *p : {(void *)A->vtab, (void *)A->tent})
    if (p) dev_free(p, st);
  A->vtab = nullptr; A->tent = nullptr;
  A->vconst_entries = 0;
  A->dia = krb_diatable();
}

// Build the value tables of an offset-coded matrix with row templates; kept
// when at least half of the entries lie on constant diagonals (otherwise the
// matrix stays plainly offset-coded).  One pass over the CSR copy (~1 ms at
// C5) and two tiny kernels.
static int build_vcode(krb_matrix *A, cudaStream_t st) {
  if (!A->dcode || !A->rep || !A->tid || !A->code_count || A->n == 0 || A->nnz == 0 ||
      tuning().value_coding == 0)
    return KRB_OK;
  const int nd = A->ndict;
  int *varies = nullptr;
  KRB_CHECK_CUDA(dev_alloc((void **)&A->vtab, 256 * sizeof(double) + 256, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&varies, 256 * sizeof(int), st));
  KRB_CHECK_CUDA(cudaMemsetAsync(varies, 0, 256 * sizeof(int), st));
  k_vc_pick<<<1, 256, 0, st>>>(nd, A->rep, A->val, A->vtab);
  KRB_CHECK_LAUNCH();
  k_vc_check<<<(unsigned)((A->n + 255) / 256), 256, 0, st>>>(A->n, A->rp, A->ci, A->val, A->dict,
                                                             nd, A->vtab, varies);
  KRB_CHECK_LAUNCH();
  k_vc_flags<<<1, 256, 0, st>>>(nd, varies, A->vtab);
  KRB_CHECK_LAUNCH();
  double h_vtab[256 + 32];
  KRB_CHECK_CUDA(cudaMemcpyAsync(h_vtab, A->vtab, sizeof(h_vtab), cudaMemcpyDeviceToHost, st));
  KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  const uint8_t *fl = reinterpret_cast<const uint8_t *>(h_vtab + 256);
  dev_free(varies, st);
  int64_t cnt = 0;
  for (int d = 0; d < nd; ++d)
    if (fl[d]) cnt += A->code_count[d];
  if (2 * cnt < A->nnz) {
    free_vcode(A, st);
    return KRB_OK;
  }
  A->vconst_entries = cnt;
  A->dia = krb_diatable();
  if (A->tmask && nd <= 32) {
    A->dia.nd = nd;
    for (int d = 0; d < nd; ++d) {
      A->dia.off[d] = (int32_t)A->code_count[256 + d];
      A->dia.val[d] = fl[d] ? h_vtab[d] : 0.0;
      if (fl[d]) A->dia.cst |= 1ull << d;
    }
  }
  KRB_CHECK_CUDA(dev_alloc((void **)&A->tent, sizeof(krb_tentry) * (size_t)A->ntmpl * A->tstride, st));
  k_tent_fill<<<A->ntmpl, 64, 0, st>>>(A->ntmpl, A->tstride, A->tlen, A->tcode, A->dict, A->vtab,
                                       A->tent);
  KRB_CHECK_LAUNCH();
  A->bytes += vcode_bytes(A);
  return KRB_OK;
}

// ---- shared sparsity patterns --------------------------------------------
// Matrices of a sequence (A_j = s_j E - K: the same row_ptr / col_idx, new
// values) share their structure work: the SELL layout, the offset codes and
// the transpose's permutation are built once and reused while any matrix of
// that pattern is alive (found by comparing the new index arrays on the
// device against every live pattern of the same size).
}  // namespace krb

struct krb_pattern {
  int refs = 0;
  int64_t n = 0, nnz = 0;
  int req_format = 0, format = 0, ndict = 0;
  int64_t nslices = 0, sell_elems = 0, dcode_bytes = 0, uniform_slices = 0, bytes = 0;
  int64_t *rp = nullptr, *sl_ptr = nullptr, *dptr = nullptr;
  int32_t *ci = nullptr, *rlen = nullptr, *s_col = nullptr, *perm = nullptr, *dict = nullptr;
  uint8_t *dcode = nullptr;
  int32_t *rep = nullptr;
  int32_t *tid = nullptr, *tlen = nullptr;
  uint8_t *tcode = nullptr;
  int ntmpl = 0, tstride = 0;
  int64_t *code_count = nullptr;   // host: entries per offset code, then the 256 offsets
  uint64_t *tmask = nullptr;
  krb_pattern *tpat = nullptr;   // pattern of the transpose (may be this one)
  int32_t *tperm = nullptr;      // transpose entry t = this pattern's CSR entry tperm[t]
};

namespace krb {

static std::vector<krb_pattern *> &patterns() {
  static std::vector<krb_pattern *> v;
  return v;
}
static std::recursive_mutex &patterns_mu() {
  static std::recursive_mutex m;
  return m;
}
void matrix_free(krb_matrix *A, bool async, cudaStream_t st);

static void pattern_release(krb_pattern *P, bool async, cudaStream_t st) {
  std::lock_guard<std::recursive_mutex> lk(patterns_mu());
  if (!P || --P->refs > 0) return;
  auto &v = patterns();
  for (size_t i = 0; i < v.size(); ++i)
    if (v[i] == P) { v.erase(v.begin() + i); break; }
  void *arrays[] = {P->rp, P->ci, P->sl_ptr, P->rlen, P->s_col, P->perm,
                    P->dcode, P->dptr, P->dict, P->tperm, P->rep, P->tid, P->tlen, P->tcode, P->tmask};
  for (void *p : arrays)
    if (p) dev_free(p, async ? st : nullptr);
  delete[] P->code_count;
  krb_pattern *T = P->tpat;
  delete P;
  if (T && T != P) pattern_release(T, async, st);
}

// move the structure arrays of a freshly built matrix into a new pattern
static void pattern_adopt(krb_matrix *A) {
  std::lock_guard<std::recursive_mutex> lk(patterns_mu());
  krb_pattern *P = new krb_pattern();
  P->refs = 1;
  P->n = A->n; P->nnz = A->nnz; P->req_format = A->req_format; P->format = A->format;
  P->ndict = A->ndict; P->nslices = A->nslices; P->sell_elems = A->sell_elems;
  P->dcode_bytes = A->dcode_bytes; P->uniform_slices = A->uniform_slices;
  P->rp = A->rp; P->ci = A->ci; P->sl_ptr = A->sl_ptr; P->rlen = A->rlen; P->s_col = A->s_col;
  P->perm = A->perm; P->dcode = A->dcode; P->dptr = A->dptr; P->dict = A->dict;
  P->rep = A->rep; P->tid = A->tid; P->tlen = A->tlen; P->tcode = A->tcode;
  P->ntmpl = A->ntmpl; P->tstride = A->tstride; P->code_count = A->code_count;
  P->tmask = A->tmask;
  P->bytes = A->bytes - 8 * A->nnz - (A->s_val ? 8 * A->sell_elems : 0) - vcode_bytes(A);
  A->pat = P;
  patterns().push_back(P);
}

static void pattern_attach(krb_matrix *A, krb_pattern *P) {
  std::lock_guard<std::recursive_mutex> lk(patterns_mu());
  P->refs++;
  A->pat = P;
  A->format = P->format; A->ndict = P->ndict; A->nslices = P->nslices;
  A->sell_elems = P->sell_elems; A->dcode_bytes = P->dcode_bytes;
  A->uniform_slices = P->uniform_slices;
  A->rp = P->rp; A->ci = P->ci; A->sl_ptr = P->sl_ptr; A->rlen = P->rlen; A->s_col = P->s_col;
  A->perm = P->perm; A->dcode = P->dcode; A->dptr = P->dptr; A->dict = P->dict;
  A->rep = P->rep; A->tid = P->tid; A->tlen = P->tlen; A->tcode = P->tcode;
  A->ntmpl = P->ntmpl; A->tstride = P->tstride; A->code_count = P->code_count;
  A->tmask = P->tmask;
}

__global__ void k_pattern_neq(int64_t n, int64_t nnz, const int64_t *__restrict__ rp_a,
                              const int64_t *__restrict__ rp_b, const int32_t *__restrict__ ci_a,
                              const int32_t *__restrict__ ci32_b,
                              const int64_t *__restrict__ ci64_b, int *neq) {
  const int64_t m = n + 1 > nnz ? n + 1 : nnz;
  bool diff = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i <= n && rp_a[i] != rp_b[i]) diff = true;
    if (i < nnz && ci_a[i] != (ci32_b ? ci32_b[i] : (int32_t)ci64_b[i])) diff = true;
  }
  if (__syncthreads_or(diff) && threadIdx.x == 0) *neq = 1;
}

static krb_pattern *pattern_find(int64_t n, int64_t nnz, int req_format, const int64_t *d_rp,
                                 const int32_t *d_ci32, const int64_t *d_ci64,
                                 cudaStream_t st) {
  std::lock_guard<std::recursive_mutex> lk(patterns_mu());
  int *flag = nullptr;
  for (krb_pattern *P : patterns()) {
    if (P->n != n || P->nnz != nnz || P->req_format != req_format) continue;
    if (!flag && dev_alloc((void **)&flag, sizeof(int), st) != cudaSuccess) return nullptr;
    int h = 0;
    if (cudaMemsetAsync(flag, 0, sizeof(int), st) != cudaSuccess) break;
    const int64_t m = n + 1 > nnz ? n + 1 : nnz;
    k_pattern_neq<<<(unsigned)((m + 1023) / 1024), 256, 0, st>>>(n, nnz, P->rp, d_rp, P->ci,
                                                                 d_ci32, d_ci64, flag);
    launch_counter()++;
    if (cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      break;
    if (h == 0) {
      dev_free(flag, st);
      return P;
    }
  }
  if (flag) dev_free(flag, st);
  cudaGetLastError();
  return nullptr;
}

// values of row p's slice column (padding slots of the row zeroed: no
// separate pass over the padded array)
__global__ void k_sell_fill_vals(int64_t n, const int64_t *__restrict__ rp,
                                 const double *__restrict__ val,
                                 const int64_t *__restrict__ sl_ptr,
                                 const int32_t *__restrict__ perm, double *__restrict__ s_val) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t row = perm ? perm[p] : p;
  const int64_t s0 = sl_ptr[p >> 5], width = (sl_ptr[(p >> 5) + 1] - s0) / 32;
  const int64_t base = s0 + (p & 31);
  const int64_t b = rp[row], e = rp[row + 1];
  for (int64_t j = 0; j < width; ++j) s_val[base + 32 * j] = b + j < e ? val[b + j] : 0.0;
}

// the SELL values of a matrix attached to a pattern
static int fill_values(krb_matrix *A, cudaStream_t st) {
  if (A->format != 2 || A->n == 0) return KRB_OK;
  const int64_t total = A->sell_elems;
  KRB_CHECK_CUDA(dev_alloc((void **)&A->s_val, sizeof(double) * (total > 0 ? total : 1), st));
  // (slots of the missing lanes of a partial last slice stay unwritten:
  // no row reads them)
  k_sell_fill_vals<<<(unsigned)((A->n + 255) / 256), 256, 0, st>>>(A->n, A->rp, A->val,
                                                                   A->sl_ptr, A->perm, A->s_val);
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int matrix_create(krb_matrix **out, int64_t n, int64_t nnz,
                  const int64_t *d_rp, const int32_t *d_ci32,
                  const int64_t *d_ci64, const double *d_val, int format,
                  cudaStream_t st) {
  KRB_REQUIRE(out != nullptr, "krb_matrix_create: out is NULL");
  KRB_REQUIRE(n >= 0 && nnz >= 0, "krb_matrix_create: negative size");
  KRB_REQUIRE(nnz < ((int64_t)1 << 31), "krb_matrix_create: nnz >= 2^31");
  KRB_REQUIRE(n < ((int64_t)1 << 31), "krb_matrix_create: n >= 2^31");
  static bool pool_ready = false;
  if (!pool_ready) {
    // keep up to 4 GB of freed blocks in the default pool: re-creating a
    // small sequence's matrices every step must not pay cudaMalloc /
    // implicit syncs again, while the blocks of large matrices (a C5 matrix
    // with its transpose is ~22 GB) go back to the device at the next
    // synchronisation, where the caller's allocator (torch) can reuse them
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = (uint64_t)4 << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_ready = true;
  }
  krb_matrix *A = new krb_matrix();
  A->n = n;
  A->nnz = nnz;
  A->req_format = format;
  A->uid = next_uid();
  if (krb_pattern *P = pattern_find(n, nnz, format, d_rp, d_ci32, d_ci64, st)) {
    pattern_attach(A, P);
    cudaError_t e = dev_alloc((void **)&A->val, sizeof(double) * (nnz > 0 ? nnz : 1), st);
    if (e != cudaSuccess) {
      set_error("krb_matrix_create: %s", cudaGetErrorString(e));
      pattern_release(P, true, st);
      delete A;
      return KRB_ENOMEM;
    }
    if (nnz > 0)
      KRB_CHECK_CUDA(cudaMemcpyAsync(A->val, d_val, sizeof(double) * nnz,
                                     cudaMemcpyDeviceToDevice, st));
    int rc = fill_values(A, st);
    A->bytes = P->bytes + 8 * nnz + (A->s_val ? 8 * A->sell_elems : 0);
    if (rc == KRB_OK) rc = build_vcode(A, st);
    if (rc != KRB_OK) {
      matrix_free(A, true, st);
      return rc;
    }
    *out = A;
    return KRB_OK;
  }
  cudaError_t e = dev_alloc((void **)&A->rp, sizeof(int64_t) * (n + 1), st);
  if (e == cudaSuccess) e = dev_alloc((void **)&A->ci, sizeof(int32_t) * (nnz > 0 ? nnz : 1), st);
  if (e == cudaSuccess) e = dev_alloc((void **)&A->val, sizeof(double) * (nnz > 0 ? nnz : 1), st);
  if (e != cudaSuccess) {
    set_error("krb_matrix_create: %s", cudaGetErrorString(e));
    dev_free(A->rp, st); dev_free(A->ci, st); dev_free(A->val, st);
    delete A;
    return KRB_ENOMEM;
  }
  KRB_CHECK_CUDA(cudaMemcpyAsync(A->rp, d_rp, sizeof(int64_t) * (n + 1),
                                 cudaMemcpyDeviceToDevice, st));
  if (nnz > 0) {
    if (d_ci32)
      KRB_CHECK_CUDA(cudaMemcpyAsync(A->ci, d_ci32, sizeof(int32_t) * nnz,
                                     cudaMemcpyDeviceToDevice, st));
    else {
      k_i64_to_i32<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(nnz, d_ci64, A->ci);
      KRB_CHECK_LAUNCH();
    }
    KRB_CHECK_CUDA(cudaMemcpyAsync(A->val, d_val, sizeof(double) * nnz,
                                   cudaMemcpyDeviceToDevice, st));
  }
  A->bytes = (n + 1) * 8 + nnz * 12;
  // 4 = SELL-32 with the offset-coded stream (when the matrix qualifies);
  // 2 = plain SELL-32; 0 = auto (the offset-coded stream when it qualifies)
  int rc = build_sell(A, format == 4 ? 2 : format, st);
  if (rc == KRB_OK && (format == 0 || format == 4)) rc = build_dict(A, st);
  if (rc == KRB_OK) rc = build_templates(A, st);
  if (rc == KRB_OK) rc = build_vcode(A, st);
  if (rc != KRB_OK) {
    delete A;
    return rc;
  }
  pattern_adopt(A);
  *out = A;
  return KRB_OK;
}

__global__ void k_entry_rows(int64_t n, const int64_t *__restrict__ rp,
                             int32_t *__restrict__ rows) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t jj = rp[i]; jj < rp[i + 1]; ++jj) rows[jj] = (int32_t)i;
}


__global__ void k_col_count(int64_t nnz, const int32_t *__restrict__ ci,
                            int64_t *__restrict__ cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nnz) atomicAdd(reinterpret_cast<unsigned long long *>(cnt + ci[i]), 1ull);
}

__global__ void k_gather_vals(int64_t nnz, const int32_t *__restrict__ perm,
                              const double *__restrict__ val, double *__restrict__ tval) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nnz) tval[t] = val[perm[t]];
}

__global__ void k_gather_t(int64_t nnz, const int32_t *__restrict__ perm,
                           const int32_t *__restrict__ rows,
                           const double *__restrict__ val,
                           int32_t *__restrict__ tci, double *__restrict__ tval) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  int32_t p = perm[t];
  tci[t] = rows[p];
  tval[t] = val[p];
}

int ensure_transpose(krb_matrix *A, cudaStream_t st) {
  if (A->T) return KRB_OK;
  if (A->borrowed) {
    // operator view: its adjoint is a view of the base's transpose carrying
    // the same factors (applied as the adjoint composite)
    KRB_TRY(ensure_transpose(A->base, st));
    krb_matrix *T = new krb_matrix(*A->base->T);
    T->T = nullptr;
    T->base = A->base->T;
    T->borrowed = true;
    T->pre = A->pre;
    T->pre_adj = !A->pre_adj;
    A->T = T;
    return KRB_OK;
  }
  const int64_t n = A->n, nnz = A->nnz;
  krb_pattern *P = A->pat;
  if (P && P->tpat) {
    // the pattern's transpose is known: values by one gather through its
    // permutation, structure shared
    krb_matrix *T = new krb_matrix();
    T->n = n;
    T->nnz = nnz;
    T->uid = next_uid();
    T->req_format = P->tpat->req_format;
    pattern_attach(T, P->tpat);
    KRB_CHECK_CUDA(dev_alloc((void **)&T->val, sizeof(double) * (nnz > 0 ? nnz : 1), st));
    if (nnz > 0) {
      k_gather_vals<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(nnz, P->tperm, A->val, T->val);
      KRB_CHECK_LAUNCH();
    }
    int rc = fill_values(T, st);
    T->bytes = P->tpat->bytes + 8 * nnz + (T->s_val ? 8 * T->sell_elems : 0);
    if (rc == KRB_OK) rc = build_vcode(T, st);
    if (rc != KRB_OK) {
      matrix_free(T, true, st);
      return rc;
    }
    A->T = T;
    return KRB_OK;
  }
  int32_t *rows = nullptr, *keys_out = nullptr, *perm_in = nullptr,
          *perm_out = nullptr, *tci = nullptr;
  int64_t *cnt = nullptr, *trp = nullptr;
  double *tval = nullptr;
  size_t m = nnz > 0 ? nnz : 1;
  KRB_CHECK_CUDA(dev_alloc((void **)&rows, sizeof(int32_t) * m, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&keys_out, sizeof(int32_t) * m, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&perm_in, sizeof(int32_t) * m, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&perm_out, sizeof(int32_t) * m, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&cnt, sizeof(int64_t) * (n + 1), st));
  KRB_CHECK_CUDA(dev_alloc((void **)&trp, sizeof(int64_t) * (n + 1), st));
  KRB_CHECK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (n + 1), st));
  unsigned nb = (unsigned)((nnz + 255) / 256), rb = (unsigned)((n + 255) / 256);
  if (n > 0) {
    k_entry_rows<<<rb, 256, 0, st>>>(n, A->rp, rows);
    KRB_CHECK_LAUNCH();
  }
  if (nnz > 0) {
    k_iota<<<nb, 256, 0, st>>>(nnz, perm_in);
    KRB_CHECK_LAUNCH();
    k_col_count<<<nb, 256, 0, st>>>(nnz, A->ci, cnt);
    KRB_CHECK_LAUNCH();
  }
  void *tmp = nullptr;
  size_t tb1 = 0, tb2 = 0;
  int end_bit = 1;
  while (end_bit < 31 && ((int64_t)1 << end_bit) < n) ++end_bit;
  cub::DeviceRadixSort::SortPairs(nullptr, tb1, A->ci, keys_out, perm_in,
                                  perm_out, (int)nnz, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt, trp, n + 1, st);
  KRB_CHECK_CUDA(dev_alloc((void **)&tmp, tb1 > tb2 ? tb1 : tb2, st));
  if (nnz > 0)
    cub::DeviceRadixSort::SortPairs(tmp, tb1, A->ci, keys_out, perm_in,
                                    perm_out, (int)nnz, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(tmp, tb2, cnt, trp, n + 1, st);
  KRB_CHECK_CUDA(cudaGetLastError());
  KRB_CHECK_CUDA(dev_alloc((void **)&tci, sizeof(int32_t) * m, st));
  KRB_CHECK_CUDA(dev_alloc((void **)&tval, sizeof(double) * m, st));
  if (nnz > 0) {
    k_gather_t<<<nb, 256, 0, st>>>(nnz, perm_out, rows, A->val, tci, tval);
    KRB_CHECK_LAUNCH();
  }
  dev_free(tmp, st);
  dev_free(rows, st);
  dev_free(keys_out, st);
  dev_free(perm_in, st);
  dev_free(cnt, st);
  krb_matrix *T = nullptr;
  int rc = matrix_create(&T, n, nnz, trp, tci, nullptr, tval,
                         A->req_format == 2 || A->req_format == 4 ? A->req_format : 0, st);
  dev_free(trp, st);
  dev_free(tci, st);
  dev_free(tval, st);
  if (rc != KRB_OK) {
    dev_free(perm_out, st);
    return rc;
  }
  if (P && T->pat && !P->tpat) {
    // remember the transpose's pattern and permutation (a symmetric
    // pattern is its own transpose pattern: no counted self-reference)
    P->tpat = T->pat;
    if (T->pat != P) T->pat->refs++;
    P->tperm = perm_out;
  } else {
    dev_free(perm_out, st);
  }
  A->T = T;
  return KRB_OK;
}

// async: free stream-ordered on `st` (no device-wide synchronisation; the
// arrays return to the memory pool once the work queued on `st` before the
// call is done -- the caller guarantees no other stream still reads them);
// otherwise cudaFree (synchronises the device).
void matrix_free(krb_matrix *A, bool async, cudaStream_t st) {
  if (!A) return;
  if (A->borrowed) {   // a view: the arrays belong to its base, the factors
    if (A->T) matrix_free(A->T, async, st);   // to their krb_precond
    delete A;
    return;
  }
  matrix_free(A->T, async, st);
  if (!async) cudaDeviceSynchronize();
  if (A->pat) {   // structure arrays belong to the pattern
    for (void *p : {(void *)A->val, (void *)A->s_val, (void *)A->vtab, (void *)A->tent})
      if (p) dev_free(p, async ? st : nullptr);
    pattern_release(A->pat, async, st);
  } else {
    void *arrays[] = {A->rp, A->ci, A->val, A->sl_ptr, A->rlen, A->s_col, A->s_val, A->perm,
                      A->dcode, A->dptr, A->dict, A->rep, A->vtab, A->tent, A->tid, A->tlen,
                      A->tcode, A->tmask};
    for (void *p : arrays)
      if (p) dev_free(p, async ? st : nullptr);
    delete[] A->code_count;
  }
  delete A;
}

}  // namespace krb

using namespace krb;

extern "C" {

int krb_matrix_create(krb_matrix **out, int64_t n, int64_t nnz,
                      const int64_t *d_row_ptr, const int32_t *d_col_idx,
                      const double *d_values, int format, void *stream) {
  cudaStream_t st = as_stream(stream);
  int rc = matrix_create(out, n, nnz, d_row_ptr, d_col_idx, nullptr, d_values,
                         format, st);
  if (rc == KRB_OK) KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  return rc;
}

int krb_matrix_create_i64(krb_matrix **out, int64_t n, int64_t nnz,
                          const int64_t *d_row_ptr, const int64_t *d_col_idx,
                          const double *d_values, int format, void *stream) {
  cudaStream_t st = as_stream(stream);
  int rc = matrix_create(out, n, nnz, d_row_ptr, nullptr, d_col_idx, d_values,
                         format, st);
  if (rc == KRB_OK) KRB_CHECK_CUDA(cudaStreamSynchronize(st));
  return rc;
}

int krb_matrix_destroy(krb_matrix *A) {
  matrix_free(A, false, nullptr);
  return KRB_OK;
}

int krb_matrix_destroy_async(krb_matrix *A, void *stream) {
  matrix_free(A, true, as_stream(stream));
  return KRB_OK;
}

int krb_matrix_info(const krb_matrix *A, int64_t *n, int64_t *nnz, int *format,
                    int64_t *bytes) {
  KRB_REQUIRE(A != nullptr, "krb_matrix_info: NULL matrix");
  if (n) *n = A->n;
  if (nnz) *nnz = A->nnz;
  if (format)
    *format = (A->format == 2 && A->perm) ? 3
              : (A->tent && tuning().value_coding) ? 5 : (A->dcode ? 4 : A->format);
  if (bytes) *bytes = A->bytes + (A->T ? A->T->bytes : 0);
  return KRB_OK;
}

int krb_matrix_stream_stats(const krb_matrix *A, int64_t *stream_bytes, int64_t *nslices,
                            int64_t *uniform_slices, int *ndict) {
  KRB_REQUIRE(A != nullptr, "krb_matrix_stream_stats: NULL matrix");
  const krb_matrix *B = A->base ? A->base : A;
  int64_t b = 16 * B->n;   // x read once, y written once
  if (B->tent && tuning().value_coding)
    // value-coded: only the entries off the constant diagonals stream their
    // values; per slice the offset row / code bytes, the value row and mask
    // (values of the other entries, the rows' template ids, slice pointers, tables)
    b += 8 * (B->nnz - B->vconst_entries) + 4 * B->n + 8 * B->nslices +
         16 * (int64_t)B->ntmpl * B->tstride + 4 * B->ntmpl;
  else if (B->dcode)
    b += 8 * B->sell_elems + B->dcode_bytes + 4 * B->n + 16 * B->nslices + 1024;
  else if (B->format == 2)
    b += 12 * B->sell_elems + 4 * B->n + 8 * (B->nslices + 1) + (B->perm ? 4 * B->n : 0);
  else
    b += 12 * B->nnz + 8 * (B->n + 1);
  if (stream_bytes) *stream_bytes = b;
  if (nslices) *nslices = B->format == 2 ? B->nslices : 0;
  if (uniform_slices) *uniform_slices = B->uniform_slices;
  if (ndict) *ndict = B->ndict;
  return KRB_OK;
}

int krb_matrix_value_stats(const krb_matrix *A, int64_t *const_entries, int *templates,
                           int *const_diagonals, int *diagonal_form) {
  KRB_REQUIRE(A != nullptr, "krb_matrix_value_stats: NULL matrix");
  const krb_matrix *B = A->base ? A->base : A;
  const bool on = B->tent && tuning().value_coding;
  if (const_entries) *const_entries = on ? B->vconst_entries : 0;
  if (templates) *templates = on ? B->ntmpl : 0;
  if (diagonal_form) *diagonal_form = on && B->dia.nd && tuning().value_coding != 2 ? 1 : 0;
  if (const_diagonals) {
    *const_diagonals = 0;
    if (on) {
      uint8_t fl[256];
      KRB_CHECK_CUDA(cudaMemcpy(fl, B->vtab + 256, 256, cudaMemcpyDeviceToHost));
      for (int d = 0; d < B->ndict; ++d) *const_diagonals += fl[d] ? 1 : 0;
    }
  }
  return KRB_OK;
}

int krb_matrix_pattern_info(const krb_matrix *A, uint64_t *pattern_id, int *refs,
                            int *transpose_known) {
  KRB_REQUIRE(A != nullptr, "krb_matrix_pattern_info: NULL matrix");
  const krb_matrix *B = A->base ? A->base : A;
  std::lock_guard<std::recursive_mutex> lk(patterns_mu());
  if (pattern_id) *pattern_id = (uint64_t)(uintptr_t)B->pat;
  if (refs) *refs = B->pat ? B->pat->refs : 0;
  if (transpose_known) *transpose_known = B->pat && B->pat->tperm ? 1 : 0;
  return KRB_OK;
}

int krb_spmv(const krb_matrix *A, const double *d_x, double *d_y,
             void *stream) {
  KRB_REQUIRE(A != nullptr, "krb_spmv: NULL matrix");
  return spmv_launch(A, d_x, d_y, nullptr, as_stream(stream));
}

int krb_spmv_t(krb_matrix *A, const double *d_x, double *d_y, void *stream) {
  KRB_REQUIRE(A != nullptr, "krb_spmv_t: NULL matrix");
  int rc = ensure_transpose(A, as_stream(stream));
  if (rc) return rc;
  return spmv_launch(A->T, d_x, d_y, nullptr, as_stream(stream));
}

int krb_spmm(krb_matrix *A, int transpose, int64_t ncols, const double *d_X,
             int64_t ldx, double *d_Y, int64_t ldy, void *stream) {
  KRB_REQUIRE(A != nullptr, "krb_spmm: NULL matrix");
  KRB_REQUIRE(ldx >= A->n && ldy >= A->n, "krb_spmm: leading dimension < n");
  cudaStream_t st = as_stream(stream);
  const krb_matrix *M = A;
  if (transpose) {
    int rc = ensure_transpose(A, st);
    if (rc) return rc;
    M = A->T;
  }
  return spmm_launch(M, ncols, d_X, ldx, d_Y, ldy, st);
}

}  // extern "C"
