/*
 * oracle/canon.c -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C restatement of the floating-point primitives on the recycling
 * BiCGSTAB hot path, each evaluated in ONE fixed ("canonical") order.  The
 * B200 kernels in paper_1406_2831_b200/csrc implement exactly these orders, so
 * the GPU path and this oracle agree bit for bit; the reference's own
 * primitives (OpenBLAS ddot/dgemv, whose order depends on CPU model and thread
 * count) are compared against this oracle within the reference's own noise
 * floor.
 *
 * Reference call sites each primitive stands in for
 * (/root/reference/pkg/src/krecycle/...):
 *   canon_spmv   <- SparseMatrix.matvec / rmatvec (sparse.py:117-130), scipy
 *                   csr_matvec: per-row sequential sum from 0.0 in CSR order,
 *                   separate multiply and add (no FMA).  Bit-identical to scipy.
 *   canon_dot    <- np.vdot / np.linalg.norm (solvers.py:308-352,
 *                   recycling.py:155,159,333-335)
 *   canon_tdot   <- R.Chat.conj().T @ v (solvers.py:306,328; recycling.py:203)
 *   canon_gemv   <- R.C @ zeta, R.U @ xc (solvers.py:307,329,359)
 *   canon_gram   <- Ct_raw^H C_raw, Wt^H AW, Wt^H W (recycling.py:140,342-343)
 *   canon_gemm   <- W @ Z, U_raw @ Y (recycling.py:151-154,351-352,365-368)
 *   canon_trsv   <- the ILUTP triangular solves L^{-1}, L^{-H}, U^{-1}, U^{-H}
 *                   (ilutp.py:76-97; the reference uses SuperLU's supernodal
 *                   solve, whose order this does not reproduce)
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off; fma() is the libm
 * correctly-rounded fused multiply-add, identical to CUDA __fma_rn).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- canonical dot --------------------------------------------------------
 * E = elements per lane per block; a block is 1024 lanes x E elements.
 * Block stage : lane l accumulates x[i]*y[i] (fma) for i = b*1024E + 1024e + l,
 *               e = 0..E-1 ; then a 32-lane tree inside each warp (offsets
 *               16,8,4,2,1) and a 32-lane tree over the 32 warp results.
 * Final stage : lane L (of 32) sums block partials b = L, L+32, ... in order,
 *               then the 32-lane tree.
 * E = smallest power of two >= n / (1024 * 296), clamped to [1, 16]
 * (296 = 2 resident 1024-thread CTAs on each of the 148 SMs).             */
#define CANON_LANES 1024
#define CANON_TARGET_BLOCKS 296 /* 148 SMs x 2 */

int64_t canon_E(int64_t n) {
  int64_t t = (n + (int64_t)CANON_LANES * CANON_TARGET_BLOCKS - 1) /
              ((int64_t)CANON_LANES * CANON_TARGET_BLOCKS);
  int64_t E = 1;
  while (E < t && E < 16) E *= 2;
  return E;
}

int64_t canon_nblocks(int64_t n) {
  int64_t B = CANON_LANES * canon_E(n);
  return n <= 0 ? 0 : (n + B - 1) / B;
}

static void tree32(double *a) {
  for (int off = 16; off >= 1; off >>= 1)
    for (int l = 0; l < off; ++l) a[l] = a[l] + a[l + off];
}

static double block_partial(int64_t n, int64_t E, int64_t b, const double *x,
                            int64_t incx, const double *y, int64_t incy) {
  double lane[CANON_LANES];
  int64_t base = b * CANON_LANES * E;
  for (int l = 0; l < CANON_LANES; ++l) {
    double acc = 0.0;
    for (int64_t e = 0; e < E; ++e) {
      int64_t i = base + CANON_LANES * e + l;
      if (i < n) acc = fma(x[i * incx], y[i * incy], acc);
    }
    lane[l] = acc;
  }
  double warp[32];
  for (int w = 0; w < 32; ++w) {
    tree32(lane + 32 * w);
    warp[w] = lane[32 * w];
  }
  tree32(warp);
  return warp[0];
}

double canon_final(int64_t nb, const double *P, int64_t incp) {
  double a[32];
  for (int L = 0; L < 32; ++L) {
    double acc = 0.0;
    for (int64_t b = L; b < nb; b += 32) acc = acc + P[b * incp];
    a[L] = acc;
  }
  tree32(a);
  return a[0];
}

void canon_dot_partials(int64_t n, const double *x, int64_t incx,
                        const double *y, int64_t incy, double *P) {
  int64_t E = canon_E(n), nb = canon_nblocks(n);
  for (int64_t b = 0; b < nb; ++b) P[b] = block_partial(n, E, b, x, incx, y, incy);
}

double canon_dot(int64_t n, const double *x, int64_t incx, const double *y,
                 int64_t incy) {
  int64_t nb = canon_nblocks(n);
  if (nb == 0) return 0.0;
  double *P = (double *)malloc(sizeof(double) * nb);
  canon_dot_partials(n, x, incx, y, incy, P);
  double r = canon_final(nb, P, 1);
  free(P);
  return r;
}

/* out[j] = canon_dot(M[:,j], v); M element (i,j) at M[i*rs + j*cs]. */
void canon_tdot(int64_t n, int64_t k, const double *M, int64_t rs, int64_t cs,
                const double *v, double *out) {
  for (int64_t j = 0; j < k; ++j) out[j] = canon_dot(n, M + j * cs, rs, v, 1);
}

/* out[i] = sum_j M[i,j]*y[j], sequential in j from 0.0 with fma. */
void canon_gemv(int64_t n, int64_t k, const double *M, int64_t rs, int64_t cs,
                const double *y, double *out) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t j = 0; j < k; ++j) acc = fma(M[i * rs + j * cs], y[j], acc);
    out[i] = acc;
  }
}

/* y = A x for canonical CSR: per row sequential from 0.0, mul then add. */
void canon_spmv(int64_t n, const int64_t *rp, const int32_t *ci,
                const double *v, const double *x, double *y) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t jj = rp[i]; jj < rp[i + 1]; ++jj) {
      double prod = v[jj] * x[ci[jj]];
      s = s + prod;
    }
    y[i] = s;
  }
}

/* ---- canonical Gram --------------------------------------------------------
 * G[a][c] = sum_i X[i,a] Y[i,c].  Rows are cut into chunks of R = canon_R(n)
 * consecutive rows; each chunk partial is a sequential fma over its rows in
 * order (from 0.0); chunk partials are combined by canon_final.             */
int64_t canon_R(int64_t n) {
  int64_t t = (n + 65535) / 65536;
  if (t < 1) t = 1;
  return 64 * t;
}

void canon_gram(int64_t n, int64_t na, int64_t nc, const double *X,
                int64_t rsx, int64_t csx, const double *Y, int64_t rsy,
                int64_t csy, double *G /* na x nc row-major */) {
  int64_t R = canon_R(n);
  int64_t nch = n <= 0 ? 0 : (n + R - 1) / R;
  double *P = (double *)malloc(sizeof(double) * (nch > 0 ? nch : 1));
  for (int64_t a = 0; a < na; ++a)
    for (int64_t c = 0; c < nc; ++c) {
      for (int64_t ch = 0; ch < nch; ++ch) {
        double acc = 0.0;
        int64_t i1 = (ch + 1) * R < n ? (ch + 1) * R : n;
        for (int64_t i = ch * R; i < i1; ++i)
          acc = fma(X[i * rsx + a * csx], Y[i * rsy + c * csy], acc);
        P[ch] = acc;
      }
      G[a * nc + c] = nch ? canon_final(nch, P, 1) : 0.0;
    }
  free(P);
}

/* out[i,c] = sum_j X[i,j] Z[j,c] (sequential in j from 0.0 with fma).
 * Z is m x nc row-major; out element (i,c) at out[i*rso + c*cso].          */
void canon_gemm(int64_t n, int64_t m, int64_t nc, const double *X, int64_t rsx,
                int64_t csx, const double *Z, double *out, int64_t rso,
                int64_t cso) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t c = 0; c < nc; ++c) {
      double acc = 0.0;
      for (int64_t j = 0; j < m; ++j)
        acc = fma(X[i * rsx + j * csx], Z[j * nc + c], acc);
      out[i * rso + c * cso] = acc;
    }
}

/* ---- canonical triangular solve ------------------------------------------
 * Off-diagonal CSR (rp, ci, v) of a lower (lower != 0: rows in increasing
 * order) or upper triangular factor, diag = NULL for a unit diagonal.
 * Row i: lane l (of 32) accumulates fma(v_e, x[c_e], acc) over the row's
 * off-diagonal entries e = l, l+32, ... in CSR (column) order; the 32-lane
 * tree gives S; x_i = b_i - S, then / diag_i.  (The B200 kernel: a warp per
 * row, csrc/precond.cu.)                                                    */
void canon_trsv(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                const double *diag, int lower, const double *b, double *x) {
  double a[32];
  for (int64_t t = 0; t < n; ++t) {
    const int64_t i = lower ? t : n - 1 - t;
    memset(a, 0, sizeof(a));
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const int l = (int)((e - rp[i]) & 31);
      a[l] = fma(v[e], x[ci[e]], a[l]);
    }
    tree32(a);
    double s = b[i] - a[0];
    if (diag) s = s / diag[i];
    x[i] = s;
  }
}
