/*
 * krb.h -- C ABI of libkrb.so, the B200 (sm_100a) kernels behind the
 * recycling-BiCGSTAB hot path of arXiv 1406.2831 ("krecycle").
 *
 * The reference (/root/reference/pkg) is pure Python; it has no C ABI.  Its
 * native arithmetic lives in scipy/OpenBLAS calls made from solvers.py and
 * recycling.py.  Each entry point below replaces one such call site (cited),
 * or one whole loop of it.  The Python drop-in layer
 * (paper_1406_2831_b200/) binds these with ctypes exactly like the stub in
 * INTEGRATION.md.
 *
 * Conventions
 *   - every pointer named d_* is DEVICE memory (any allocator; torch in the
 *     Python layer); h_* is host memory.
 *   - dense n x k blocks are COLUMN-major with leading dimension ld >= n.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - all calls are asynchronous on `stream` unless stated otherwise and
 *     return 0 on success, a negative KRB_E* code on failure; the message is
 *     in krb_last_error() (thread-local).
 *   - floating point: fp64 only.  Every reduction is evaluated in the fixed
 *     "canonical" order documented in oracle/canon.c, so results are
 *     bit-reproducible run to run and equal to the CPU oracle.
 */
#ifndef KRB_H
#define KRB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KRB_OK 0
#define KRB_EINVAL -1
#define KRB_ECUDA -2
#define KRB_ENOMEM -3
#define KRB_ESTATE -4
#define KRB_EFACTOR -5   /* ILUTP: no usable pivot (reference FactorizationError) */

/* solver status codes (history.status strings of solvers.py:33-37) */
#define KRB_RUNNING 0
#define KRB_CONVERGED 1
#define KRB_MAX_ITN 2
#define KRB_BREAKDOWN_SERIOUS 3
#define KRB_BREAKDOWN_OMEGA 4
#define KRB_BREAKDOWN_SECOND_KIND 5

int krb_abi_version(void);
const char *krb_last_error(void);
/* number of kernel launches issued by this library since load (counter) */
int64_t krb_launch_count(void);

/* Driver / kernel-variant knobs (process-wide; every variant computes the
 * same bits).  Keys: "persist0", "p0_grid_half", "p0_onchip", "p0_prof_cta",
 * "cluster", "persist_v1", "gemm_mode", "l2keep", "phase_variant",
 * "tdot_variant", "spmv_variant", "spmm_variant", "phase_pf_rows",
 * "spmv_prefetch_mb" (bulk L2 prefetch
 * distance of the offset-coded SpMV, default 6), "value_coding" (value
 * tables for constant diagonals, default 1).  Unknown key -> KRB_EINVAL.
 * No reference counterpart (the reference has no device drivers). */
int krb_set_tuning(const char *key, int64_t value);
int krb_reset_tuning(void);

/* Device allocator for the library's own arrays (matrices, transposes and
 * their build temporaries).  Default: the stream-ordered CUDA pool.  A host
 * framework installs its caching allocator here so both share one pool
 * (the Python binding installs torch's).  Must be called before the first
 * allocation; alloc returns NULL on failure (-> KRB_ENOMEM).             */
typedef void *(*krb_alloc_fn)(size_t bytes, void *stream);
typedef void (*krb_free_fn)(void *ptr, void *stream);
int krb_set_allocator(krb_alloc_fn alloc, krb_free_fn free_fn);

/* ------------------------------------------------------------- ILUTP */
/* ilutp_factor (ilutp.py:131-281) on the host, bit-identical to the
 * reference: A*P ~= L*U, L unit lower (diagonal stored), U upper, perm[j] =
 * original column at position j.  fill_limit < 0: none.  KRB_EFACTOR with
 * the reference's FactorizationError message when a row has no pivot.    */
typedef struct krb_ilutp krb_ilutp;
int krb_ilutp_factor(int64_t n, const int64_t *h_row_ptr, const int32_t *h_col_idx,
                     const double *h_values, double drop_tol, double pivot_tol,
                     int64_t fill_limit, krb_ilutp **out);
int krb_ilutp_sizes(const krb_ilutp *F, int64_t *nnz_L, int64_t *nnz_U);
/* copy the factors into caller-owned host arrays (any may be NULL) */
int krb_ilutp_export(const krb_ilutp *F, int64_t *L_rp, int32_t *L_ci, double *L_val,
                     int64_t *U_rp, int32_t *U_ci, double *U_val, int64_t *perm);
int krb_ilutp_free(krb_ilutp *F);

/* stream-ordered device-to-device copy (ring views -> caller tensors) */
int krb_memcpy_d2d(void *d_dst, const void *d_src, int64_t bytes, void *stream);

/* ---------------------------------------------------------------- context */
/* Owns scratch buffers, the CUDA-graph cache and the solver state block. */
typedef struct krb_context krb_context;
int krb_context_create(krb_context **out);
int krb_context_destroy(krb_context *ctx);

/* ----------------------------------------------------------------- matrix */
/* Device sparse matrix.  Replaces SparseMatrix's scipy CSR
 * (sparse.py:27-69); the transpose used by rmatvec (sparse.py:123-130) is
 * built on the device, once, on first use.  The handle copies the CSR into
 * its own storage and builds the SELL-32 variant when it is selected
 * (format: 0 = auto, 1 = CSR, 2 = SELL-32). */
typedef struct krb_matrix krb_matrix;
int krb_matrix_create(krb_matrix **out, int64_t n, int64_t nnz,
                      const int64_t *d_row_ptr, const int32_t *d_col_idx,
                      const double *d_values, int format, void *stream);
/* Same, from int64 column indices (the reference's SparseMatrix dtype). */
int krb_matrix_create_i64(krb_matrix **out, int64_t n, int64_t nnz,
                          const int64_t *d_row_ptr, const int64_t *d_col_idx,
                          const double *d_values, int format, void *stream);
int krb_matrix_destroy(krb_matrix *A);
/* Stream-ordered destroy: storage returns to the device memory pool after
 * the work already queued on `stream`; no device-wide synchronisation.  No
 * other stream may still use the matrix. */
int krb_matrix_destroy_async(krb_matrix *A, void *stream);
/* n, nnz, chosen format (1 CSR, 2 SELL-32, 3 SELL-C-sigma, 4 SELL-32 with
 * offset-coded columns, 5 = 4 with value tables for the constant
 * diagonals), device bytes held (incl. transpose when built) */
int krb_matrix_info(const krb_matrix *A, int64_t *n, int64_t *nnz,
                    int *format, int64_t *bytes);
/* Bytes one y = A x streams in the chosen format (matrix arrays the kernel
 * reads + x once + y once), the SELL slice count, the uniform slices of the
 * offset-coded format (one shared offset row) and its dictionary size. */
int krb_matrix_stream_stats(const krb_matrix *A, int64_t *stream_bytes, int64_t *nslices,
                            int64_t *uniform_slices, int *ndict);
/* Value-coded format (5): a diagonal col - row whose entries are all
 * bit-identical (constant-coefficient stencils: every diagonal of K in
 * s E - K but the main one) is served from a table instead of the value
 * stream -- same value bits, same row order, so the same products as
 * sparse.py:117-121.  Rows with the same offset sequence share a template
 * (offsets + table values, a few KB per matrix); a row then reads its
 * template id and only the values of its varying entries.  const_entries:
 * entries served from the tables (0: not value-coded), templates: distinct
 * row templates, const_diagonals: constant diagonals among the ndict offsets,
 * diagonal_form: the SpMV walks the <= 64 diagonals with the table in its
 * kernel argument (rows sorted by column, at least half of the n x ndict
 * positions filled) instead of the per-row templates.
 * Chosen automatically when at least half of the entries qualify. */
int krb_matrix_value_stats(const krb_matrix *A, int64_t *const_entries, int *templates,
                           int *const_diagonals, int *diagonal_form);

/* Identity and reference count of the shared sparsity pattern behind A
 * (matrices with equal row_ptr / col_idx share the SELL layout, the offset
 * codes and the transpose permutation while any of them is alive);
 * transpose_known: the pattern's transpose permutation is built. */
int krb_matrix_pattern_info(const krb_matrix *A, uint64_t *pattern_id, int *refs,
                            int *transpose_known);

/* y = A x  (SparseMatrix.matvec, sparse.py:117-121; scipy csr_matvec order:
 * per-row sequential sum from 0.0, separate multiply and add) */
int krb_spmv(const krb_matrix *A, const double *d_x, double *d_y,
             void *stream);
/* y = A^T x (SparseMatrix.rmatvec, sparse.py:123-130) */
int krb_spmv_t(krb_matrix *A, const double *d_x, double *d_y, void *stream);
/* Y[:,c] = A X[:,c] (or A^T X[:,c]) for c < ncols: _apply_columns
 * (recycling.py:28-32).  Bit-identical to ncols separate SpMVs. */
int krb_spmm(krb_matrix *A, int transpose, int64_t ncols, const double *d_X,
             int64_t ldx, double *d_Y, int64_t ldy, void *stream);

/* ------------------------------------------- split ILUTP operator */
/* Level schedule of a triangular CSR (host): lev_out[i] = 1 + max level of
 * the rows its off-diagonal entries reference (0 without); lower: entries
 * left of the diagonal, else right.  KRB_EINVAL on an entry on the wrong
 * side. */
int krb_tri_levels(int64_t n, const int64_t *rp, const int32_t *ci, int lower,
                   int32_t *lev_out, int32_t *nlev_out);

/* One triangular factor for the device solve (host arrays, uploaded by
 * krb_precond_create): off-diagonal CSR, diagonal (NULL = unit), and the
 * level schedule as per-warp task lists -- task t = row t_row[t] of level
 * t_lev[t], its t_len[t] off-diagonal entries at t_start[t]; warp w owns
 * tasks warp_ptr[w] .. warp_ptr[w+1]-1 in level order (16 warps: 17
 * entries; row r of a level goes to warp r mod 16).                        */
typedef struct krb_tri_host {
  int64_t n, nnz_off, ntasks;
  int32_t nlev;
  const int64_t *rp;
  const int32_t *ci;
  const double *val;
  const double *diag;
  const int32_t *warp_ptr, *t_row, *t_lev, *t_len;
  const int64_t *t_start;
} krb_tri_host;

/* The ILUTP factors on the device (L unit lower, Lt its transpose, U upper
 * with diagonal, Ut its transpose, h_perm the column permutation). */
typedef struct krb_precond krb_precond;
int krb_precond_create(const krb_tri_host *L, const krb_tri_host *Lt, const krb_tri_host *U,
                       const krb_tri_host *Ut, const int64_t *h_perm, krb_precond **out,
                       void *stream);
int krb_precond_destroy(krb_precond *P);
/* SplitPreconditionedOperator (ilutp.py:106-128) on the device: a view of
 * A whose products are L^{-1} A P U^{-1} (krb_spmv / krb_spmm) and
 * U^{-H} P^T A^H L^{-H} (krb_spmv_t / transposed krb_spmm), usable by every
 * solver entry point.  A and P must outlive the view; destroy it with
 * krb_matrix_destroy(_async).                                             */
int krb_operator_create(krb_matrix *A, const krb_precond *P, krb_matrix **op_out);
/* apply_left / apply_left_h / U^{-1} / U^{-H} (ilutp.py:76-97):
 * which = 0 L^{-1}, 1 L^{-H}, 2 U^{-1}, 3 U^{-H}                         */
int krb_precond_apply(const krb_precond *P, int which, const double *d_in, double *d_out,
                      void *stream);


/* ------------------------------------------------- canonical primitives */
/* *d_out = (x, y)        (np.vdot, solvers.py:308-352) */
int krb_dot(krb_context *ctx, int64_t n, const double *d_x, const double *d_y,
            double *d_out, void *stream);
/* d_out[j] = (M[:,j], v), j < k      (R.Chat.conj().T @ v, solvers.py:306) */
int krb_tdot(krb_context *ctx, int64_t n, int64_t k, const double *d_M,
             int64_t ldm, const double *d_v, double *d_out, void *stream);
/* d_out[i] = beta_i + sign * sum_j M[i,j] y[j]   with d_y on the device;
 * sign = -1: v - C y (solvers.py:307), +1: x + U y (recycling.py:204);
 * d_base may equal d_out; d_base == NULL means plain M y. */
int krb_gemv(int64_t n, int64_t k, const double *d_M, int64_t ldm,
             const double *d_y, const double *d_base, int sign, double *d_out,
             void *stream);
/* G[a*nc + c] = (X[:,a], Y[:,c])  (Wt^H AW, recycling.py:342-343) */
int krb_gram(krb_context *ctx, int64_t n, int64_t na, int64_t nc,
             const double *d_X, int64_t ldx, const double *d_Y, int64_t ldy,
             double *d_G, void *stream);
/* out[:,c] = X Z[:,c], Z an m x nc row-major device matrix
 * (W @ Zr, recycling.py:365-368) */
int krb_gemm(int64_t n, int64_t m, int64_t nc, const double *d_X, int64_t ldx,
             const double *d_Z, double *d_out, int64_t ldo, void *stream);
/* d_out[j] = ||X[:,j]||_2   (np.linalg.norm(X, axis=0), recycling.py:155) */
int krb_colnorms(krb_context *ctx, int64_t n, int64_t k, const double *d_X,
                 int64_t ldx, double *d_out, void *stream);
/* d_out[j] = (X[:,j], X[:,j]) without the square root (squared norms used
 * by the near-null eigen-residual test, recycling.py:353-354) */
int krb_colsq(krb_context *ctx, int64_t n, int64_t k, const double *d_X,
              int64_t ldx, double *d_out, void *stream);
/* Ritz eigen-residual in real arithmetic (recycling.py:351-352):
 * Are -= Yre*thr - Yim*thi ; Aim -= Yre*thi + Yim*thr   (per column c) */
int krb_ritz_combine(int64_t n, int64_t m, const double *d_Yre,
                     const double *d_Yim, double *d_Are, double *d_Aim,
                     int64_t ld, const double *d_thr, const double *d_thi,
                     void *stream);
/* X[:, j] *= 1/s[j] done as a division X[i,j] / s[j] (recycling.py:156,337) */
int krb_colscale_div(int64_t n, int64_t k, double *d_X, int64_t ldx,
                     const double *d_s, void *stream);
/* Y[:, j] = X[:, j] / s[j], out of place: the column scaling of
 * recycling.py:156,337 fused with the assembly of W = [U_prev, V] (the
 * hstacks of recycling.py:326-329) or with the Chat / Ccheck copies
 * (recycling.py:168-169) -- one read and one write per element */
int krb_colscale_div_to(int64_t n, int64_t k, const double *d_X, int64_t ldx,
                        const double *d_s, double *d_Y, int64_t ldy, void *stream);
/* numpy default_rng(seed).uniform(lo, hi, n), bit-identical: PCG64
 * (XSL-RR) from the 128-bit (state, inc) that numpy seeds
 * (solvers.py:111-113, 268-269). */
int krb_uniform_pcg64(int64_t n, uint64_t state_hi, uint64_t state_lo,
                      uint64_t inc_hi, uint64_t inc_lo, double lo, double hi,
                      double *d_out, void *stream);

/* ------------------------------------------------------------ recycle space */
/* View of a biorthonormalized recycle space (RecycleSpace,
 * recycling.py:35-77); all blocks n x k column-major with leading dim ld. */
typedef struct krb_space_view {
  int64_t n, k, ld;
  const double *U, *Ut, *C, *Ct, *Chat, *Ccheck;
} krb_space_view;

/* --------------------------------------------------------------- solvers */
typedef struct krb_solve_config {
  double tol;            /* relative tolerance on ||r|| / ||b||           */
  double breakdown_tol;  /* SolverConfig.breakdown_tol                    */
  int64_t max_itn;
  /* shadow residual: d_shadow (device, n) if non-NULL, else drawn on the
   * device from these PCG64 words (numpy default_rng(seed) state)          */
  const double *d_shadow;
  uint64_t pcg_state_hi, pcg_state_lo, pcg_inc_hi, pcg_inc_lo;
  int use_graph;         /* 0 host loop, 1 CUDA graph with a device WHILE
                            node, 2 persistent cooperative kernel           */
  /* optional (persistent driver): %globaltimer stamp after each of the 10
   * phase boundaries of iteration i at d_phase_stamps[16 i + slot]        */
  uint64_t *d_phase_stamps;
  int64_t phase_stamps_cap;  /* iterations covered                        */
  /* optional (graph / host-loop drivers): live per-kernel device time.  For
   * the 9 kernels of one iteration (slot 0 P, 1 q=Ap, 2 Chat^T q, 3 Q,
   * 4 S, 5 t=As, 6 Chat^T t, 7 T, 8 X) d_kernel_times[4 slot + 1] gains
   * (last CTA's end - CTA 0's start) in ns and [4 slot + 2] one per launch
   * that did work.  384 uint64 zeroed by the caller (36 totals; from 64 on,
   * per-SM end stamps of the SpMV kernels); accumulates across solves.  */
  uint64_t *d_kernel_times;
  /* optional record_iterates (solvers.py:40-56, recording at :168-172,
   * :209-218, :281-286, :340-346; host-loop driver only): per history entry
   * j (0 = start) d_rec_x / d_rec_r[j n ..] = x, r and d_rec_xc[j k ..] = xc
   * (the iterate is x - U xc); per full iteration i (0-based)
   * d_rec_s / d_rec_t[i n ..] = s, t and d_rec_omega[i] = omega.  NULL
   * d_rec_x = off; capacity max_itn + 1 entries.                          */
  double *d_rec_x, *d_rec_r, *d_rec_xc, *d_rec_s, *d_rec_t, *d_rec_omega;
} krb_solve_config;

typedef struct krb_solve_result {
  int32_t status;        /* KRB_CONVERGED ...                              */
  int64_t hist_len;      /* entries in resid/matvecs/stamps                */
  int64_t matvecs;       /* total counted products                         */
  double rhs_norm;
  double final_true_resid;
  uint64_t t_start_ns;   /* device %globaltimer at setup                   */
  int64_t iterations_run;   /* loop-body executions (incl. no-op tail)     */
  int64_t kernel_launches;  /* libkrb kernels executed by this solve       */
  int32_t driver;        /* loop driver that ran: KRB_DRIVER_*              */
} krb_solve_result;

/* krb_solve_result.driver */
#define KRB_DRIVER_HOST_LOOP 0
#define KRB_DRIVER_GRAPH 1
#define KRB_DRIVER_PERSISTENT 2     /* grid-wide persistent, nine barriers   */
#define KRB_DRIVER_FUSED 3          /* fused persistent (k_persist2)        */
#define KRB_DRIVER_CLUSTER 4        /* single thread-block cluster          */
#define KRB_DRIVER_BATCH_GRAPH 5    /* multi-rhs graph                      */

/* rbicgstab_solve (solvers.py:245-361), bicgstab_solve when R == NULL or
 * R->k == 0 (solvers.py:156-242, identical arithmetic).  Synchronous: returns
 * after the solve; d_x_out receives x - U xc; history arrays (device, length
 * >= max_itn + 2) receive ||r_i||, cumulative matvecs and device ns stamps. */
int krb_rbicgstab(krb_context *ctx, const krb_matrix *A, const double *d_b,
                  const double *d_x_init, const krb_space_view *R,
                  const krb_solve_config *cfg, double *d_x_out,
                  double *d_hist_resid, int64_t *d_hist_matvecs,
                  uint64_t *d_hist_stamp, krb_solve_result *h_result,
                  void *stream);

/* ---------------------------------------------------- generation solve */
/* rbicg_solve (solvers.py:460-638): two-sided deflated BiCG with capture of
 * normalized Lanczos-direction pairs into a device ring of s+2 columns.  The
 * host drives it: create -> start (projected initial residuals, dual-start
 * test scalars; repeated for the reference's re-draws) -> set_counts ->
 * begin -> run (returns at every completed cycle of s iterations, so the
 * recycle-space update can run, or when the solve stops) -> rotate after an
 * emitted cycle -> finish. */
/* Multi-right-hand-side RBiCGSTAB: nrhs <= 4
 * independent solves with the same matrix and recycle space (k <= 128) in
 * lockstep -- each iteration reads A, C and Chat once for all of them.  Every
 * per-rhs argument is a host array of nrhs device pointers (d_x_init may be
 * NULL, or hold NULL entries); cfgs and h_results are host arrays of nrhs.
 * Results are bit-identical to nrhs separate krb_rbicgstab calls.
 * use_graph (cfgs[0]): 0 host loop, otherwise CUDA graph. */
int krb_rbicgstab_batch(krb_context *ctx, const krb_matrix *A, int64_t nrhs,
                        const double *const *d_b, const double *const *d_x_init,
                        const krb_space_view *R, const krb_solve_config *cfgs,
                        double *const *d_x_out, double *const *d_hist_resid,
                        int64_t *const *d_hist_matvecs, uint64_t *const *d_hist_stamp,
                        krb_solve_result *h_results, void *stream);

typedef struct krb_rbicg krb_rbicg;
int krb_rbicg_create(krb_rbicg **out, krb_context *ctx, krb_matrix *A,
                     const krb_space_view *R, int64_t s, int64_t max_itn,
                     void *stream);
int krb_rbicg_destroy(krb_rbicg *H);
int krb_rbicg_start(krb_rbicg *H, const double *d_b, const double *d_bt,
                    const double *d_x0, const double *d_xt0, double tol,
                    double breakdown_tol, int use_graph, double *h_dual,
                    void *stream);
int krb_rbicg_set_counts(krb_rbicg *H, int64_t n_matvec, int64_t n_rmatvec,
                         void *stream);
int krb_rbicg_begin(krb_rbicg *H, int32_t *h_status, void *stream);
/* h_state[7] = status, emit, ncols, itn, nalpha, capture, npush */
int krb_rbicg_run(krb_rbicg *H, int64_t *h_state, void *stream);
/* krb_rbicg_run split in two (the loop of solvers.py:593-634 up to the next
 * `itn % s == 0` emit): launch without waiting, so the harvest of the
 * previous cycle (the cycle_callback's device work and host eigenproblem)
 * overlaps the next cycle's iterations; then wait and read the state. */
int krb_rbicg_launch(krb_rbicg *H, int32_t *launched, void *stream);
int krb_rbicg_wait(krb_rbicg *H, int64_t *h_state, void *stream);
int krb_rbicg_views(krb_rbicg *H, double **V, double **Vt, double **rhos,
                    double **alphas, double **betas);
int krb_rbicg_rotate(krb_rbicg *H, int64_t keep, void *stream);
int krb_rbicg_finish(krb_rbicg *H, double *d_x_out, double *d_xt_out,
                     double *d_hist_r, double *d_hist_rt, int64_t *d_hist_m,
                     uint64_t *d_hist_t, krb_solve_result *res,
                     int64_t *h_counts, double *h_btnorm, void *stream);

/* Per-iteration device scalars of the last solve (debug/tests): alpha,
 * omega, rho, beta written to h_out[0..3]. */
int krb_last_scalars(krb_context *ctx, double *h_out);

#ifdef __cplusplus
}
#endif
#endif /* KRB_H */
