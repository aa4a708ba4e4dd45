// Shared pieces of the BiCGSTAB drivers (graph kernels and persistent
// kernels): the solve descriptor, the per-phase scalar logic and the
// fused elementwise + canonical-partial phase bodies.
#pragma once

#include "ctx.cuh"

namespace krb {

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
  int l2keep;   // keep C / Chat resident in L2 (evict_last loads)
  int pf_rows;  // graph P / S / X phases: L2 prefetch distance in 1024-element rows
  cudaGraphConditionalHandle cond;
  const double *C, *Chat, *U;
  double *x, *r, *p, *q, *s, *t, *rt0, *b;
  double *p2, *q2;        // second p / q buffers (fused persistent kernel)
  double *zeta, *gamma, *xc;
  double *part, *part2;   // part2: second partial buffer (persistent kernel)
  uint64_t *prof;         // optional per-phase %globaltimer stamps (16/iter)
  int64_t prof_cap;
  uint64_t *ktime;        // optional live per-kernel time (krb_solve_config)
  // optional record_iterates snapshots (krb_solve_config.d_rec_*)
  double *rec_x, *rec_r, *rec_xc, *rec_s, *rec_t, *rec_omega;
  unsigned int *counters;
  unsigned int *flags;    // per-CTA phase epochs, 128 B apart (persist0.cu)
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

// Live per-kernel device time (graph / host-loop drivers; krb.h
// krb_solve_config.d_kernel_times): CTA 0 stamps the start, the last CTA to
// finish adds (end - start) to the slot's total.  Slots: 0 P, 1 q = A p,
// 2 Chat^T q, 3 Q, 4 S, 5 t = A s, 6 Chat^T t, 7 T, 8 X.
__host__ __device__ constexpr int ktime_slot_of(int PH) {
  return PH == PH_PUPDATE ? 0 : PH == PH_PROJ_Q ? 3 : PH == PH_SUPD ? 4
       : PH == PH_PROJ_T ? 7 : PH == PH_XR ? 8 : -1;
}

// The SpMV kernels (slots 1, 5: one CTA per 256 rows, 65536 CTAs at C5)
// mark their end per SM instead of electing a last CTA: each CTA's thread 0
// does a fire-and-forget atomicMax into its SM's slot (kKtSpmvBase + 160 s'
// + smid; one address per SM, so no single-address atomic queue -- that
// cost ~25 % of the launch), and the X phase's leader (after both SpMVs of
// the iteration) folds the maximum over the SMs into the slots' totals.
constexpr int kKtSpmvBase = 64;     // d_kernel_times[64 .. 64 + 2 x 160)
constexpr int kKtSmSlots = 160;

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// by warp 0 of CTA 0
__device__ __forceinline__ void ktime_fold_spmv(const IterArgs &a) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s2 = 0; s2 < 2; ++s2) {
    volatile uint64_t *sm = (volatile uint64_t *)a.ktime + kKtSpmvBase + kKtSmSlots * s2;
    uint64_t mx = 0;
    for (int q = lane; q < kKtSmSlots; q += 32) {
      const uint64_t v = sm[q];
      mx = v > mx ? v : mx;
      if (v) sm[q] = 0;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, mx, off);
      mx = o > mx ? o : mx;
    }
    if (lane == 0 && mx != 0) {
      volatile uint64_t *kt = (volatile uint64_t *)a.ktime + 4 * (s2 == 0 ? 1 : 5);
      kt[1] = kt[1] + (mx - kt[0]);
      kt[2] = kt[2] + 1;
    }
  }
}

// CTA 0 stamps the kernel's start (one store; the SpMV ends are folded by
// the X phase's leader, ktime_fold_spmv, so the hot kernels carry no extra
// code: the fold loop inlined into every kernel cost them registers)
__device__ __forceinline__ void ktime_start(const IterArgs &a, int slot) {
  if (a.ktime && slot >= 0 && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
    *(volatile uint64_t *)&a.ktime[4 * slot] = globaltimer();
}

__device__ __forceinline__ void ktime_end_spmv(const IterArgs &a, int slot) {
  if (!a.ktime) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int s2 = slot == 1 ? 0 : 1;
    atomicMax((unsigned long long *)&a.ktime[kKtSpmvBase + kKtSmSlots * s2 + smid()],
              (unsigned long long)globaltimer());
  }
}

// by thread 0 of the CTA known to finish last
__device__ __forceinline__ void ktime_add(const IterArgs &a, int slot) {
  if (!a.ktime || slot < 0) return;
  const uint64_t t1 = globaltimer();
  const uint64_t t0 = *(volatile uint64_t *)&a.ktime[4 * slot];
  a.ktime[4 * slot + 1] += t1 - t0;
  a.ktime[4 * slot + 2] += 1;
}

// every thread of every CTA: elects the last CTA with the slot's own
// counter (kernels without a last-CTA election of their own)
__device__ __forceinline__ void ktime_finish(const IterArgs &a, int slot) {
  if (!a.ktime || slot < 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long total = (unsigned long long)gridDim.x * gridDim.y;
    unsigned long long *cnt = (unsigned long long *)&a.ktime[4 * slot + 3];
    if (atomicAdd(cnt, 1ull) == total - 1) {
      __threadfence();
      ktime_add(a, slot);
      *cnt = 0;
    }
  }
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
// kRec: compile the record_iterates snapshot stores in (the host-loop
// record kernels only; the stores' pointer checks cost the hot X kernel
// registers)
template <int kE, int PH, int kU = 4, bool kRec = false, bool kPf = false>
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
  const uint64_t pol = l2_policy(a.l2keep);
  for (int64_t blk = first; blk < nb; blk += step) {
    const int64_t base = blk * ((int64_t)kLanes * kE) + threadIdx.x;
    double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll(kE < kU ? kE : kU)
    for (int e = 0; e < kE; ++e) {
      const int64_t i = base + (int64_t)kLanes * e;
      if (kPf && a.pf_rows > 0 && threadIdx.x < 8 && e + a.pf_rows < kE) {
        // bounded L2 prefetch: the 1024-element rows pf_rows ahead of this
        // CTA's current row, one 8 KB bulk prefetch per read stream (at most
        // 2 x 148 CTAs x streams x pf_rows x 8 KB in flight: fits in L2)
        const int64_t r0 = blk * ((int64_t)kLanes * kE) + (int64_t)kLanes * (e + a.pf_rows);
        const double *src = nullptr;
        const int lane = threadIdx.x;
        if (PH == PH_PUPDATE) src = lane == 0 ? r : lane == 1 ? p : lane == 2 ? q : nullptr;
        else if (PH == PH_SUPD) src = lane == 0 ? r : lane == 1 ? q : nullptr;
        else if (PH == PH_XR)
          src = lane == 0 ? x : lane == 1 ? p : lane == 2 ? s : lane == 3 ? t : lane == 4 ? rt0
                                                                                           : nullptr;
        if (src && r0 + kLanes <= n) prefetch_l2_bulk(src + r0, 8 * kLanes);
      }
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
            double c0 = ldg_pol(Cm + (int64_t)j * ld + i, pol);
            double c1 = ldg_pol(Cm + (int64_t)(j + 1) * ld + i, pol);
            double c2 = ldg_pol(Cm + (int64_t)(j + 2) * ld + i, pol);
            double c3 = ldg_pol(Cm + (int64_t)(j + 3) * ld + i, pol);
            cz = __fma_rn(c0, coef[j], cz);
            cz = __fma_rn(c1, coef[j + 1], cz);
            cz = __fma_rn(c2, coef[j + 2], cz);
            cz = __fma_rn(c3, coef[j + 3], cz);
          }
          for (; j < k; ++j) cz = __fma_rn(ldg_pol(Cm + (int64_t)j * ld + i, pol), coef[j], cz);
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
        double tv = t[i];
        double rv = __dsub_rn(sv, __dmul_rn(omega, tv));
        r[i] = rv;
        if (kRec && a.rec_x) {      // record_iterates: entry hist_len, step itn
          const int64_t j = a.S->hist_len, it = a.S->itn;
          a.rec_x[j * n + i] = x[i];
          a.rec_r[j * n + i] = rv;
          a.rec_s[it * n + i] = sv;
          a.rec_t[it * n + i] = tv;
        }
        acc[0] = __fma_rn(rv, rv, acc[0]);
        acc[1] = __fma_rn(rt0[i], rv, acc[1]);
      } else if (PH == PH_BNORM) {
        double bv = bvec[i];
        acc[0] = __fma_rn(bv, bv, acc[0]);
      } else if (PH == PH_INIT) {
        double rv = r[i], tv = rt0[i];
        if (kRec && a.rec_x) {      // record_iterates: entry 0
          a.rec_x[i] = x[i];
          a.rec_r[i] = rv;
        }
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
    const int64_t hj = a.S->hist_len;
    for (int j = threadIdx.x; j < a.k; j += blockDim.x) {
      const double v = __dadd_rn(__dadd_rn(a.xc[j], __dmul_rn(sc.alpha, a.zeta[j])),
                                 __dmul_rn(sc.omega, a.gamma[j]));
      a.xc[j] = v;
      if (a.rec_x) a.rec_xc[hj * a.k + j] = v;
    }
    if (a.rec_x && threadIdx.x == 0) a.rec_omega[a.S->itn] = sc.omega;
  }
  if (PH == PH_INIT && a.rec_x)
    for (int j = threadIdx.x; j < a.k; j += blockDim.x) a.rec_xc[j] = a.xc[j];
  __syncthreads();
  if (threadIdx.x == 0) finalize<PH>(a, a.S, dfin);
  __syncthreads();
}

// half-step exit (solvers.py:315-325): x += alpha p, xc += alpha zeta
// (record_iterates: entry hist_len - 1 gets x, r = s and xc)
__device__ __forceinline__ void half_exit_update(const IterArgs &a, double alpha,
                                                 int64_t first, int64_t step) {
  const int64_t hj = a.rec_x ? a.S->hist_len - 1 : 0;
  for (int64_t i = first * blockDim.x + threadIdx.x; i < a.n; i += step * blockDim.x) {
    const double xv = __dadd_rn(a.x[i], __dmul_rn(alpha, a.p[i]));   // solvers.py:316
    a.x[i] = xv;
    if (a.rec_x) {
      a.rec_x[hj * a.n + i] = xv;
      a.rec_r[hj * a.n + i] = a.s[i];                               // solvers.py:319
    }
  }
  if (first == 0)
    for (int j = threadIdx.x; j < a.k; j += blockDim.x) {   // solvers.py:318
      const double v = __dadd_rn(a.xc[j], __dmul_rn(alpha, a.zeta[j]));
      a.xc[j] = v;
      if (a.rec_x) a.rec_xc[hj * a.k + j] = v;
    }
}

// per-solve setup / tail shared by the single and batched drivers
// (bicgstab.cu)
int solve_setup(krb_context *ctx, const krb_matrix *A, const double *d_b,
                const double *d_x_init, const krb_space_view *R,
                const krb_solve_config *cfg, const IterArgs &h, const IterArgs *d,
                double *w, double *ybuf, cudaStream_t st);
int solve_tail(const krb_matrix *A, const krb_space_view *R, const IterArgs &h,
               const IterArgs *d, double *d_x_out, cudaStream_t st);

}  // namespace krb
