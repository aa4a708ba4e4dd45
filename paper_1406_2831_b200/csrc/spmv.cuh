// One-thread-per-row SpMV row kernel, scipy csr_matvec order (shared by the
// standalone SpMV and the SpMV nodes of the solver graphs).
#pragma once

#include "krb_internal.cuh"

namespace krb {

template <bool kRO>
__device__ __forceinline__ double ldx(const double *p) {
  if (kRO) return __ldg(p);
  return *p;
}

// ---- SpMV kernels: one thread per row, CSR order, mul then add ----------
// kXro: x is read-only for the whole kernel (ld.global.nc); false inside the
// persistent solver, where x was written by other CTAs earlier in the kernel.
template <bool kSell, bool kXro = true>
__device__ __forceinline__ double spmv_row(int64_t i, const krb_matrix &A,
                                          const double *__restrict__ x) {
  double sum = 0.0;
  if (kSell) {
    const int len = __ldg(A.rlen + i);
    const int64_t base = __ldg(A.sl_ptr + (i >> 5)) + (i & 31);
    const int32_t *__restrict__ cp = A.s_col + base;
    const double *__restrict__ vp = A.s_val + base;
    int j = 0;
    for (; j + 4 <= len; j += 4) {
      int c0 = __ldg(cp + 32 * j), c1 = __ldg(cp + 32 * (j + 1));
      int c2 = __ldg(cp + 32 * (j + 2)), c3 = __ldg(cp + 32 * (j + 3));
      double v0 = __ldg(vp + 32 * j), v1 = __ldg(vp + 32 * (j + 1));
      double v2 = __ldg(vp + 32 * (j + 2)), v3 = __ldg(vp + 32 * (j + 3));
      double x0 = ldx<kXro>(x + c0), x1 = ldx<kXro>(x + c1), x2 = ldx<kXro>(x + c2),
             x3 = ldx<kXro>(x + c3);
      sum = __dadd_rn(sum, __dmul_rn(v0, x0));
      sum = __dadd_rn(sum, __dmul_rn(v1, x1));
      sum = __dadd_rn(sum, __dmul_rn(v2, x2));
      sum = __dadd_rn(sum, __dmul_rn(v3, x3));
    }
    for (; j < len; ++j)
      sum = __dadd_rn(sum, __dmul_rn(__ldg(vp + 32 * j), ldx<kXro>(x + __ldg(cp + 32 * j))));
  } else {
    int64_t b = __ldg(A.rp + i), e = __ldg(A.rp + i + 1);
    int64_t jj = b;
    for (; jj + 4 <= e; jj += 4) {
      int c0 = __ldg(A.ci + jj), c1 = __ldg(A.ci + jj + 1);
      int c2 = __ldg(A.ci + jj + 2), c3 = __ldg(A.ci + jj + 3);
      double v0 = __ldg(A.val + jj), v1 = __ldg(A.val + jj + 1);
      double v2 = __ldg(A.val + jj + 2), v3 = __ldg(A.val + jj + 3);
      double x0 = ldx<kXro>(x + c0), x1 = ldx<kXro>(x + c1), x2 = ldx<kXro>(x + c2),
             x3 = ldx<kXro>(x + c3);
      sum = __dadd_rn(sum, __dmul_rn(v0, x0));
      sum = __dadd_rn(sum, __dmul_rn(v1, x1));
      sum = __dadd_rn(sum, __dmul_rn(v2, x2));
      sum = __dadd_rn(sum, __dmul_rn(v3, x3));
    }
    for (; jj < e; ++jj)
      sum = __dadd_rn(sum, __dmul_rn(__ldg(A.val + jj), ldx<kXro>(x + __ldg(A.ci + jj))));
  }
  return sum;
}


}  // namespace krb
