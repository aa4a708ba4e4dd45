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
// xf(c) supplies x[c] (a plain load, or a value recomputed on the fly from
// other vectors by the fused persistent phases).  Entries go in batches of
// kB with predicated tails, so a row of up to kB entries costs two dependent
// memory round trips (indices, then gathers); the sum stays sequential in
// CSR order.
template <bool kSell, int kB = 4, bool kHint = false, class XF>
__device__ __forceinline__ double spmv_row_f(int64_t i, const krb_matrix &A, XF xf,
                                            uint64_t pol = 0) {
  double sum = 0.0;
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
    const int64_t b = __ldg(A.rp + i);
    len = (int)(__ldg(A.rp + i + 1) - b);
    cp = A.ci + b;
    vp = A.val + b;
    stride = 1;
  }
  for (int j = 0; j < len; j += kB) {
    int c[kB];
    double v[kB], xv[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const bool ok = j + u < len;
      if (kHint) {   // matrix entries with an L2 policy (evict_first: streamed)
        c[u] = ok ? ldg_pol_i32(cp + (int64_t)stride * (j + u), pol) : 0;
        v[u] = ok ? ldg_pol(vp + (int64_t)stride * (j + u), pol) : 0.0;
      } else {
        c[u] = ok ? __ldg(cp + (int64_t)stride * (j + u)) : 0;
        v[u] = ok ? __ldg(vp + (int64_t)stride * (j + u)) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) xv[u] = j + u < len ? xf(c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kB; ++u)
      if (j + u < len) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
  }
  return sum;
}

// ---- SpMV row: one thread per row, CSR order, mul then add --------------
// kXro: x is read-only for the whole kernel (ld.global.nc); false inside the
// persistent solver, where x was written by other CTAs earlier in the kernel.
template <bool kSell, bool kXro = true>
__device__ __forceinline__ double spmv_row(int64_t i, const krb_matrix &A,
                                          const double *__restrict__ x) {
  return spmv_row_f<kSell>(i, A, [x](int c) { return ldx<kXro>(x + c); });
}

// ---- offset-coded SELL-32 row (identity row order: i is the row) ---------
// Same entries, same CSR order, same mul-then-add as spmv_row_f<true>; the
// column of element j is i + sdict[code_j] with the 1-byte code read from
// the slice's code stream (a uniform slice's stream is shared by its 32
// lanes: one broadcast byte per element instead of 4 index bytes per lane).
// sdict: the matrix's offset dictionary staged in shared memory.
template <int kB = 4, class XF>
__device__ __forceinline__ double spmv_row_dict(int64_t i, const krb_matrix &A,
                                               const int32_t *sdict, XF xf) {
  const int64_t s = i >> 5;
  const int l = (int)(i & 31);
  const int len = __ldg(A.rlen + i);
  const double *__restrict__ vp = A.s_val + __ldg(A.sl_ptr + s) + l;
  const int64_t dp = __ldg(A.dptr + s);
  const bool uni = dp & 1;
  const uint8_t *__restrict__ cp = A.dcode + (dp >> 1) + (uni ? 0 : l);
  const int cs = uni ? 1 : 32;
  const int row = (int)i;
  double sum = 0.0;
  for (int j = 0; j < len; j += kB) {
    int c[kB];
    double v[kB], xv[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const bool ok = j + u < len;
      c[u] = ok ? row + sdict[__ldg(cp + cs * (j + u))] : 0;
      v[u] = ok ? __ldg(vp + 32 * (j + u)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) xv[u] = j + u < len ? xf(c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kB; ++u)
      if (j + u < len) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
  }
  return sum;
}

// stage the offset dictionary (256 entries) in shared memory; every thread
// of the CTA must call it (one barrier)
__device__ __forceinline__ void stage_dict(const krb_matrix &A, int32_t *sdict) {
  for (int t = threadIdx.x; t < 256; t += blockDim.x) sdict[t] = __ldg(A.dict + t);
  __syncthreads();
}

}  // namespace krb
