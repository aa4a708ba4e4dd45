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
// Same entries, same CSR order, same mul-then-add as spmv_row_f<true>; only
// the column of element j is encoded differently: a uniform slice (its 32
// rows share one offset sequence: interior stencil rows) keeps ONE row of
// int32 offsets col - row for all its lanes (16-byte broadcast loads, 4
// elements each); any other slice keeps one code byte per element,
// column-major like s_col, decoded through the matrix's offset dictionary
// (1 KB, L1-resident).  No shared-memory staging, no CTA barrier.
// Uniform slice: lane l loads entry l (l + 32, ...) of the shared offset row
// with one coalesced load per 32 entries and the entries reach every lane by
// warp shuffles -- no dependent memory round trip before each batch's
// gathers (all 32 lanes of a uniform slice exist and share the trip count).
// kV = 1: round-2 first version (the 4 offsets of each batch loaded by every
// lane as one int4 broadcast, tuning spmv_variant=1).
// pf > 0: lane 0 of each warp bulk-prefetches into L2 the value bytes pf
// beyond its own slice (the slices a later wave will stream).
template <int kV = 0, class XF, int kBU = 4>
__device__ __forceinline__ double spmv_row_dict(int64_t i, const krb_matrix &A, XF xf,
                                               int64_t pf = 0) {
  constexpr int kB = 4;
  const int64_t s = i >> 5;
  const int l = (int)(i & 31);
  const int len = __ldg(A.rlen + i);
  const int64_t vbase = __ldg(A.sl_ptr + s);
  const double *__restrict__ vp = A.s_val + vbase + l;
  if (pf > 0 && l == 0) {
    const int64_t at = vbase + pf / 8, nb = 256 * (int64_t)len;
    if (at + nb / 8 <= A.sell_elems && nb > 0) prefetch_l2_bulk(A.s_val + at, (uint32_t)nb);
  }
  const int64_t dp = __ldg(A.dptr + s);
  const bool uni = dp & 1;
  const uint8_t *__restrict__ cp = A.dcode + (dp >> 1) + (uni ? 0 : l);
  const int row = (int)i;
  double sum = 0.0;
  if (uni && kV == 0) {
    const int32_t *__restrict__ orow = reinterpret_cast<const int32_t *>(cp);
    for (int j0 = 0; j0 < len; j0 += 32) {
      const int mine = j0 + l < len ? __ldg(orow + j0 + l) : 0;
      const int m = min(32, len - j0);
      const double *__restrict__ vj = vp + 32 * j0;
      int j = 0;
      // full batches: no per-element predicates, so all 2 kB loads issue
      // before the first multiply
      for (; j + kBU <= m; j += kBU) {
        int c[kBU];
        double v[kBU], xv[kBU];
#pragma unroll
        for (int u = 0; u < kBU; ++u) c[u] = row + __shfl_sync(0xffffffffu, mine, j + u);
#pragma unroll
        for (int u = 0; u < kBU; ++u) v[u] = __ldg(vj + 32 * (j + u));
#pragma unroll
        for (int u = 0; u < kBU; ++u) xv[u] = xf(c[u]);
#pragma unroll
        for (int u = 0; u < kBU; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
      }
      for (; j < m; ++j) {
        const int c = row + __shfl_sync(0xffffffffu, mine, j);
        sum = __dadd_rn(sum, __dmul_rn(__ldg(vj + 32 * j), xf(c)));
      }
    }
    return sum;
  }
  for (int j = 0; j < len; j += kB) {
    int c[kB];
    double v[kB], xv[kB];
    if (uni) {
      const int4 o = __ldg(reinterpret_cast<const int4 *>(cp) + (j >> 2));
      c[0] = row + o.x; c[1] = row + o.y; c[2] = row + o.z; c[3] = row + o.w;
    } else {
#pragma unroll
      for (int u = 0; u < kB; ++u)
        c[u] = j + u < len ? row + __ldg(A.dict + __ldg(cp + 32 * (j + u))) : 0;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) v[u] = j + u < len ? __ldg(vp + 32 * (j + u)) : 0.0;
#pragma unroll
    for (int u = 0; u < kB; ++u) xv[u] = j + u < len ? xf(c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kB; ++u)
      if (j + u < len) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
  }
  return sum;
}

// ---- value-coded row (row templates; identity row order) -----------------
// Row i follows template tid[i]: entry j has column i + off_j and -- on a
// constant diagonal -- the table's value, else the row's own s_val entry
// (same position as in SELL-32).  Same entries, same CSR order, same
// mul-then-add as spmv_row_f<true>, so the same bits; the template entries
// (16 bytes each, a few KB per matrix) stay in L1 and the lanes of a warp
// that share a template read them as one broadcast.  No collectives: any
// mix of templates and row lengths inside a warp is handled by predication.
template <class XF, int kB = 4>
__device__ __forceinline__ double spmv_row_tmpl(int64_t i, const krb_matrix &A, XF xf) {
  const int t = __ldg(A.tid + i);
  const double *__restrict__ vp = A.s_val + __ldg(A.sl_ptr + (i >> 5)) + (i & 31);
  const int len = __ldg(A.tlen + t);
  const int4 *__restrict__ te = reinterpret_cast<const int4 *>(A.tent) + (int64_t)t * A.tstride;
  const int row = (int)i;
  double sum = 0.0;
  int j = 0;
  for (; j + kB <= len; j += kB) {
    int4 e[kB];
    double v[kB], xv[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) e[u] = __ldg(te + j + u);
#pragma unroll
    for (int u = 0; u < kB; ++u)
      v[u] = e[u].y ? __hiloint2double(e[u].w, e[u].z) : __ldg(vp + 32 * (j + u));
#pragma unroll
    for (int u = 0; u < kB; ++u) xv[u] = xf(row + e[u].x);
#pragma unroll
    for (int u = 0; u < kB; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
  }
  for (; j < len; ++j) {
    const int4 e = __ldg(te + j);
    const double v = e.y ? __hiloint2double(e.w, e.z) : __ldg(vp + 32 * j);
    sum = __dadd_rn(sum, __dmul_rn(v, xf(row + e.x)));
  }
  return sum;
}

// ---- value-coded row in diagonal form (A.dia.nd > 0: <= 32 diagonals) ----
// The row's entries are the set bits of its template mask, walked in
// ascending diagonal order (= CSR order: rows are sorted by column).  The
// loop over the diagonals is fully unrolled, so offset and constant value of
// diagonal c are fixed constant-bank operands of the matrix argument (no
// load/store-unit traffic, no table loads at all); a varying diagonal's
// value comes from the row's s_val entry at its CSR position (the number of
// lower set bits).  Batches of 4 diagonals with predicated gathers.  Same
// products and sums as spmv_row_f<true>.
// (An absent entry adds +-0.0 = 0.0 * table value to the running sum instead
// of being skipped: the sum starts at +0.0 and a round-to-nearest sum is -0.0
// only when both addends are, so it never is -0.0 and adding a zero leaves
// every bit unchanged.  Diagonals with a non-finite value are kept out of
// the table -- 0 * inf -- and take the varying path.)
static __device__ __noinline__ double spmv_dia_varying(double sum, unsigned m, int c,
                                                const double *__restrict__ vp, double xv) {
  if ((m >> c) & 1)
    sum = __dadd_rn(sum, __dmul_rn(__ldg(vp + 32 * __popc(m & ((1u << c) - 1u))), xv));
  return sum;
}

// x: the gathered vector (plain read-only loads).  cst and the x pointer are
// pinned in registers (the compiler otherwise re-reads them from the constant
// bank before every entry and the kernel ends up bound by the constant cache:
// 91 % busy, 453 us at C5; with them 340 us, with the batch-level constancy
// test and uniform-register values 265 us; an unpredicated path for batches
// whose four entries are all present: 275 us, not kept; unconditional gather
// addresses: 257 us; a warp-uniform copy of the loop without predicates for
// warps whose rows have every diagonal: 261 us, not kept; batches of 8
// diagonals (40 registers, 48 instead of 64 warps per SM): 337 us, not kept;
// prefetch.global.L1 of the next batch's gathers: 283 us, not kept).
__device__ __forceinline__ double spmv_row_dia(int64_t i, const krb_matrix &A,
                                               const double *__restrict__ x) {
  const unsigned m = (unsigned)__ldg(reinterpret_cast<const unsigned long long *>(A.tmask) +
                                     __ldg(A.tid + i));
  const double *__restrict__ vp = A.s_val + __ldg(A.sl_ptr + (i >> 5)) + (i & 31);
  const int nd = A.dia.nd;
  unsigned cst = (unsigned)A.dia.cst;
  const double *xr = x + i;
  asm volatile("" : "+r"(cst), "+l"(xr));
  double sum = 0.0;
#pragma unroll
  for (int c0 = 0; c0 < 32; c0 += 4) {
    if (c0 >= nd) break;   // (mask bits >= nd are clear)
    // the batch's offsets as one 16-byte constant read, its constancy bits as
    // one test: the common all-constant batch runs without per-entry tests
    const int4 o4 = *reinterpret_cast<const int4 *>(&A.dia.off[c0]);
    const int o[4] = {o4.x, o4.y, o4.z, o4.w};
    // the four gather addresses are formed unconditionally (offsets through
    // uniform registers; formed under the entry's predicate they are per-lane
    // LDC reads and the address-divergence unit becomes the limiter: 82 % busy)
    const double *px[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) px[u] = xr + o[u];
    asm volatile("" : "+l"(px[0]), "+l"(px[1]), "+l"(px[2]), "+l"(px[3]));
    double xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = ((m >> (c0 + u)) & 1) ? __ldg(px[u]) : 0.0;
    if (((cst >> c0) & 15u) == 15u) {   // warp-uniform
#pragma unroll
      for (int u = 0; u < 4; ++u) sum = __dadd_rn(sum, __dmul_rn(A.dia.val[c0 + u], xv[u]));
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u;
        if ((cst >> c) & 1)
          sum = __dadd_rn(sum, __dmul_rn(A.dia.val[c], xv[u]));
        else
          sum = spmv_dia_varying(sum, m, c, vp, xv[u]);
      }
    }
  }
  return sum;
}

}  // namespace krb
