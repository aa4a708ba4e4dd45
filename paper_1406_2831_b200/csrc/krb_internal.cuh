// Internal helpers shared by the libkrb translation units (sm_100a).
//
// Floating-point policy: the library is compiled with -fmad=false, so no
// multiply/add pair is ever contracted by the compiler.  Fused multiply-adds
// appear only where the canonical order (oracle/canon.c) asks for them, via
// explicit __fma_rn.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/krb.h"

// Device sparse matrix (CSR + optional SELL-32 + lazily built transpose).
struct krb_precond;
struct krb_pattern;   // shared sparsity structure (matrix.cu)
struct __align__(16) krb_tentry {
  int32_t off;    // col - row
  int32_t cst;    // 1: the value below; 0: the row's own s_val entry
  double val;
};
// Diagonal table of a value-coded matrix with at most 32 distinct diagonals,
// carried BY VALUE inside krb_matrix: a kernel that takes the matrix as a
// parameter reads it from the constant bank with warp-uniform indices (no
// load/store-unit traffic, no per-lane copies of the same 16 bytes).
struct __align__(16) krb_diatable {
  int32_t nd = 0;            // 0: not available
  int32_t pad = 0;
  uint64_t cst = 0;          // bit c: diagonal c is constant (value val[c])
  int32_t off[32] = {};      // col - row of diagonal c (ascending)
  double val[32] = {};
};
struct krb_matrix {
  int64_t n = 0, nnz = 0;
  int format = 0;  // 1 CSR, 2 SELL
  int req_format = 0;  // as requested at creation (the transpose follows it)
  int64_t *rp = nullptr;
  int32_t *ci = nullptr;
  double *val = nullptr;
  // SELL-32
  int64_t nslices = 0, sell_elems = 0;
  int64_t *sl_ptr = nullptr;
  int32_t *rlen = nullptr;
  int32_t *s_col = nullptr;
  double *s_val = nullptr;
  int32_t *perm = nullptr;  // SELL-C-sigma: slice position -> row (NULL: identity)
  // offset-coded SELL-32 (built beside s_col when the matrix has <= 255
  // distinct diagonals col - row, i.e. stencils / banded matrices): element
  // j of row i has col = i + dict[code]; a slice whose 32 rows share one
  // code sequence ("uniform": interior stencil rows) stores it once
  // (dptr = byte offset << 1 | 1, codes at dcode[off + j]), any other slice
  // stores one byte per element, column-major like s_col (dcode[off + 32 j + l]).
  uint8_t *dcode = nullptr;
  int64_t *dptr = nullptr;
  int32_t *dict = nullptr;  // 256 entries (sorted distinct offsets, zero-padded)
  int ndict = 0;
  int64_t dcode_bytes = 0, uniform_slices = 0;
  int32_t *rep = nullptr;   // 256: one CSR entry index per offset code (pattern)
  // row templates (pattern level, built with the offset codes when no row is
  // longer than 64 and the rows use at most 1024 distinct offset sequences):
  // row i has the offset sequence of template tid[i]; template t has tlen[t]
  // entries with codes tcode[64 t + j]
  int32_t *tid = nullptr;
  int32_t *tlen = nullptr;
  uint8_t *tcode = nullptr;
  int ntmpl = 0, tstride = 0;   // tstride: longest template, rounded up to 4
  int64_t *code_count = nullptr;   // HOST array: [0, 256) entries per offset code,
                                   // [256, 512) the offsets themselves (pattern)
  // value-coded format (matrix level, built beside s_val when most entries
  // lie on diagonals col - row whose values are all bit-identical:
  // constant-coefficient stencils, where only the main diagonal of s E - K
  // varies).  Entries of such a diagonal come from a table instead of the
  // s_val stream (same value bits, same order, same arithmetic -> same
  // results): vtab[d] = the value of offset code d, then 256 flag bytes
  // (1 = constant); tent[tstride t + j] = {offset, constant?, value} of
  // entry j of template t -- a few KB, L1-resident, so a row costs its tid,
  // its varying entries and its x gathers.
  double *vtab = nullptr;
  krb_tentry *tent = nullptr;
  int64_t vconst_entries = 0;   // entries served from the tables
  // diagonal form (<= 32 diagonals, rows sorted by column, at least half of
  // the n x ndict positions filled): row i's entries are the set bits of
  // tmask[tid[i]] (bit c = diagonal c present), walked in ascending c = CSR
  // order; constants and offsets from `dia`
  uint64_t *tmask = nullptr;   // pattern
  krb_diatable dia;            // matrix
  int64_t uid = 0;             // creation serial (the graph cache keys the by-value table on it)
  krb_matrix *T = nullptr;  // lazily built transpose
  // the structure arrays above (rp, ci, sl_ptr, rlen, s_col, perm, dcode,
  // dptr, dict) belong to this reference-counted pattern, shared by every
  // live matrix with the same row_ptr / col_idx (a sequence A_j = s_j E - K);
  // val and s_val are the matrix's own
  krb_pattern *pat = nullptr;
  int64_t bytes = 0;
  // preconditioned-operator view (precond.cu): shares `base`'s arrays; every
  // application runs the split-ILUTP composite (pre_adj: its adjoint)
  krb_matrix *base = nullptr;
  krb_precond *pre = nullptr;
  bool borrowed = false;
  bool pre_adj = false;
};


namespace krb {

// ---------------------------------------------------------- allocation
// Device memory of matrices / transposes / their build temporaries: the
// caller's allocator when one is installed (krb_set_allocator: the Python
// binding installs torch's caching allocator, so the library and torch
// share one pool), else the stream-ordered CUDA pool.
cudaError_t dev_alloc(void **p, size_t bytes, cudaStream_t st);
void dev_free(void *p, cudaStream_t st);

// Every device pointer a kernel launched on this matrix may receive as a
// parameter (a graph bakes kernel parameters: a cached graph is reused only
// for a matrix with the same signature -- freed and re-allocated arrays can
// come back at the address of another matrix's CSR values).
struct MatrixSig {
  const void *p[28];
  int64_t n = -1, serial = 0;
  int64_t uid = 0;   // of a matrix whose diagonal table travels by value in kernel parameters
  int format = -1;
};
MatrixSig matrix_sig(const krb_matrix *A);
bool same_sig(const MatrixSig &a, const MatrixSig &b);

// preconditioned operator (precond.cu)
int precond_apply_op(const krb_matrix *A, const double *x, double *y, const int *status,
                     cudaStream_t st);
void precond_free(krb_precond *P);
int64_t precond_serial(const krb_precond *P);

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
int64_t &launch_counter();

#define KRB_CHECK_CUDA(call)                                                \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess) {                                                \
      krb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                     cudaGetErrorString(e_));                               \
      return KRB_ECUDA;                                                     \
    }                                                                       \
  } while (0)

#define KRB_CHECK_LAUNCH()                                                  \
  do {                                                                      \
    krb::launch_counter()++;                                                \
    cudaError_t e_ = cudaGetLastError();                                    \
    if (e_ != cudaSuccess) {                                                \
      krb::set_error("%s:%d launch: %s", __FILE__, __LINE__,                \
                     cudaGetErrorString(e_));                               \
      return KRB_ECUDA;                                                     \
    }                                                                       \
  } while (0)

#define KRB_REQUIRE(cond, msg)                                              \
  do {                                                                      \
    if (!(cond)) {                                                          \
      krb::set_error("%s", msg);                                            \
      return KRB_EINVAL;                                                    \
    }                                                                       \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------- canonical order
constexpr int kLanes = 1024;           // lanes (= threads) per canonical block
constexpr int kTargetBlocks = 296;     // 148 SMs x 2 resident 1024-thread CTAs
constexpr int kNumSMs = 148;

inline int64_t canon_E(int64_t n) {
  int64_t t = (n + (int64_t)kLanes * kTargetBlocks - 1) /
              ((int64_t)kLanes * kTargetBlocks);
  int64_t E = 1;
  while (E < t && E < 16) E *= 2;
  return E;
}
inline int64_t canon_nblocks(int64_t n) {
  int64_t B = kLanes * canon_E(n);
  return n <= 0 ? 0 : (n + B - 1) / B;
}
inline int64_t canon_R(int64_t n) {
  int64_t t = (n + 65535) / 65536;
  if (t < 1) t = 1;
  return 64 * t;
}

// lane 0 receives the canonical 32-lane tree (offsets 16,8,4,2,1)
__device__ __forceinline__ double warp_tree(double a) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
    a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, off));
  return a;
}

// The canonical 32-lane tree for NCP (power of two <= 8) independent columns
// at once, "transposed": at offsets 16, 8, 4 the two partner lanes split the
// columns between them (each computes exactly the canonical pair sums, lower
// lane's value first, for half of the columns), so only NCP-1 + (5 - log2 NCP)
// shuffles are needed instead of 5 NCP.  On return the lanes whose low
// (5 - log2 NCP) bits are zero hold column `col` (bit-identical to warp_tree
// applied per column).
template <int NCP>
__device__ __forceinline__ double warp_tree_multi(double (&a)[NCP], int &col) {
  constexpr int H = NCP == 1 ? 0 : NCP == 2 ? 1 : NCP == 4 ? 2 : 3;
  const int lane = threadIdx.x & 31;
  int c = 0;
#pragma unroll
  for (int lvl = 0; lvl < H; ++lvl) {
    const int off = 16 >> lvl;
    const int half = NCP >> (lvl + 1);
    const bool hi = (lane & off) != 0;
#pragma unroll
    for (int u = 0; u < half; ++u) {
      double send = hi ? a[u] : a[half + u];
      double recv = __shfl_xor_sync(0xffffffffu, send, off);
      a[u] = hi ? __dadd_rn(recv, a[half + u]) : __dadd_rn(a[u], recv);
    }
    if (hi) c += half;
  }
  double v = a[0];
#pragma unroll
  for (int off = 16 >> H; off >= 1; off >>= 1)
    v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
  col = c;
  return v;
}

// Block stage for ND <= 4 dots of a 1024-lane canonical block: lane
// accumulators acc[d] -> per-warp transposed trees -> red[d][warp] ->
// warp d: canonical 32-lane tree over the 32 warp results.  The block partial
// of dot d lands on lane 0 of warp d (returned there; `red` needs 4 x 32).
// Contains __syncthreads (call uniformly).
template <int ND>
__device__ __forceinline__ double block_tree_multi(const double *acc,
                                                   double (*red)[32]) {
  constexpr int NCP = ND == 1 ? 1 : ND == 2 ? 2 : 4;
  constexpr int H = NCP == 1 ? 0 : NCP == 2 ? 1 : 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a[NCP];
#pragma unroll
  for (int d = 0; d < NCP; ++d) a[d] = d < ND ? acc[d] : 0.0;
  int col;
  double v = warp_tree_multi<NCP>(a, col);
  if ((lane & ((32 >> H) - 1)) == 0 && col < ND) red[col][warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp < ND) r = warp_tree(red[warp][lane]);
  __syncthreads();
  return r;
}

// Block stage of one canonical dot (1024 threads); block partial on thread 0.
__device__ __forceinline__ double block_tree(double acc, double (*red)[32]) {
  return block_tree_multi<1>(&acc, red);
}

// Final stage over nb block partials (one warp): lane L sums b = L, L+32, ...
// in order, then the 32-lane tree.  Result on lane 0.
__device__ __forceinline__ double warp_final(const double *P, int64_t nb) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  int64_t b = lane;
  for (; b + 7 * 32 < nb; b += 8 * 32) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = P[b + 32 * u];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
  }
  for (; b < nb; b += 32) acc = __dadd_rn(acc, P[b]);
  return warp_tree(acc);
}

// Same, reading through volatile loads (partials written by other CTAs of
// the same kernel, consumed by the last CTA after a fence).
__device__ __forceinline__ double warp_final_volatile(const double *P,
                                                      int64_t nb) {
  // L2-coherent loads (ld.global.cg), issued 8 at a time so the partials of
  // one lane stream in parallel; the adds stay in the canonical order.
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  int64_t b = lane;
  for (; b + 7 * 32 < nb; b += 8 * 32) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(P + b + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
  }
  for (; b < nb; b += 32) acc = __dadd_rn(acc, __ldcg(P + b));
  return warp_tree(acc);
}

// "last CTA" election: every CTA calls after writing its partials; returns
// true on exactly one CTA, which then sees all partials.
__device__ __forceinline__ bool elect_last_cta(unsigned int *counter,
                                               int *sflag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    *sflag = (prev == gridDim.x - 1);
  }
  __syncthreads();
  bool last = *sflag != 0;
  if (last) __threadfence();
  return last;
}

// L2 eviction-priority policy (createpolicy) for loads of blocks that should
// stay resident across iterations (the recycle blocks of small systems).
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t p;
  if (keep)
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// read-only global load carrying an L2 cache policy
__device__ __forceinline__ double ldg_pol(const double *ptr, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
  return v;
}

// Ampere-style per-thread async copies (LDGSTS): each thread stages the
// elements it will consume itself, so no CTA barrier is needed between the
// copy and its use -- the copies just add memory-level parallelism without
// registers.  valid == false zero-fills (src-size 0).
__device__ __forceinline__ void cp_async8(double *smem, const double *g, bool valid,
                                          uint64_t pol) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2, %3;\n" ::"r"(s),
               "l"(g), "r"(valid ? 8 : 0), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ int ldg_pol_i32(const int32_t *ptr, uint64_t pol) {
  int v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// bulk L2 prefetch (TMA unit; no registers, no completion tracking):
// 16-byte aligned address, size a multiple of 16
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#define KRB_TRY(x)          \
  do {                      \
    int rc_ = (x);          \
    if (rc_) return rc_;    \
  } while (0)

#define KRB_DISPATCH_E(E, ...)                 \
  switch (E) {                                 \
    case 1: { constexpr int kE = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int kE = 2; __VA_ARGS__; } break;   \
    case 4: { constexpr int kE = 4; __VA_ARGS__; } break;   \
    case 8: { constexpr int kE = 8; __VA_ARGS__; } break;   \
    default: { constexpr int kE = 16; __VA_ARGS__; } break; \
  }

inline int grid_for(int64_t nb, int per_sm = 2) {
  int64_t g = (int64_t)kNumSMs * per_sm;
  if (nb < g) g = nb;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace krb
