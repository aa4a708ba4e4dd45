// k = 0 fused persistent BiCGSTAB with the operator held on chip (persist0).
//
// The unrecycled solve (bicgstab_solve, solvers.py:156-242; rbicgstab_solve
// with an empty space, :245-361) of a mid-size system (canon_E(n) == 1,
// n <= 303104) in ONE cooperative kernel, three grid barriers per
// iteration -- the same phases, formulas and canonical reductions as the
// k = 0 path of k_persist2 (persist.cu), so the results are bit-identical to
// it and to the CanonOps oracle.  What changes is where the SpMV operands
// live:
//
//  * each CTA owns canonical blocks me and me + G (1024 rows each); at kernel
//    start it copies its rows' matrix slots (SELL-32 or CSR, values + a
//    16-bit operand index per slot) into shared memory and builds its HALO:
//    the sorted list of off-block columns its rows reference (a bitmap over
//    the column space plus a block-wide prefix count, then compaction);
//  * a SpMV phase then gathers only the halo from L2 (all loads of a thread
//    issued together: one round trip) into the operand array xs = [own
//    rows' values | halo values], and runs every row entirely out of shared
//    memory -- no index loads, no dependent round trips per entry;
//  * the vectors other CTAs gather live in global memory: r and w = p -
//    omega q (for p' = r + beta w) and q (for s = r - alpha q); a thread's
//    own elements of them (and of x, rt0) are re-read in the same round trip
//    as the halo, so nothing but p', q, s, t is register-resident across
//    phases (no spills: with 220 KB of shared memory the L1 is too small to
//    hold spilled registers, and every spill reload would be an L2 trip).  p' and s are recomputed per gathered column from
//    them, with the reference's formulas (same bits).
//
//   A  p' = r + beta w;  q = A p';  (rt0, q), (q, q) -> alpha          | sync
//   C  s = r - alpha q;  t = A s;  (s, s), (t, t), (t, s) -> omega      | sync
//   E  x += alpha p' + omega s;  r = s - omega t;  w = p' - omega q;
//      (r, r), (rt0, r) -> beta, convergence                           | sync
//
// A CTA whose rows do not fit (wide rows, scattered columns: halo or slots
// over the shared-memory budget) runs its SpMV rows from global memory
// instead (same order, same bits); the choice is per CTA.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "iter.cuh"
#include "spmv.cuh"

namespace krb {
namespace p0 {

namespace cg = cooperative_groups;

constexpr int kOwn = 2;                    // canonical blocks per CTA (nb <= 2 G)
constexpr int kLoc = kOwn * kLanes;        // xs slots of the owned rows
constexpr int kDynBytes = 220 * 1024;      // dynamic shared memory per CTA
constexpr int kMaxXs = 65535;              // operand index is 16-bit
constexpr int kRows = 3;                   // wred rows per owned block
#ifndef KRB_P0_HU
#define KRB_P0_HU 5
#endif
constexpr int kHU = KRB_P0_HU;             // halo elements in flight per thread

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// warp stage of ND (2 or 3) dots: canonical 32-lane trees -> wred[row0 + d][warp]
template <int ND>
__device__ __forceinline__ void wstage(const double (&acc)[ND], double (*wred)[32], int row0) {
  constexpr int NCP = ND == 2 ? 2 : 4;
  constexpr int H = NCP == 2 ? 1 : 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v[NCP];
#pragma unroll
  for (int d = 0; d < NCP; ++d) v[d] = d < ND ? acc[d] : 0.0;
  int col;
  const double s = warp_tree_multi<NCP>(v, col);
  if ((lane & ((32 >> H) - 1)) == 0 && col < ND) wred[row0 + col][warp] = s;
}

// ---- barrier-free phase hand-off -----------------------------------------
// Each CTA writes its block partials of a phase to the phase's partial
// buffer and then publishes the phase epoch in its own flag with a release
// store (after a CTA barrier: cumulative over the CTA's stores of the phase,
// like the cooperative-groups barrier's release atomic).  Readers poll every
// CTA's flag -- one warp per CTA, relaxed loads all in flight at once, each
// flag on its own 128-byte line so a line is polled by the CTAs rather than
// by every warp of the grid -- then an acquire fence orders their reads of
// the partials and of the vectors the phase wrote (q; r, w).  No global
// atomic and no arrival counter: the last CTA's partials are visible one
// poll after its store.  Two partial buffers alternate by phase; a CTA can
// run at most one phase ahead of the slowest reader.
constexpr int kFlagStride = 32;   // unsigned ints between two CTAs' flags

__device__ __forceinline__ unsigned int ld_relaxed(const unsigned int *p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// CTA stage (after a __syncthreads): 32-warp trees; dot d of owned block bi
// -> part[d * nb + me + bi G]; then the release of the phase epoch
__device__ __forceinline__ void cstage(const double (*wred)[32], int nown, int nd, int me,
                                       int G, int nb, double *part, unsigned int *flags,
                                       unsigned int ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < nown * nd) {   // nown * nd <= 6: one tree per warp
    const int bi = warp >= nd ? 1 : 0, d = warp - bi * nd;
    const double v = warp_tree(wred[bi * kRows + d][lane]);
    if (lane == 0) part[d * nb + me + bi * G] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + me * kFlagStride), "r"(ep)
                 : "memory");
}

// canonical final stage of ND dots of phase ep (warp d: lane L sums blocks
// L, L + 32, ... in order, then the 32-lane tree), every CTA redundantly,
// once every CTA has published (warp 0 polls, G <= 160)
template <int ND>
__device__ __forceinline__ void await_finals(const double *part, int nb, double *dfin,
                                             const unsigned int *flags, int G,
                                             unsigned int ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    for (;;) {
      bool ok = true;
      unsigned int v[5];
#pragma unroll
      for (int u = 0; u < 5; ++u) {
        const int b = lane + 32 * u;
        v[u] = b < G ? ld_relaxed(flags + b * kFlagStride) : ep;
      }
#pragma unroll
      for (int u = 0; u < 5; ++u) ok = ok && (int)(v[u] - ep) >= 0;
      if (__all_sync(0xffffffffu, ok)) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();   // warp 0's acquire orders every warp's later reads
  if (warp < ND) {
    // warp_final_volatile's order (lane L: 0.0 + P[L] + P[L + 32] + ...),
    // all <= 10 loads per lane in flight, 32-bit indices (nb <= 320)
    const double *P = part + warp * nb;
    double v[10];
#pragma unroll
    for (int u = 0; u < 10; ++u) {
      const int b = lane + 32 * u;
      v[u] = b < nb ? __ldcg(P + b) : 0.0;
    }
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < 10; ++u)
      if (lane + 32 * u < nb) acc = __dadd_rn(acc, v[u]);
    acc = warp_tree(acc);
    if (lane == 0) dfin[warp] = acc;
  }
  __syncthreads();
}

// block-wide exclusive scan of one int per thread (1024 threads)
__device__ __forceinline__ int block_excl_scan(int v, int *sh, int &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int z = sh[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, off);
      if (lane >= off) z += y;
    }
    sh[lane] = z;
  }
  __syncthreads();
  const int excl = x - v + (warp > 0 ? sh[warp - 1] : 0);
  total = sh[31];
  __syncthreads();
  return excl;
}

// one row gathered from global memory (CTAs whose rows do not fit on chip):
// x[c] = u[c] + f v[c] (sign = +1: p' = r + beta w) or u[c] - f v[c]
// (sign = -1: s = r - alpha q), recomputed per column -- same bits as the
// owner's value.  Out of line: it keeps the on-chip path's registers free.
template <bool kSell, int kSign>
__device__ __noinline__ double row_global(int i, const krb_matrix &A, const double *u,
                                          const double *v, double f) {
  auto xf = [=](int c) {
    const double fv = __dmul_rn(f, __ldcg(v + c));
    return kSign > 0 ? __dadd_rn(__ldcg(u + c), fv) : __dsub_rn(__ldcg(u + c), fv);
  };
  return spmv_row_f<kSell>(i, A, xf);
}

template <bool kSell>
__global__ void __launch_bounds__(1024, 1)
    k_persist0(const __grid_constant__ IterArgs a, int force_global, int prof_cta) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ double wred[kOwn * kRows][32];
  __shared__ double dfin[3];
  __shared__ int scan_sh[32];
  __shared__ SolveScalars L;
  cg::grid_group grid = cg::this_grid();
  // n <= 303104 here: 32-bit indices throughout; the descriptor is a
  // kernel parameter (constant bank), so its pointers cost no registers
  const int G = gridDim.x, me = blockIdx.x;
  const int n = (int)a.n, nb = (int)a.nb;
  const int tid = threadIdx.x;
  const int nown = me < nb ? (nb - 1 - me) / G + 1 : 0;   // <= kOwn
  const bool writer = me == 0;
  const krb_matrix &A = a.A;
  constexpr int stride = kSell ? 32 : 1;
  const int32_t *__restrict__ gcol = kSell ? A.s_col : A.ci;
  const double *__restrict__ gval = kSell ? A.s_val : A.val;
  double *__restrict__ r = a.r;
  double *__restrict__ w = a.p2;   // w = p - omega q (solvers.py:303's inner term)
  double *__restrict__ q = a.q;
  double *__restrict__ x = a.x;
  const double *__restrict__ rt0 = a.rt0;
  const int b0 = me, b1 = nown > 1 ? me + G : -1;   // owned blocks (-1: none)
  auto row_of = [me, G, tid](int bi) { return (me + bi * G) * kLanes + tid; };
  if (tid == 0) L = *a.S;

  // ---- owned rows: metadata and vector elements in registers ------------
  bool ok[kOwn];
  int len[kOwn];
  int64_t gb[kOwn], bstart[kOwn], bend[kOwn];
  double pv0[kOwn], qv0[kOwn];
  int64_t cnt = 0;
  int loff[kOwn];
#pragma unroll
  for (int bi = 0; bi < kOwn; ++bi) {
    const int b = me + bi * G;
    const int i = b * kLanes + tid;
    ok[bi] = bi < nown && i < n;
    len[bi] = 0;
    gb[bi] = 0;
    pv0[bi] = qv0[bi] = 0.0;
    bstart[bi] = bend[bi] = 0;
    if (bi < nown) {
      if (kSell) {
        bstart[bi] = __ldg(A.sl_ptr + b * 32);
        bend[bi] = __ldg(A.sl_ptr + min64((int64_t)b * 32 + 32, A.nslices));
      } else {
        bstart[bi] = __ldg(A.rp + b * kLanes);
        bend[bi] = __ldg(A.rp + min64((int64_t)b * kLanes + kLanes, n));
      }
    }
    if (ok[bi]) {
      if (kSell) {
        len[bi] = __ldg(A.rlen + i);
        gb[bi] = __ldg(A.sl_ptr + (i >> 5)) + (i & 31);
      } else {
        gb[bi] = __ldg(A.rp + i);
        len[bi] = (int)(__ldg(A.rp + i + 1) - gb[bi]);
      }
      pv0[bi] = a.p[i];
      qv0[bi] = a.q[i];
    }
    loff[bi] = (int)cnt;
    cnt += bend[bi] - bstart[bi];
  }
  __syncthreads();   // L
  {
    // w for the first p' (p = q = 0 after setup; computed, not assumed)
    const double omega0 = L.omega;
#pragma unroll
    for (int bi = 0; bi < kOwn; ++bi) {
      if (ok[bi]) w[row_of(bi)] = __dsub_rn(pv0[bi], __dmul_rn(omega0, qv0[bi]));
    }
  }

  // ---- on-chip operator: slots + halo in shared memory -------------------
  double *xs = reinterpret_cast<double *>(dyn);
  uint16_t *midx = nullptr;
  int32_t *halo = nullptr;
  double *mval = nullptr;
  int nh = 0;
  const int nwords = (n + 31) >> 5;
  const int tmp_bytes = 6 * ((nwords + 1) & ~1);
  bool on_chip = !force_global && nown > 0 &&
                 (int64_t)kLoc * 8 + cnt * 10 + tmp_bytes <= kDynBytes;
  if (on_chip) {
    uint32_t *bm = reinterpret_cast<uint32_t *>(dyn + kDynBytes - 4 * ((nwords + 1) & ~1));
    uint16_t *wpre = reinterpret_cast<uint16_t *>(dyn + kDynBytes - tmp_bytes);
    for (int u = tid; u < nwords; u += kLanes) bm[u] = 0u;
    __syncthreads();
    // mark the off-block columns
#pragma unroll
    for (int bi = 0; bi < kOwn; ++bi) {
      if (!ok[bi]) continue;
      for (int j = 0; j < len[bi]; ++j) {
        const int c = __ldg(gcol + gb[bi] + (int64_t)j * stride);
        const int cb = c >> 10;
        if (cb != b0 && cb != b1) atomicOr(bm + (c >> 5), 1u << (c & 31));
      }
    }
    __syncthreads();
    // prefix count of the bitmap: thread t scans words [t per, (t + 1) per)
    const int per = (nwords + kLanes - 1) / kLanes;
    const int w0 = tid * per;
    int mine = 0;
    for (int u = 0; u < per; ++u)
      if (w0 + u < nwords) mine += __popc(bm[w0 + u]);
    int total = 0;
    int run = block_excl_scan(mine, scan_sh, total);
    nh = total;
    const int64_t xs_bytes = 8 * ((int64_t)kLoc + nh);
    const int64_t idx_bytes = (2 * cnt + 15) & ~(int64_t)15;
    const int64_t halo_bytes = (4 * (int64_t)nh + 15) & ~(int64_t)15;
    const int64_t val_off = xs_bytes + idx_bytes + halo_bytes;
    on_chip = kLoc + nh <= kMaxXs && val_off + 8 * cnt <= kDynBytes &&
              val_off <= kDynBytes - tmp_bytes;
    if (on_chip) {
      midx = reinterpret_cast<uint16_t *>(dyn + xs_bytes);
      halo = reinterpret_cast<int32_t *>(dyn + xs_bytes + idx_bytes);
      mval = reinterpret_cast<double *>(dyn + val_off);
      // word prefixes + compacted halo list (sorted by column)
      for (int u = 0; u < per; ++u) {
        const int wd = w0 + u;
        if (wd >= nwords) break;
        uint32_t bits = bm[wd];
        wpre[wd] = (uint16_t)run;
        while (bits) {
          const int bpos = __ffs(bits) - 1;
          halo[run++] = wd * 32 + bpos;
          bits &= bits - 1;
        }
      }
      __syncthreads();
      // operand index of every slot: own rows -> [0, kLoc), halo -> kLoc + rank
#pragma unroll
      for (int bi = 0; bi < kOwn; ++bi) {
        if (!ok[bi]) continue;
        const int base = loff[bi] + (int)(gb[bi] - bstart[bi]);
        for (int j = 0; j < len[bi]; ++j) {
          const int c = __ldg(gcol + gb[bi] + (int64_t)j * stride);
          const int cb = c >> 10;
          int xi;
          if (cb == b0) {
            xi = c - b0 * kLanes;
          } else if (cb == b1) {
            xi = kLanes + c - b1 * kLanes;
          } else {
            const uint32_t below = bm[c >> 5] & ((1u << (c & 31)) - 1u);
            xi = kLoc + wpre[c >> 5] + __popc(below);
          }
          midx[base + j * stride] = (uint16_t)xi;
        }
      }
      __syncthreads();   // bitmap and prefixes dead: the values go over them
#pragma unroll
      for (int bi = 0; bi < kOwn; ++bi) {
        const int64_t m = bend[bi] - bstart[bi];
        for (int64_t e = tid; e < m; e += kLanes) mval[loff[bi] + e] = __ldg(gval + bstart[bi] + e);
      }
    }
    __syncthreads();
  }
  unsigned int *flags = a.flags;
  unsigned int ep = 0;   // phase epoch (the same sequence on every CTA)
  if (tid == 0) flags[me * kFlagStride] = 0u;
  grid.sync();   // w (and the setup's r, q) visible to every CTA; flags reset

  int rb[kOwn];   // first shared-memory slot of each owned row
#pragma unroll
  for (int bi = 0; bi < kOwn; ++bi) rb[bi] = loff[bi] + (int)(gb[bi] - bstart[bi]);
  // one row, operands from shared memory (CSR order, mul then add)
  auto row_on_chip = [mval, midx, xs](int base, int n_ent) -> double {
    double sum = 0.0;
#pragma unroll 4
    for (int j = 0; j < n_ent; ++j) {
      const int e = base + j * stride;
      sum = __dadd_rn(sum, __dmul_rn(mval[e], xs[midx[e]]));
    }
    return sum;
  };

  int cur = 0;   // partial buffer: a.part / a.part2 alternate per phase
  // tuning "p0_prof_cta" picks the CTA whose phase stamps are recorded
  const bool profiling = me == prof_cta && a.prof != nullptr;
  uint64_t *prof = (profiling && tid == 0) ? a.prof : nullptr;
#define KRB_STAMP(slot)                                                        \
  do {                                                                         \
    if (profiling) __syncthreads();                                            \
    if (prof && L.itn < a.prof_cap) prof[L.itn * 16 + (slot)] = globaltimer(); \
  } while (0)
  for (;;) {
    if (L.status != KRB_RUNNING) break;
    const double beta = L.beta;
    KRB_STAMP(0);
    // ---- A: p' = r + beta w; q = A p'; (rt0, q), (q, q) ------------------
    double pp[kOwn], qq[kOwn], rta[kOwn];
#pragma unroll
    for (int bi = 0; bi < kOwn; ++bi) {
      // own r, w, rt0: loads issued with the halo gather (one round trip)
      const double rv = ok[bi] ? __ldcg(r + row_of(bi)) : 0.0;
      const double wv = ok[bi] ? __ldcg(w + row_of(bi)) : 0.0;
      rta[bi] = ok[bi] ? rt0[row_of(bi)] : 0.0;
      pp[bi] = __dadd_rn(rv, __dmul_rn(beta, wv));  // :303
    }
    if (on_chip) {
      for (int h0 = 0; h0 < nh; h0 += kHU * kLanes) {
        int c[kHU];
        double rv[kHU], wv[kHU];
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
          const int hh = h0 + u * kLanes + tid;
          c[u] = hh < nh ? halo[hh] : -1;
        }
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
          rv[u] = c[u] >= 0 ? __ldcg(r + c[u]) : 0.0;
          wv[u] = c[u] >= 0 ? __ldcg(w + c[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kHU; ++u)
          if (c[u] >= 0) xs[kLoc + h0 + u * kLanes + tid] = __dadd_rn(rv[u], __dmul_rn(beta, wv[u]));
      }
      // own rows last: their loads share the halo's round trip
#pragma unroll
      for (int bi = 0; bi < kOwn; ++bi)
        if (bi < nown) xs[bi * kLanes + tid] = pp[bi];
      __syncthreads();
      KRB_STAMP(13);
#pragma unroll
      for (int bi = 0; bi < kOwn; ++bi) qq[bi] = ok[bi] ? row_on_chip(rb[bi], len[bi]) : 0.0;
      KRB_STAMP(14);
    } else {
#pragma unroll
      for (int bi = 0; bi < kOwn; ++bi)
        qq[bi] = ok[bi] ? row_global<kSell, 1>(row_of(bi), A, r, w, beta) : 0.0;
    }
#pragma unroll
    for (int bi = 0; bi < kOwn; ++bi) {
      if (bi >= nown) break;
      if (ok[bi]) q[row_of(bi)] = qq[bi];
      double acc[2] = {0.0, 0.0};
      if (ok[bi]) {
        acc[0] = __fma_rn(rta[bi], qq[bi], acc[0]);   // (rt0, q)
        acc[1] = __fma_rn(qq[bi], qq[bi], acc[1]);   // (q, q)
      }
      wstage<2>(acc, wred, bi * kRows);
    }
    KRB_STAMP(6);
    __syncthreads();
    ++ep;
    cstage(wred, nown, 2, me, G, nb, cur ? a.part2 : a.part, flags, ep);
    KRB_STAMP(7);
    await_finals<2>(cur ? a.part2 : a.part, nb, dfin, flags, G, ep);
    KRB_STAMP(8);
    cur ^= 1;
    if (tid == 0) finalize<PH_PROJ_Q>(a, &L, dfin, writer);
    __syncthreads();
    KRB_STAMP(2);
    if (L.status != KRB_RUNNING) break;
    const double alpha = L.alpha;
    // ---- C: s = r - alpha q; t = A s; (s, s), (t, t), (t, s) -------------
    double ss[kOwn], tt[kOwn];
#pragma unroll
    for (int bi = 0; bi < kOwn; ++bi) {
      const double rv = ok[bi] ? __ldcg(r + row_of(bi)) : 0.0;
      ss[bi] = __dsub_rn(rv, __dmul_rn(alpha, qq[bi]));  // :313
    }
    if (on_chip) {
      for (int h0 = 0; h0 < nh; h0 += kHU * kLanes) {
        int c[kHU];
        double rv[kHU], qv[kHU];
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
          const int hh = h0 + u * kLanes + tid;
          c[u] = hh < nh ? halo[hh] : -1;
        }
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
          rv[u] = c[u] >= 0 ? __ldcg(r + c[u]) : 0.0;
          qv[u] = c[u] >= 0 ? __ldcg(q + c[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kHU; ++u)
          if (c[u] >= 0) xs[kLoc + h0 + u * kLanes + tid] = __dsub_rn(rv[u], __dmul_rn(alpha, qv[u]));
      }
#pragma unroll
      for (int bi = 0; bi < kOwn; ++bi)
        if (bi < nown) xs[bi * kLanes + tid] = ss[bi];
      __syncthreads();
#pragma unroll
      for (int bi = 0; bi < kOwn; ++bi) tt[bi] = ok[bi] ? row_on_chip(rb[bi], len[bi]) : 0.0;
    } else {
#pragma unroll
      for (int bi = 0; bi < kOwn; ++bi)
        tt[bi] = ok[bi] ? row_global<kSell, -1>(row_of(bi), A, r, q, alpha) : 0.0;
    }
#pragma unroll
    for (int bi = 0; bi < kOwn; ++bi) {
      if (bi >= nown) break;
      double acc[3] = {0.0, 0.0, 0.0};
      if (ok[bi]) {
        acc[0] = __fma_rn(ss[bi], ss[bi], acc[0]);   // (s, s)
        acc[1] = __fma_rn(tt[bi], tt[bi], acc[1]);   // (t, t)
        acc[2] = __fma_rn(tt[bi], ss[bi], acc[2]);   // (t, s)
      }
      wstage<3>(acc, wred, bi * kRows);
    }
    // x and rt0 for E (and the half-step exit), in flight across the barrier
    double xe[kOwn], rte[kOwn];
#pragma unroll
    for (int bi = 0; bi < kOwn; ++bi) {
      xe[bi] = ok[bi] ? x[row_of(bi)] : 0.0;
      rte[bi] = ok[bi] ? rt0[row_of(bi)] : 0.0;
    }
    KRB_STAMP(9);
    __syncthreads();
    ++ep;
    cstage(wred, nown, 3, me, G, nb, cur ? a.part2 : a.part, flags, ep);
    KRB_STAMP(10);
    await_finals<3>(cur ? a.part2 : a.part, nb, dfin, flags, G, ep);
    KRB_STAMP(11);
    cur ^= 1;
    if (tid == 0) {
      finalize<PH_SUPD>(a, &L, dfin, writer);
      if (L.status == KRB_RUNNING) finalize<PH_PROJ_T>(a, &L, dfin + 1, writer);
    }
    __syncthreads();
    KRB_STAMP(3);
    if (L.status != KRB_RUNNING) {
      if (L.early) {
        // solvers.py:315-316: converged at the half step, x += alpha p
#pragma unroll
        for (int bi = 0; bi < kOwn; ++bi)
          if (ok[bi]) x[row_of(bi)] = __dadd_rn(xe[bi], __dmul_rn(alpha, pp[bi]));
      }
      break;
    }
    const double omega = L.omega;
    // ---- E: x, r, w; (r, r), (rt0, r) -------------------------------------
#pragma unroll
    for (int bi = 0; bi < kOwn; ++bi) {
      if (bi >= nown) break;
      double acc[2] = {0.0, 0.0};
      if (ok[bi]) {
        const int i = row_of(bi);
        x[i] = __dadd_rn(__dadd_rn(xe[bi], __dmul_rn(alpha, pp[bi])),
                         __dmul_rn(omega, ss[bi]));                     // :338
        const double rv = __dsub_rn(ss[bi], __dmul_rn(omega, tt[bi]));  // :341
        r[i] = rv;
        w[i] = __dsub_rn(pp[bi], __dmul_rn(omega, qq[bi]));   // next :303's inner term
        acc[0] = __fma_rn(rv, rv, acc[0]);
        acc[1] = __fma_rn(rte[bi], rv, acc[1]);
      }
      wstage<2>(acc, wred, bi * kRows);
    }
    KRB_STAMP(4);
    __syncthreads();
    ++ep;
    cstage(wred, nown, 2, me, G, nb, cur ? a.part2 : a.part, flags, ep);
    KRB_STAMP(1);
    await_finals<2>(cur ? a.part2 : a.part, nb, dfin, flags, G, ep);
    KRB_STAMP(12);
    cur ^= 1;
    KRB_STAMP(5);
    if (tid == 0) finalize<PH_XR>(a, &L, dfin, writer);
    __syncthreads();
  }
#undef KRB_STAMP
  if (writer && tid == 0) {
    L.bodies = L.itn;
    *a.S = L;
  }
}

}  // namespace p0

bool persist0_eligible(const IterArgs &h) {
  if (!tuning().persist0) return false;
  return h.k == 0 && h.A.perm == nullptr && canon_E(h.n) == 1 && h.n > 0 &&
         h.flags != nullptr;
}

template <bool kSell>
static int launch0(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  static int grid = 0;
  if (grid == 0) {
    KRB_CHECK_CUDA(cudaFuncSetAttribute(p0::k_persist0<kSell>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        p0::kDynBytes));
    int per_sm = 0;
    KRB_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, p0::k_persist0<kSell>, 1024, p0::kDynBytes));
    int dev = 0, sms = kNumSMs;
    KRB_CHECK_CUDA(cudaGetDevice(&dev));
    KRB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = per_sm > 0 ? sms : 0;
    if (grid == 0) {
      set_error("persist0 kernel does not fit on an SM");
      return KRB_ECUDA;
    }
  }
  const int64_t nb = h.nb;
  if ((int64_t)grid * p0::kOwn < nb) {
    set_error("persist0: %lld blocks > %d x %d CTAs", (long long)nb, p0::kOwn, grid);
    return KRB_EINVAL;
  }
  int g = nb < grid ? (int)nb : grid;
  // tuning "p0_grid_half": one CTA per two canonical blocks (every CTA owns two)
  if (tuning().p0_grid_half) g = (int)((nb + 1) / 2);
  if (g > 160) g = 160;   // flag slots reserved / polled (nb <= 296 < 2 x 160)
  int force_global = tuning().p0_onchip ? 0 : 1;
  int prof_cta = tuning().p0_prof_cta;
  IterArgs hv = h;   // by value: the kernel reads the descriptor from its parameters
  void *args[] = {(void *)&hv, (void *)&force_global, (void *)&prof_cta};
  KRB_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)p0::k_persist0<kSell>, dim3(g),
                                             dim3(1024), args, p0::kDynBytes, st));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

int persist0_launch(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  return h.A.format == 2 ? launch0<true>(h, d, st) : launch0<false>(h, d, st);
}

}  // namespace krb
