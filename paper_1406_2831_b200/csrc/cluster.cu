// Single-cluster RBiCGSTAB for tiny systems (n <= 16384, k <= 10: C1): one
// thread-block cluster of nb <= 16 CTAs x 1024 threads, CTA r owning the
// canonical block r (E = 1: 1024 rows / elements).  Everything the iteration
// touches lives on chip:
//   * the CTA's rows of Chat and C in its shared memory (16 KB per column
//     pair), loaded once per solve;
//   * the vectors other CTAs gather for the SpMV (r, p, q; p and q
//     double-buffered) in shared memory, read by the neighbours through
//     distributed shared memory (DSMEM) -- p' = r + beta (p - omega q) and
//     s = r - alpha q are recomputed on the fly per gathered column, as in the
//     grid-wide fused kernel (same formula, same bits);
//   * x, s, t, rt0 and the CTA's q / p in registers;
//   * block partials of every dot in shared memory, the canonical final
//     stages read them from all CTAs of the cluster through DSMEM.
// Phases are separated by hardware cluster barriers (barrier.cluster with
// release / acquire semantics) instead of grid-wide software barriers.
// The arithmetic is exactly the fused persistent kernel's (persist.cu), so
// the results are bit-identical to every other driver.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "iter.cuh"
#include "spmv.cuh"

namespace krb {

namespace cgc = cooperative_groups;

constexpr int kClMaxK = 10;
constexpr int kClMaxCTAs = 16;
constexpr int kClSlots = kClMaxK + 3;   // dot partial slots per phase
constexpr size_t kClSmem = sizeof(double) * (2 * kClMaxK * kLanes + 5 * kLanes);

struct ClShared {
  double part[2][kClSlots];   // block partials, ping-pong by phase
  double zeta[kClMaxK], gamma[kClMaxK], xc[kClMaxK];
  double dfin[4];
  double red[8][32];
  double red16[16][32];
  SolveScalars L;
};

__device__ __forceinline__ void cl_sync(cgc::cluster_group &cl) {
  cl.sync();   // barrier.cluster.arrive.release + wait.acquire
}

// canonical block stage of ND <= 2 dots (1024 lanes) -> this CTA's slot
template <int ND>
__device__ __forceinline__ void cl_block(double (&acc)[2], ClShared &sh, double *slot) {
  double r = block_tree_multi<ND>(acc, sh.red);
  const int warp = threadIdx.x >> 5;
  if (warp < ND && (threadIdx.x & 31) == 0) slot[warp] = r;
}

// canonical block stage of the k <= 16 projection columns at once: per-warp
// transposed 8-column trees, one CTA barrier, then warp c runs the 32-warp
// tree of column c (bit-identical to k separate block trees)
__device__ __forceinline__ void cl_block_cols(const double *col0, double v, bool own, int k,
                                              double (*red16)[32], double *slot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (8 * h >= k) break;
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int j = 8 * h + c;
      acc[c] = (own && j < k) ? __fma_rn(col0[j * kLanes + threadIdx.x], v, 0.0) : 0.0;
    }
    int col;
    double w = warp_tree_multi<8>(acc, col);
    if ((lane & 3) == 0) red16[8 * h + col][warp] = w;
  }
  __syncthreads();
  if (warp < k) {
    double r = warp_tree(red16[warp][lane]);
    if (lane == 0) slot[warp] = r;
  }
  __syncthreads();
}

// canonical final stage of partial d over the cluster's nb blocks (one warp)
__device__ __forceinline__ double cl_final(cgc::cluster_group &cl, ClShared &sh, int buf,
                                           int d, int nb) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  if (lane < nb) {
    const ClShared *rs = cl.map_shared_rank(&sh, lane);
    v = __dadd_rn(0.0, rs->part[buf][d]);   // lane L sums partials L, L + 32, ...
  }
  return warp_tree(v);
}

template <bool kSell>
__global__ void __launch_bounds__(1024, 1) k_cluster(const IterArgs *__restrict__ pa) {
  extern __shared__ __align__(16) double dyn[];
  __shared__ ClShared sh;
  cgc::cluster_group cl = cgc::this_cluster();
  const IterArgs &a = *pa;
  const int nb = (int)a.nb, k = a.k, n = (int)a.n;
  const int me = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const int i = me * kLanes + tid;     // owned element / row
  const bool own = i < n;
  const bool writer = me == 0;
  const krb_matrix A = a.A;
  double *sChat = dyn;                       // [k][1024]
  double *sC = dyn + kClMaxK * kLanes;       // [k][1024]
  double *sr = dyn + 2 * kClMaxK * kLanes;   // r
  double *sp[2] = {sr + kLanes, sr + 2 * kLanes};   // p old / new
  double *sq[2] = {sr + 3 * kLanes, sr + 4 * kLanes};   // q old / new
  // ---- load the solve state and the recycle rows ----------------------
  for (int j = 0; j < k; ++j) {
    sChat[j * kLanes + tid] = own ? a.Chat[(int64_t)j * a.ld + i] : 0.0;
    sC[j * kLanes + tid] = own ? a.C[(int64_t)j * a.ld + i] : 0.0;
  }
  sr[tid] = own ? a.r[i] : 0.0;
  sp[0][tid] = own ? a.p[i] : 0.0;
  sq[0][tid] = own ? a.q[i] : 0.0;
  double x = own ? a.x[i] : 0.0;
  const double rt0 = own ? a.rt0[i] : 0.0;
  if (tid == 0) sh.L = *a.S;
  for (int j = tid; j < k; j += blockDim.x) sh.xc[j] = a.xc[j];
  cl_sync(cl);

  int po = 0, buf = 0;
  double preg = 0.0, qreg = 0.0, sreg = 0.0, treg = 0.0;
  SolveScalars &L = sh.L;
  uint64_t *prof = (writer && tid == 0) ? a.prof : nullptr;   // KRB_PHASE_PROF
#define CL_STAMP(slot)                                                          \
  do {                                                                          \
    if (prof && L.itn < a.prof_cap) prof[L.itn * 16 + (slot)] = globaltimer(); \
  } while (0)
  const int warp = tid >> 5, lane = tid & 31;
  for (;;) {
    if (L.status != KRB_RUNNING) break;
    const double omega0 = L.omega, beta = L.beta;
    CL_STAMP(0);
    // ---- A: p' on the fly, q' = A p', Chat^T q' (or, k = 0, the B dots)
    {
      auto pf = [&](int c) {
        const int owner = c >> 10, l = c & (kLanes - 1);
        const double *r_ = cl.map_shared_rank(sr, owner);
        const double *p_ = cl.map_shared_rank(sp[po], owner);
        const double *q_ = cl.map_shared_rank(sq[po], owner);
        return __dadd_rn(r_[l], __dmul_rn(beta, __dsub_rn(p_[l], __dmul_rn(omega0, q_[l]))));
      };
      preg = qreg = 0.0;
      if (own) {
        preg = __dadd_rn(sr[tid], __dmul_rn(beta, __dsub_rn(sp[po][tid],
                                                           __dmul_rn(omega0, sq[po][tid]))));
        qreg = spmv_row_f<kSell>(i, A, pf);
      }
      sp[po ^ 1][tid] = preg;
      sq[po ^ 1][tid] = qreg;
      if (k > 0) {
        cl_block_cols(sChat, qreg, own, k, sh.red16, &sh.part[buf][0]);   // Chat^T q'
      } else {
        double acc[2] = {0.0, 0.0};
        if (own) {
          acc[0] = __fma_rn(rt0, qreg, 0.0);    // (rt0, q)
          acc[1] = __fma_rn(qreg, qreg, 0.0);   // (q, q)
        }
        cl_block<2>(acc, sh, &sh.part[buf][0]);
      }
    }
    CL_STAMP(1);
    cl_sync(cl);
    CL_STAMP(2);
    if (k > 0) {
      for (int j = warp; j < k; j += 32) {
        double v = cl_final(cl, sh, buf, j, nb);
        if (lane == 0) sh.zeta[j] = v;
      }
      __syncthreads();
      buf ^= 1;
      // ---- B: q' -= C zeta ; (rt0, q'), (q', q')
      double acc[2] = {0.0, 0.0};
      if (own) {
        double cz = 0.0;
        for (int j = 0; j < k; ++j) cz = __fma_rn(sC[j * kLanes + tid], sh.zeta[j], cz);
        qreg = __dsub_rn(qreg, cz);   // solvers.py:307
        acc[0] = __fma_rn(rt0, qreg, 0.0);
        acc[1] = __fma_rn(qreg, qreg, 0.0);
      }
      sq[po ^ 1][tid] = qreg;
      cl_block<2>(acc, sh, &sh.part[buf][0]);
      CL_STAMP(3);
      cl_sync(cl);
      CL_STAMP(4);
    }
    if (warp < 2) {
      double v = cl_final(cl, sh, buf, warp, nb);
      if (lane == 0) sh.dfin[warp] = v;
    }
    __syncthreads();
    buf ^= 1;
    if (tid == 0) finalize<PH_PROJ_Q>(a, &L, sh.dfin, writer);
    __syncthreads();
    CL_STAMP(5);
    if (L.status != KRB_RUNNING) break;
    const double alpha = L.alpha;
    // ---- C: s = r - alpha q' ; (s, s) ; t = A s ; Chat^T t (k = 0: D dots)
    {
      const int qn = po ^ 1;
      auto sf = [&](int c) {
        const int owner = c >> 10, l = c & (kLanes - 1);
        const double *r_ = cl.map_shared_rank(sr, owner);
        const double *q_ = cl.map_shared_rank(sq[qn], owner);
        return __dsub_rn(r_[l], __dmul_rn(alpha, q_[l]));
      };
      sreg = treg = 0.0;
      if (own) {
        sreg = __dsub_rn(sr[tid], __dmul_rn(alpha, qreg));   // solvers.py:313
        treg = spmv_row_f<kSell>(i, A, sf);
      }
      double acc[2] = {own ? __fma_rn(sreg, sreg, 0.0) : 0.0, 0.0};
      cl_block<1>(acc, sh, &sh.part[buf][kClMaxK + 2]);   // (s, s)
      if (k > 0) {
        cl_block_cols(sChat, treg, own, k, sh.red16, &sh.part[buf][0]);   // Chat^T t
      } else {
        double ac[2] = {0.0, 0.0};
        if (own) {
          ac[0] = __fma_rn(treg, treg, 0.0);   // (t, t)
          ac[1] = __fma_rn(treg, sreg, 0.0);   // (t, s)
        }
        cl_block<2>(ac, sh, &sh.part[buf][0]);
      }
    }
    CL_STAMP(6);
    cl_sync(cl);
    if (warp == 31) {
      double v = cl_final(cl, sh, buf, kClMaxK + 2, nb);
      if (lane == 0) sh.dfin[0] = v;
    }
    if (k > 0) {
      for (int j = warp; j < k; j += 32) {
        double v = cl_final(cl, sh, buf, j, nb);
        if (lane == 0) sh.gamma[j] = v;
      }
    } else if (warp < 2) {
      double v = cl_final(cl, sh, buf, warp, nb);
      if (lane == 0) sh.dfin[1 + warp] = v;
    }
    __syncthreads();
    buf ^= 1;
    if (tid == 0) finalize<PH_SUPD>(a, &L, sh.dfin, writer);
    __syncthreads();
    CL_STAMP(7);
    if (L.status != KRB_RUNNING) {
      // solvers.py:315-325: x += alpha p, xc += alpha zeta
      if (own) x = __dadd_rn(x, __dmul_rn(alpha, preg));
      for (int j = tid; j < k; j += blockDim.x)
        sh.xc[j] = __dadd_rn(sh.xc[j], __dmul_rn(alpha, sh.zeta[j]));
      __syncthreads();
      break;
    }
    // ---- D: t -= C gamma ; (t, t), (t, s)   (k = 0: finalized from C)
    if (k > 0) {
      double acc[2] = {0.0, 0.0};
      if (own) {
        double cg = 0.0;
        for (int j = 0; j < k; ++j) cg = __fma_rn(sC[j * kLanes + tid], sh.gamma[j], cg);
        treg = __dsub_rn(treg, cg);   // solvers.py:329
        acc[0] = __fma_rn(treg, treg, 0.0);
        acc[1] = __fma_rn(treg, sreg, 0.0);
      }
      cl_block<2>(acc, sh, &sh.part[buf][0]);
      cl_sync(cl);
      if (warp < 2) {
        double v = cl_final(cl, sh, buf, warp, nb);
        if (lane == 0) sh.dfin[1 + warp] = v;
      }
      __syncthreads();
      buf ^= 1;
    }
    if (tid == 0) finalize<PH_PROJ_T>(a, &L, sh.dfin + 1, writer);
    __syncthreads();
    CL_STAMP(8);
    if (L.status != KRB_RUNNING) break;
    const double omega = L.omega;
    // ---- E: x += alpha p' + omega s ; r = s - omega t ; (r, r), (rt0, r)
    {
      double acc[2] = {0.0, 0.0};
      if (own) {
        x = __dadd_rn(__dadd_rn(x, __dmul_rn(alpha, preg)), __dmul_rn(omega, sreg));   // :338
        const double rv = __dsub_rn(sreg, __dmul_rn(omega, treg));                     // :341
        sr[tid] = rv;
        acc[0] = __fma_rn(rv, rv, 0.0);
        acc[1] = __fma_rn(rt0, rv, 0.0);
      }
      cl_block<2>(acc, sh, &sh.part[buf][0]);
      for (int j = tid; j < k; j += blockDim.x)   // solvers.py:340
        sh.xc[j] = __dadd_rn(__dadd_rn(sh.xc[j], __dmul_rn(alpha, sh.zeta[j])),
                             __dmul_rn(omega, sh.gamma[j]));
    }
    cl_sync(cl);
    if (warp < 2) {
      double v = cl_final(cl, sh, buf, warp, nb);
      if (lane == 0) sh.dfin[warp] = v;
    }
    __syncthreads();
    buf ^= 1;
    CL_STAMP(9);
    if (tid == 0) finalize<PH_XR>(a, &L, sh.dfin, writer);
    __syncthreads();
    po ^= 1;
  }
#undef CL_STAMP
  // ---- write back what the tail needs -----------------------------------
  if (own) a.x[i] = x;
  if (writer) {
    if (tid == 0) {
      L.bodies = L.itn;
      *a.S = L;
    }
    for (int j = tid; j < k; j += blockDim.x) {
      a.xc[j] = sh.xc[j];
      a.zeta[j] = sh.zeta[j];
      a.gamma[j] = sh.gamma[j];
    }
  }
  cl_sync(cl);   // no CTA may exit while others still read its shared memory
}

bool cluster_eligible(const IterArgs &h) {
  if (!tuning().cluster) return false;
  return h.n > 0 && h.nb <= kClMaxCTAs && canon_E(h.n) == 1 && h.k <= kClMaxK &&
         h.A.perm == nullptr;
}

template <bool kSell>
static int cluster_launch_t(const IterArgs *d, int nb, cudaStream_t st) {
  static int ready = 0;   // 1 ok, -1 unavailable
  if (ready == 0) {
    ready = -1;
    if (cudaFuncSetAttribute(k_cluster<kSell>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kClSmem) == cudaSuccess &&
        cudaFuncSetAttribute(k_cluster<kSell>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                             1) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kClMaxCTAs);
      cfg.blockDim = dim3(1024);
      cfg.dynamicSmemBytes = kClSmem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kClMaxCTAs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int clusters = 0;
      if (cudaOccupancyMaxActiveClusters(&clusters, k_cluster<kSell>, &cfg) == cudaSuccess &&
          clusters > 0)
        ready = 1;
    }
    cudaGetLastError();
  }
  if (ready < 0) return KRB_EINVAL;   // caller falls back
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = kClSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nb;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KRB_CHECK_CUDA(cudaLaunchKernelEx(&cfg, k_cluster<kSell>, d));
  KRB_CHECK_LAUNCH();
  return KRB_OK;
}

// returns KRB_EINVAL (nothing launched) when clusters of this size cannot be
// scheduled, so the caller can use the grid-wide kernel
int cluster_launch(const IterArgs &h, const IterArgs *d, cudaStream_t st) {
  return h.A.format == 2 ? cluster_launch_t<true>(d, (int)h.nb, st)
                         : cluster_launch_t<false>(d, (int)h.nb, st);
}

}  // namespace krb
