// Grid-barrier latency microbenchmark on B200 (cooperative launch, 1024-thread
// CTAs): flat atomic counter vs two-level counters vs cooperative_groups.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
struct GS { unsigned count, gen; unsigned sub[64][32]; };   // sub counters padded to 128 B

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_acqrel(unsigned* p, unsigned v) {
  unsigned old; asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory"); return old;
}

template <int kMode, int kGroup>
__global__ void __launch_bounds__(1024) kbar(GS* g, int iters) {
  for (int it = 0; it < iters; ++it) {
    if (kMode == 3) { cg::this_grid().sync(); continue; }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned ge = ld_acq(&g->gen);
      bool lead;
      if (kMode == 0) {            // flat: fence + atomic
        __threadfence();
        lead = atomicAdd(&g->count, 1u) == gridDim.x - 1;
      } else if (kMode == 1) {     // flat, acq_rel atomic (no separate fence)
        lead = atom_acqrel(&g->count, 1u) == gridDim.x - 1;
      } else {                     // two-level: group counters then top
        unsigned grp = blockIdx.x / kGroup;
        unsigned gsize = min((unsigned)kGroup, gridDim.x - grp * kGroup);
        unsigned ngroups = (gridDim.x + kGroup - 1) / kGroup;
        lead = false;
        if (atom_acqrel(&g->sub[grp][0], 1u) == gsize - 1) {
          g->sub[grp][0] = 0;
          lead = atom_acqrel(&g->count, 1u) == ngroups - 1;
        }
      }
      if (lead) { g->count = 0; red_rel(&g->gen, 1u); }
      else { while (ld_acq(&g->gen) == ge) { } }
    }
    __syncthreads();
  }
}
template <int M, int G>
void run(GS* g, int sms, int per, const char* name) {
  int iters = 4000; void* args[] = {&g, &iters};
  cudaMemset(g, 0, sizeof(GS));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaLaunchCooperativeKernel((const void*)kbar<M, G>, sms * per, 1024, args, 0, 0);
  cudaDeviceSynchronize();
  cudaMemset(g, 0, sizeof(GS));
  cudaEventRecord(a);
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)kbar<M, G>, sms * per, 1024, args, 0, 0);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-28s ctas/sm=%d err=%s  %.3f us/barrier\n", name, per, cudaGetErrorString(e), ms * 1000.0 / iters);
}
int main() {
  GS* g; cudaMalloc(&g, sizeof(GS));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per = 1; per <= 2; ++per) {
    run<0, 1>(g, sms, per, "flat fence+atomic");
    run<1, 1>(g, sms, per, "flat atom.acq_rel");
    run<2, 8>(g, sms, per, "two-level groups of 8");
    run<2, 16>(g, sms, per, "two-level groups of 16");
    run<2, 32>(g, sms, per, "two-level groups of 32");
    run<3, 1>(g, sms, per, "cooperative_groups grid.sync");
  }
  return 0;
}
