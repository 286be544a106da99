// Feasibility probe for a cluster-based pipelined sweep: how many 8/16-CTA clusters can a cooperative
// launch co-schedule when every CTA allocates tensor memory and takes ~130 KB of shared memory
// (one CTA per SM)?  And what does a DSMEM gather of 64 per-pair partials (fixed order) cost?
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(352, 1) kprobe(double* out, int iters, long long* cyc) {
  __shared__ uint32_t slot;
  extern __shared__ double2 sm[];
  cg::cluster_group cl = cg::this_cluster();
  if ((threadIdx.x >> 5) == 0) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(&slot);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 4 * 513; i += blockDim.x) sm[i] = make_double2(i + blockIdx.x, 1.0);
  cl.sync();
  const unsigned nb = cl.num_blocks(), me = cl.block_rank();
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // owner gather: this CTA owns 32 entries; lanes q = 0..7 of an entry read the partials of pairs
    // q, q+8, ... (pair b lives in CTA b % nb, slot b / nb), 8 loads in flight, summed in order
    const int item = threadIdx.x / 8, q = threadIdx.x % 8;
    if (item < 32) {
      double2 buf[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = q + 8 * u;  // 64 pairs
        const double2* rem = cl.map_shared_rank(sm, b % nb);
        buf[u] = rem[(b / nb) * 513 + me * 32 + item];
      }
      double2 s = make_double2(0, 0);
#pragma unroll
      for (int u = 0; u < 8; ++u) { s.x += buf[u].x; s.y += buf[u].y; }
      acc += s.x;
      // broadcast: owner writes its 32 entries into every CTA's replica (slot 3)
      if (q == 0)
        for (unsigned r = 0; r < nb; ++r) cl.map_shared_rank(sm, r)[3 * 513 + me * 32 + item] = s;
    }
    cl.sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  if (acc == 1234.5) out[0] = acc;
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  const size_t smem = 130 * 1024;
  cudaFuncSetAttribute(kprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kprobe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(352); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 2;
    cfg.gridDim = dim3(cs);
    int maxc = 0;
    cudaError_t eq = cudaOccupancyMaxActiveClusters(&maxc, kprobe, &cfg);
    printf("cluster %d: max active clusters %d (%s)\n", cs, maxc, cudaGetErrorString(eq));
    for (int ncl : {1, maxc}) {
      if (ncl < 1) continue;
      cfg.gridDim = dim3(cs * ncl);
      int iters = 2000;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchKernelEx(&cfg, kprobe, out, iters, cyc);
      cudaEventRecord(b); cudaError_t e2 = cudaEventSynchronize(b);
      float ms = 0; cudaEventElapsedTime(&ms, a, b);
      printf("  %d clusters: %.3f us per gather+broadcast+cluster.sync  launch=%s sync=%s\n", ncl, ms * 1e3 / iters,
             cudaGetErrorString(e), cudaGetErrorString(e2));
      cudaGetLastError();
    }
  }
  return 0;
}
