// Microbenchmark: can a cooperative (co-resident) persistent kernel also use thread-block clusters
// on B200, and what do cluster.sync() and a DSMEM read cost?  (Informs the coarse-sweep design.)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void grid_bar(unsigned* bar, unsigned nb, unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    while (ld_acquire(bar) < epoch * nb) {}
  }
  __syncthreads();
}

__global__ void kmix(unsigned* bar, int iters, int mode, long long* out, double* sink) {
  __shared__ double buf[1024];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = i + blockIdx.x;
  cl.sync();
  unsigned epoch = 0;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) cl.sync();
    else if (mode == 1) grid_bar(bar, gridDim.x, epoch);
    else {  // DSMEM: read 8 values from every CTA of the cluster, then cluster.sync
      const unsigned r = cl.num_blocks();
      for (unsigned b = 0; b < r; ++b) {
        const double* rb = cl.map_shared_rank(buf, b);
        acc += rb[(threadIdx.x * 8 + it) & 1023];
      }
      cl.sync();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  unsigned* bar; long long* out; double* sink;
  cudaMalloc(&bar, 8); cudaMalloc(&out, 8); cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(kmix, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {8, 16}) {
    for (int grid : {64, 128}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = 0;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
      cfg.attrs = at; cfg.numAttrs = 2;
      int maxc = 0;
      cudaOccupancyMaxActiveClusters(&maxc, kmix, &cfg);
      for (int mode = 0; mode < 3; ++mode) {
        cudaMemset(bar, 0, 8);
        int iters = 20000;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelEx(&cfg, kmix, bar, iters, mode, out, sink);
        cudaEventRecord(b); cudaError_t e2 = cudaEventSynchronize(b);
        float ms = 0; cudaEventElapsedTime(&ms, a, b);
        printf("cluster %2d grid %3d maxActiveClusters %3d mode %d (%s): %.3f us/iter  launch=%s sync=%s\n", cs, grid, maxc, mode,
               mode == 0 ? "cluster.sync" : mode == 1 ? "grid barrier" : "DSMEM 1 read/CTA + cluster.sync",
               ms * 1e3 / iters, cudaGetErrorString(e), cudaGetErrorString(e2));
        if (e != cudaSuccess || e2 != cudaSuccess) { cudaGetLastError(); }
      }
    }
  }
  return 0;
}
