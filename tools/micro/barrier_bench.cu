// Microbenchmark: cost of a grid-wide barrier inside a cooperative persistent kernel on B200.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void bar_volatile(unsigned* bar, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nb - 1) { atomicExch(bar, 0u); __threadfence(); atomicAdd(bar + 1, 1u); }
    else { while (*gen == g) {} }
    __threadfence();
  }
  __syncthreads();
}

// release/acquire flavour: arrive with red.release.gpu, poll with ld.acquire.gpu
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void bar_acqrel(unsigned* bar, unsigned nb, unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    const unsigned target = epoch * nb;
    while (ld_acquire(bar) < target) {}
  }
  __syncthreads();
}

template <int MODE>
__global__ void kbar(unsigned* bar, int iters, long long* out) {
  unsigned epoch = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) bar_volatile(bar, gridDim.x);
    else if (MODE == 1) bar_acqrel(bar, gridDim.x, epoch);
    else cg::this_grid().sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  unsigned* bar; long long* out; cudaMalloc(&bar, 8); cudaMalloc(&out, 8);
  int iters = 20000;
  for (int grid : {16, 64, 128, 148}) {
    for (int mode = 0; mode < 3; ++mode) {
      cudaMemset(bar, 0, 8);
      void* args[] = {&bar, &iters, &out};
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e;
      if (mode == 0) e = cudaLaunchCooperativeKernel((void*)kbar<0>, grid, 128, args, 0, 0);
      else if (mode == 1) e = cudaLaunchCooperativeKernel((void*)kbar<1>, grid, 128, args, 0, 0);
      else e = cudaLaunchCooperativeKernel((void*)kbar<2>, grid, 128, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("grid %3d mode %d (%s): %.3f us/barrier  err=%s\n", grid, mode,
             mode == 0 ? "volatile+atomicAdd" : mode == 1 ? "release/acquire counter" : "cg grid.sync",
             ms * 1e3 / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}
