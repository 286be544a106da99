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

// flag barrier: every CTA publishes its epoch in its own flag (no same-address atomics); thread t
// of every CTA polls flag t (all flags polled in parallel), then a CTA barrier.  STRIDE u32 per flag.
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <int STRIDE>
__device__ __forceinline__ void bar_flags(unsigned* flags, unsigned nb, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) st_release(flags + blockIdx.x * STRIDE, epoch);
  if (threadIdx.x < nb) {
    while ((int)(ld_acquire(flags + threadIdx.x * STRIDE) - epoch) < 0) {}
  }
  __syncthreads();
}
// hierarchical counter: groups of 8 CTAs arrive on their own counter; the last of a group
// arrives on the top counter; everyone polls the top counter
__device__ __forceinline__ void bar_hier(unsigned* bar, unsigned nb, unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned g = blockIdx.x / 8, gs = min(8u, nb - g * 8), ng = (nb + 7) / 8;
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar + 64 + g * 32) : "memory");
    if (old + 1 == epoch * gs) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    while (ld_acquire(bar) < epoch * ng) {}
  }
  __syncthreads();
}

// latency floors: flags without any fence (not a valid data barrier; MODE 6), and with
// __threadfence() on the writer side only before the flag store (MODE 7)
template <bool FENCE>
__device__ __forceinline__ void bar_flags_weak(unsigned* flags, unsigned nb, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) {
    if (FENCE) __threadfence();
    *(volatile unsigned*)(flags + blockIdx.x * 32) = epoch;
  }
  if (threadIdx.x < nb) {
    while ((int)(*(volatile unsigned*)(flags + threadIdx.x * 32) - epoch) < 0) {}
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
    else if (MODE == 2) cg::this_grid().sync();
    else if (MODE == 3) bar_flags<32>(bar + 4096, gridDim.x, epoch);
    else if (MODE == 4) bar_flags<1>(bar + 4096, gridDim.x, epoch);
    else if (MODE == 5) bar_hier(bar, gridDim.x, epoch);
    else if (MODE == 6) bar_flags_weak<false>(bar + 4096, gridDim.x, epoch);
    else bar_flags_weak<true>(bar + 4096, gridDim.x, epoch);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  unsigned* bar; long long* out; cudaMalloc(&bar, 65536 * 4); cudaMalloc(&out, 8);
  int iters = 20000;
  for (int grid : {16, 64, 128, 148}) {
    for (int mode = 0; mode < 8; ++mode) {
      cudaMemset(bar, 0, 65536 * 4);
      void* args[] = {&bar, &iters, &out};
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e;
      if (mode == 0) e = cudaLaunchCooperativeKernel((void*)kbar<0>, grid, 128, args, 0, 0);
      else if (mode == 1) e = cudaLaunchCooperativeKernel((void*)kbar<1>, grid, 128, args, 0, 0);
      else if (mode == 2) e = cudaLaunchCooperativeKernel((void*)kbar<2>, grid, 128, args, 0, 0);
      else if (mode == 3) e = cudaLaunchCooperativeKernel((void*)kbar<3>, grid, 192, args, 0, 0);
      else if (mode == 4) e = cudaLaunchCooperativeKernel((void*)kbar<4>, grid, 192, args, 0, 0);
      else if (mode == 5) e = cudaLaunchCooperativeKernel((void*)kbar<5>, grid, 128, args, 0, 0);
      else if (mode == 6) e = cudaLaunchCooperativeKernel((void*)kbar<6>, grid, 192, args, 0, 0);
      else e = cudaLaunchCooperativeKernel((void*)kbar<7>, grid, 192, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("grid %3d mode %d (%s): %.3f us/barrier  err=%s\n", grid, mode,
             mode == 0 ? "volatile+atomicAdd" : mode == 1 ? "release/acquire counter" : mode == 2 ? "cg grid.sync"
             : mode == 3 ? "per-CTA flags, 128B apart" : mode == 4 ? "per-CTA flags, packed" : mode == 5 ? "8-way hierarchical counter"
             : mode == 6 ? "volatile flags, no fence (floor)" : "threadfence + volatile flags",
             ms * 1e3 / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}
