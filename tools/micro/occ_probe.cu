// Does the CUDA occupancy calculator (used by cooperative launches) treat kernels that allocate
// tensor memory differently?  Compares the same kernel with and without tcgen05.alloc.
#include <cstdio>
#include <cstdint>
template <bool TMEM>
__global__ void __launch_bounds__(192, 2) kprobe(double* out) {
  __shared__ uint32_t slot;
  extern __shared__ double sm[];
  if (TMEM && (threadIdx.x >> 5) == 0) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(&slot);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(s) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[5];
  if (TMEM && (threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(slot) : "memory");
}
int main() {
  for (int t = 0; t < 2; ++t) {
    auto k = t ? kprobe<true> : kprobe<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    for (int kb : {16, 80}) {
      int o = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, 192, kb * 1024);
      printf("tmem=%d dyn=%dKB occupancy=%d\n", t, kb, o);
    }
  }
  return 0;
}
