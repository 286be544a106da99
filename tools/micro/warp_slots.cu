// Which SM sub-partition does warp w of a CTA issue on?  Records %warpid (the warp's slot in the SM;
// sub-partition = slot mod 4) for every warp of every CTA, for 1 CTA of 480 threads per SM (the
// pipelined kernel's shape) and 2 CTAs of 192 threads per SM (k_fine at n = 256).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_slots(int* out) {
  extern __shared__ char sm[];
  unsigned wid, smid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if ((threadIdx.x & 31) == 0) {
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    out[2 * (blockIdx.x * nw + w)] = (int)wid;
    out[2 * (blockIdx.x * nw + w) + 1] = (int)smid;
    sm[w] = 1;
  }
  // stay resident long enough for the co-resident CTAs to be placed
  const long long t0 = clock64();
  while (clock64() - t0 < 2000000) {
  }
}

static void run(int threads, int blocks, int smem) {
  int* d;
  const int nw = threads / 32, n = 2 * blocks * nw;
  cudaMalloc(&d, n * sizeof(int));
  cudaFuncSetAttribute(k_slots, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_slots<<<blocks, threads, smem>>>(d);
  int* h = new int[n];
  cudaMemcpy(h, d, n * sizeof(int), cudaMemcpyDeviceToHost);
  printf("%d threads x %d CTAs, %d B smem: (CTA: sm | slot of warp 0..%d)\n", threads, blocks, smem, nw - 1);
  for (int b = 0; b < 6; ++b) {
    printf("  CTA %d: sm %d |", b, h[2 * (b * nw) + 1]);
    for (int w = 0; w < nw; ++w) printf(" %d", h[2 * (b * nw + w)]);
    printf("\n");
  }
  // histogram of slot mod 4 of warps 0..2 per SM (first 4 SMs)
  delete[] h;
  cudaFree(d);
}

int main() {
  run(480, 148, 150 * 1024);
  run(192, 296, 80 * 1024);
  run(192, 148, 80 * 1024);
  return 0;
}
