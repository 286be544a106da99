// Does a plain L2 hit tell an SM which die homes a 4 KB page?  Each CTA (one per SM) times a dependent
// chain of ld.global.cg loads over the 32 lines of page p (the lines first written by the host), for the
// first 8 pages of a 2 MB-aligned buffer.  Prints cycles per load, one row per SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_chase(const unsigned* buf, int npages, int reps, long long* out) {
  extern __shared__ char sm[];
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x) return;
  sm[0] = 0;
  for (int p = 0; p < npages; ++p) {
    const unsigned* pg = buf + (size_t)p * 1024;  // 4 KB page, 32 lines of 128 B: next index stored at line start
    unsigned i = 0;
    // warm the chain once (L2 fills), then time it
    for (int r = 0; r < 32; ++r) i = __ldcg(pg + i);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) i = __ldcg(pg + i);
    const long long t1 = clock64();
    out[smid * npages + p] = (t1 - t0) / reps + (i == 0xffffffffu);
  }
}

int main() {
  const int npages = 8, reps = 512;
  unsigned* d;
  cudaMalloc(&d, 4 << 20);
  unsigned h[1024 * npages];
  for (int p = 0; p < npages; ++p)
    for (int l = 0; l < 32; ++l) h[p * 1024 + l * 32] = ((l * 7 + 3) % 32) * 32;  // a cycle through the 32 lines
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  long long* o;
  cudaMalloc(&o, 148 * npages * sizeof(long long));
  cudaFuncSetAttribute(k_chase, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_chase<<<148, 32, 200 * 1024>>>(d, npages, reps, o);
  long long r[148 * npages];
  cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
  for (int s = 0; s < 148; ++s) {
    printf("sm%d", s);
    for (int p = 0; p < npages; ++p) printf(" %lld", r[s * npages + p]);
    printf("\n");
  }
  return 0;
}
