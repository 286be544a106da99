// Does a warp with only 16 active lanes issue FP64 work at twice the instruction rate of a full warp?
// (B200: 16 FP64 lanes per SM sub-partition, a full-warp DFMA occupies the unit for 2 cycles.)
// One CTA of W warps per SM sub-partition, dependent-free DFMA chains; time per instruction.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dp(double* out, int iters, int active) {
  const int lane = threadIdx.x & 31;
  if (lane >= active) return;
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 12345.0) out[0] = 1;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048;
  for (int warps : {1, 2, 4, 8}) {
    for (int active : {32, 16, 8}) {
      k_dp<<<148, 32 * warps>>>(d, 64, active);
      cudaEventRecord(e0);
      k_dp<<<148, 32 * warps>>>(d, iters, active);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double winst = 148.0 * warps * iters * 16 * 8;  // warp-instructions
      printf("warps/SM %d active lanes %2d: %.3f ms, %.3f warp-DFMA per SM-cycle @1.965GHz\n", warps, active, ms,
             winst / 148.0 / (ms * 1e-3 * 1.965e9));
    }
  }
  return 0;
}
