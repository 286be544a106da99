// rsw_k_fine.cu — fine propagator kernels (a2 ETDRK4 / a2' Strang) and their launcher.
#include "rsw_blocks.cuh"

#include <cstdlib>

namespace rsw {

template <typename KernelT>
static cudaError_t set_smem(KernelT k, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

#define RSW_DISPATCH(n, CALL)                  \
  switch (n) {                                 \
    case 16: return CALL(16);                  \
    case 32: return CALL(32);                  \
    case 64: return CALL(64);                  \
    case 128: return CALL(128);                \
    case 256: return CALL(256);                \
    case 512: return CALL(512);                \
    case 1024: return CALL(1024);              \
    default: return cudaErrorInvalidValue;     \
  }



template <int N, int R, int T>
struct FineLayout {  // dynamic shared memory of k_fine (double2 units first, then doubles)
  static constexpr int K = N / 3, KP = K + 1;
  static constexpr int W = 0, Y = W + 3 * N, TW = Y + 3 * N, CP = TW + fft_tw_size<N, R>(), D = CP + 6 * KP;
  static constexpr int C0 = 0, GA = C0 + 6 * KP, GP = GA + KP, GQ = GP + KP, ND = GQ + KP;      // double offsets
  static constexpr size_t bytes = sizeof(double2) * D + sizeof(double) * ND;
  static constexpr int NCOL = tmem_cols_pow2<FineTmem<N, T>::COLS>();
};

template <int N, int R, int T, int SCHEME, bool LIN>
__global__ void __launch_bounds__(T) k_fine(const double* u_in, double* u_out, int n_slices, int m_steps,
                                            double h, const FineTab tab) {
  using LY = FineLayout<N, R, T>;
  constexpr int NH = N / 2 + 1;
  extern __shared__ double2 smem[];
  __shared__ uint32_t tslot;
  if ((threadIdx.x >> 5) == 0) tmem_alloc<LY::NCOL>(&tslot);
  const FineSmemTab st_ = stage_fine_tables<N, R, T>(smem + LY::TW, smem + LY::CP,
                                                     reinterpret_cast<double*>(smem + LY::D), tab, threadIdx.x, T);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const int sA = 2 * blockIdx.x, sB = sA + 1;
  const size_t L = (size_t)3 * NH * 2;
  fine_pair_run<N, R, T, SCHEME, LIN>(CtaGroup(), smem + LY::W, smem + LY::Y, st_, tslot, tab.g, u_in + sA * L,
                                      (sB < n_slices) ? u_in + sB * L : nullptr, u_out + sA * L,
                                      (sB < n_slices) ? u_out + sB * L : nullptr, m_steps, h);
  tmem_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) {
    tmem_fence_after();
    tmem_dealloc<LY::NCOL>(tslot);
  }
}


template <int N, int R>
static cudaError_t launch_fine_nr(int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                                  const FineTab& tab, cudaStream_t st) {
  constexpr int T = core_threads<N, R>();
  const int grid = (S + 1) / 2;
  const size_t sm = FineLayout<N, R, T>::bytes;
  cudaError_t e;
#define LAUNCH_FINE(SC, LN)                                                  \
  {                                                                           \
    auto kfn = k_fine<N, R, T, SC, LN>;                                       \
    if ((e = set_smem(kfn, sm)) != cudaSuccess) return e;                     \
    kfn<<<grid, T, sm, st>>>(in, out, S, m, h, tab);                          \
  }
  if (scheme == 0 && !lin) LAUNCH_FINE(0, false)
  else if (scheme == 0 && lin) LAUNCH_FINE(0, true)
  else if (scheme == 1 && !lin) LAUNCH_FINE(1, false)
  else if (scheme == 1 && lin) LAUNCH_FINE(1, true)
  else if (scheme == 2 && !lin) LAUNCH_FINE(2, false)
  else LAUNCH_FINE(2, true)
#undef LAUNCH_FINE
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_fine_n(int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                                 const FineTab& tab, cudaStream_t st) {
  if constexpr (N == 1024 || N == 512) {  // measurement knob: the radix-16 plans (16.4.16, 16.2.16)
    static const char* e = getenv("RSW_FINE_R16");
    if (e && atoi(e) == 1) return launch_fine_nr<N, 16>(scheme, lin, in, out, S, m, h, tab, st);
  }
  return launch_fine_nr<N, fine_radix<N>()>(scheme, lin, in, out, S, m, h, tab, st);
}


cudaError_t launch_fine(int n, int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                        const FineTab& tab, cudaStream_t st) {
#define C(NN) launch_fine_n<NN>(scheme, lin, in, out, S, m, h, tab, st)
  RSW_DISPATCH(n, C)
#undef C
}

}  // namespace rsw
