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



// k_fine: NPG pair-groups of TG threads per CTA (named barriers 1..NPG, or the whole CTA when
// NPG = 1); group g advances slices 2(NPG b + g), +1.  Shared memory: per group the N-eval buffer W
// (3N) and the v1 copy V (N), then the tables shared by the groups (twiddle bases, ETDRK4 / Strang
// coefficients, geometry).  TMEM: the groups' thread-private state slots interleave (TBLK layout).
#ifndef RSW_FINE_TWT
#define RSW_FINE_TWT 2  // twiddle policy of the n >= 512 transforms (fft_tw_src): TMEM copies of the radix-R passes
#endif

template <int N, int R, int TG, int NPG>
struct FineLayout {  // dynamic shared memory of k_fine (double2 units first, then doubles)
  static constexpr int K = N / 3, KP = K + 1, Kc = 2 * K + 1;
  static constexpr int GS = nl_buf<N, R>();  // per-group stride: the N-eval buffer (padded fields + V)
  static constexpr int TW = NPG * GS, CP = TW + fft_tw_size<N, R>(), D = CP + 6 * KP;
  static constexpr int ND = 9 * KP;  // C0 [6][KP], GA, GP, GQ
  static constexpr size_t bytes = sizeof(double2) * D + sizeof(double) * ND;
  static constexpr int T = NPG * TG, OMAX = (Kc + TG - 1) / TG, BLKS = (T / 32 + 3) / 4;
  static constexpr int TWC = BLKS * OMAX * 36;  // TMEM: state slots, then the twiddle copies (TWT = 2)
  static constexpr int TWT = (TWC + fft_tw_tcols<N, R>() <= 512) ? RSW_FINE_TWT : (RSW_FINE_TWT == 2 ? 1 : RSW_FINE_TWT);
  static constexpr int NCOL = tmem_cols_pow2<TWC + (TWT == 2 ? fft_tw_tcols<N, R>() : 0)>();
  static_assert(BLKS * OMAX * 36 <= 512, "k_fine: TMEM state does not fit");
};

template <int N, int R, int TG, int NPG, int SCHEME, bool LIN>
__global__ void __launch_bounds__(NPG * TG) k_fine(const double* u_in, double* u_out, int n_slices, int m_steps,
                                                   double h, const FineTab tab, const PeerOut po) {
  using LY = FineLayout<N, R, TG, NPG>;
  constexpr int NH = N / 2 + 1;
  extern __shared__ double2 smem[];
  __shared__ uint32_t tslot;
  if ((threadIdx.x >> 5) == 0) tmem_alloc<LY::NCOL>(&tslot);
  const FineSmemTab st_ = stage_fine_tables<N, R, LY::T>(smem + LY::TW, smem + LY::CP,
                                                         reinterpret_cast<double*>(smem + LY::D), tab, threadIdx.x, LY::T);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const int g = (NPG == 1) ? 0 : (int)threadIdx.x / TG;
  if constexpr (LY::TWT == 2) {  // each thread's radix-R twiddles into its TMEM lane
    tw_tmem_fill<N, R, 2>(st_.TW, tslot + LY::TWC + ((uint32_t)(32 * ((threadIdx.x >> 5) & 3)) << 16), (int)threadIdx.x - g * TG);
    tmem_wait_st();
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
  }
  const int sA = 2 * (NPG * blockIdx.x + g), sB = sA + 1;
  const size_t L = (size_t)3 * NH * 2;
  if (sA < n_slices) {
    double2* W = smem + g * LY::GS;
    const double* uA = u_in + sA * L;
    const double* uB = (sB < n_slices) ? u_in + sB * L : nullptr;
    double* oA = u_out + sA * L;
    double* oB = (sB < n_slices) ? u_out + sB * L : nullptr;
    if constexpr (NPG == 1)
      fine_pair_run<N, R, TG, SCHEME, LIN, CtaGroup, true, LY::TWT>(CtaGroup(), W, nullptr, st_, tslot, tab.g, uA, uB, oA,
                                                                    oB, m_steps, h, nullptr, tslot + LY::TWC, &po,
                                                                    (size_t)sA * L);
    else
      fine_pair_run<N, R, TG, SCHEME, LIN, NamedGroup, true, LY::TWT>(NamedGroup{g * TG, 1 + g, TG, 3 + 3 * g}, W, nullptr, st_, tslot,
                                                                      tab.g, uA, uB, oA, oB, m_steps, h, nullptr,
                                                                      tslot + LY::TWC, &po, (size_t)sA * L);
  }
  tmem_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) {
    tmem_fence_after();
    tmem_dealloc<LY::NCOL>(tslot);
  }
#ifdef RSW_PHASE_PROF
  if (threadIdx.x == 0 && blockIdx.x == 0)
    printf("[k_fine n=%d R=%d TG=%d] cycles per N-eval: epilogue+gaps %.0f inverse %.0f products %.0f forward %.0f\n", N, R,
           TG, (double)g_phase[0] / (4.0 * m_steps), (double)g_phase[1] / (4.0 * m_steps), (double)g_phase[2] / (4.0 * m_steps),
           (double)g_phase[3] / (4.0 * m_steps));
#endif
}


template <int N, int R, int NPG, int TMUL = 1>
static cudaError_t launch_fine_nr(int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                                  const FineTab& tab, cudaStream_t st, const PeerOut& po) {
  constexpr int TG = TMUL * core_threads<N, R>();
  const int grid = ((S + 1) / 2 + NPG - 1) / NPG;
  const size_t sm = FineLayout<N, R, TG, NPG>::bytes;
  cudaError_t e;
#define LAUNCH_FINE(SC, LN)                                                  \
  {                                                                           \
    auto kfn = k_fine<N, R, TG, NPG, SC, LN>;                                 \
    if ((e = set_smem(kfn, sm)) != cudaSuccess) return e;                     \
    kfn<<<grid, NPG * TG, sm, st>>>(in, out, S, m, h, tab, po);               \
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
                                 const FineTab& tab, cudaStream_t st, const PeerOut& po) {
  if constexpr (N == 256 || N == 512) {  // measurement knob: RSW_FINE_R = 4 or 16
    static const char* e = getenv("RSW_FINE_R");
    if (e && atoi(e) == 16) return launch_fine_nr<N, 16, 1>(scheme, lin, in, out, S, m, h, tab, st, po);
    if (e && atoi(e) == 4) return launch_fine_nr<N, 4, 1>(scheme, lin, in, out, S, m, h, tab, st, po);
    if (e && atoi(e) == 82) return launch_fine_nr<N, 8, 1, 2>(scheme, lin, in, out, S, m, h, tab, st, po);  // 2x threads
  }
  if constexpr (N >= 64 && N <= 256) {
    // latency regime (at most ~2 pairs per SM, e.g. C3's 256 pairs): twice the threads per pair (the
    // extra warps split the mode loops and fill the schedulers): C3 3.16 -> 2.90 ms; throughput
    // regime keeps 3N/R threads (C3-size 4736 slices: 17.9 vs 22.0 ms)
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        sms = 148;
    }
    if ((S + 1) / 2 <= 2 * sms) return launch_fine_nr<N, fine_radix<N>(), 1, 2>(scheme, lin, in, out, S, m, h, tab, st, po);
  }
  return launch_fine_nr<N, fine_radix<N>(), fine_groups<N>()>(scheme, lin, in, out, S, m, h, tab, st, po);
}


cudaError_t launch_fine(int n, int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                        const FineTab& tab, cudaStream_t st, const PeerOut* po) {
  PeerOut none{};
  const PeerOut& pv = po ? *po : none;
#define C(NN) launch_fine_n<NN>(scheme, lin, in, out, S, m, h, tab, st, pv)
  RSW_DISPATCH(n, C)
#undef C
}

}  // namespace rsw
