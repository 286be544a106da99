// rsw_k_misc.cu — standalone N(u) (a1), batched averaged nonlinearity (a3) and the DFMA peak probe.
#include "rsw_blocks.cuh"

#include <algorithm>

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

// ---------------------------------------------------------------------------------------------
// K0: standalone N(u) for pairs of states (parity tests of step a1)
// ---------------------------------------------------------------------------------------------
// per-CTA staging of the geometry (a, p, q per |κ|) and the packed twiddles of nl_core
template <int N, int R, int T>
__device__ __forceinline__ void stage_geom_tw(const ModeGeom& g, const double2* __restrict__ tw, double2* TW,
                                              double* GA, double* GP, double* GQ) {
  fill_packed_twiddles<N, R, T>(TW, tw);
  for (int k = threadIdx.x; k <= N / 3; k += T) {
    GA[k] = __ldg(g.a + k);
    GP[k] = __ldg(g.p + k);
    GQ[k] = __ldg(g.q + k);
  }
}

template <int N, int R, int T>
struct MiscLayout {  // X (nl_core buffer), twiddle bases, C / A [3][Kc], then GA, GP, GQ
  static constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1;
  static constexpr int X = 0, Y = 0, TW = nl_buf<N, R>(), C = TW + fft_tw_size<N, R>(), A = C + 3 * Kc, D = A + 3 * Kc;
  static constexpr size_t bytes = sizeof(double2) * D + sizeof(double) * 3 * KP;
};

// ---------------------------------------------------------------------------------------------
// K0: standalone N(u) for pairs of states (parity tests of step a1), register FFT core
// ---------------------------------------------------------------------------------------------
template <int N, int R, int T>
__global__ void __launch_bounds__(T) k_nonlinear(const double* u_in, double* out, int n_states,
                                                 const FineTab tab) {
  using LY = MiscLayout<N, R, T>;
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1, KP = K + 1;
  constexpr double invN = 1.0 / N;
  extern __shared__ double2 smem[];
  double2* X = smem + LY::X;
  double2* C = smem + LY::C;
  double* GA = reinterpret_cast<double*>(smem + LY::D);
  double* GP = GA + KP;
  double* GQ = GP + KP;
  stage_geom_tw<N, R, T>(tab.g, tab.tw, smem + LY::TW, GA, GP, GQ);
  const int sA = 2 * blockIdx.x, sB = sA + 1;
  const size_t L = (size_t)3 * NH * 2;
  load_pair_eigen<N, T>(u_in + sA * L, (sB < n_states) ? u_in + sB * L : nullptr, tab.g, C);
  __syncthreads();
  for (int j = threadIdx.x; j < Kc; j += T) {
    const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
    double2 c[3], u[3];
#pragma unroll
    for (int al = 0; al < 3; ++al) c[al] = C[al * Kc + j];
    to_prim(kap < 0 ? -GA[ak] : GA[ak], GP[ak], GQ[ak], c, u);
    put_input_z<N, R>(X, full_index(kap, N), (double)kap, u);
  }
  __syncthreads();
  nl_core<N, R, T>(X, smem + LY::Y, smem + LY::TW);
  for (int j = threadIdx.x; j < Kc; j += T) {
    const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
    double2 nh[3], nn[3];
    get_output_z<N, R>(X, full_index(kap, N), (double)kap, invN, nh);
    to_eigen(kap < 0 ? -GA[ak] : GA[ak], GP[ak], GQ[ak], nh, nn);
#pragma unroll
    for (int al = 0; al < 3; ++al) C[al * Kc + j] = nn[al];
  }
  __syncthreads();
  store_pair_prim<N, T>(C, tab.g, out + sA * L, (sB < n_states) ? out + sB * L : nullptr);
}

// ---------------------------------------------------------------------------------------------
// K3: averaged nonlinearity for pairs of independent states (same sample m for both), register
// FFT core; ascending m:  acc = Σ_{m=1}^{M-1} w_m P+_m N(P-_m c),  P±_m = diag(e^{±iατ_m ω}) (eigen).
// Each thread owns the modes j = t + o T for every sample; their state c and accumulator acc live
// in the thread's private TMEM slots (columns o*24 + {c: 0..11, acc: 12..23}, lane quarter = warp
// mod 4, column block = warp / 4), which takes their read-modify-write traffic off the shared-memory
// pipe (the binding resource: ncu 81% of peak wavefronts with them in smem).  The next sample's
// phases are loaded into registers before the FFT so their L2 latency hides behind it.
// ---------------------------------------------------------------------------------------------
#ifndef RSW_AVG_MINB
#define RSW_AVG_MINB 1
#endif
#ifndef RSW_AVG_TWT
#define RSW_AVG_TWT 2  // twiddle policy of the n >= 512 transforms (fft_tw_src): TMEM copies of the radix-R passes
#endif
template <int N, int T, int R>
struct AvgTmem {
  static constexpr int Kc = 2 * (N / 3) + 1, OMAX = (Kc + T - 1) / T, BLKS = (T / 32 + 3) / 4;
  static constexpr int TWC = BLKS * OMAX * 24;  // state / accumulator slots, then the twiddle copies
  static constexpr int TWT = (TWC + fft_tw_tcols<N, R>() <= 512) ? RSW_AVG_TWT : (RSW_AVG_TWT == 2 ? 1 : RSW_AVG_TWT);
  static constexpr int NCOL = tmem_cols_pow2<TWC + (TWT == 2 ? fft_tw_tcols<N, R>() : 0)>();
  static_assert(BLKS * OMAX * 24 <= 512, "k_avg_states: TMEM slots do not fit");
};

template <int N, int R, int T>
struct AvgLayout {  // X (nl_core buffer; also stages C in and acc out), twiddle bases, then GA, GP, GQ
  static constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1;
  static_assert(3 * Kc <= nl_buf<N, R>(), "AvgLayout: staging does not fit in X");
  static constexpr int X = 0, TW = nl_buf<N, R>(), D = TW + fft_tw_size<N, R>();
  static constexpr size_t bytes = sizeof(double2) * D + sizeof(double) * 3 * KP;
};

template <int N, int R, int T>
__global__ void __launch_bounds__(T, RSW_AVG_MINB) k_avg_states(const double* u_in, double* out, int n_states, int M,
                                                  const AvgTab tab) {
  using LY = AvgLayout<N, R, T>;
  using TM = AvgTmem<N, T, R>;
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1, KP = K + 1, OMAX = TM::OMAX;
  extern __shared__ double2 smem[];
  __shared__ uint32_t tslot;
  double2* X = smem + LY::X;
  double2* C = X;  // staging of the eigen state, then of the accumulator
  double* GA = reinterpret_cast<double*>(smem + LY::D);
  double* GP = GA + KP;
  double* GQ = GP + KP;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<TM::NCOL>(&tslot);
  stage_geom_tw<N, R, T>(tab.g, tab.tw, smem + LY::TW, GA, GP, GQ);
  const int sA = 2 * blockIdx.x, sB = sA + 1;
  const size_t L = (size_t)3 * NH * 2;
  load_pair_eigen<N, T>(u_in + sA * L, (sB < n_states) ? u_in + sB * L : nullptr, tab.g, C);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t twt = tslot + TM::TWC + ((uint32_t)(32 * (warp & 3)) << 16);
  if constexpr (TM::TWT == 2) {  // each thread's radix-R twiddles into its TMEM lane (the table is staged above)
    tw_tmem_fill<N, R, 2>(smem + LY::TW, twt, (int)threadIdx.x);
    tmem_wait_st();
  }
  const uint32_t tb = tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * OMAX * 24);
  double2 ph[OMAX];
  {
    double2 cc[OMAX][3];
#pragma unroll
    for (int o = 0; o < OMAX; ++o) {
      const int j = threadIdx.x + o * T;
#pragma unroll
      for (int al = 0; al < 3; ++al) cc[o][al] = (j < Kc) ? C[al * Kc + j] : make_double2(0.0, 0.0);
    }
    __syncthreads();  // C read before X receives the first N-eval input
    const double2 z[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#pragma unroll
    for (int o = 0; o < OMAX; ++o) {  // prologue for m = 1
      const int j = threadIdx.x + o * T;
      tmem_st3(tb + o * 24, cc[o]);
      tmem_st3(tb + o * 24 + 12, z);
      if (j < Kc) {
        const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
        ph[o] = __ldg(tab.phase + (size_t)1 * KP + ak);  // e^{iωτ_1}
        double2 c[3];
        c[0] = cmul(cc[o][0], ph[o]);   // α=-1: e^{+iωτ}
        c[1] = cc[o][1];                // α=0
        c[2] = cmulc(cc[o][2], ph[o]);  // α=+1: e^{-iωτ}
        put_input_eigen<N, R>(X, full_index(kap, N), (double)kap, kap < 0 ? -GA[ak] : GA[ak], GP[ak], GQ[ak], c);
      }
    }
    tmem_wait_st();
  }
  __syncthreads();
  for (int m = 1; m <= M - 1; ++m) {
    double2 phn[OMAX];  // next sample's phases, in flight during the FFT
#pragma unroll
    for (int o = 0; o < OMAX; ++o) {
      const int j = threadIdx.x + o * T;
      const int kap = kappa_of(j < Kc ? j : 0, K), ak = kap < 0 ? -kap : kap;
      phn[o] = (j < Kc && m + 1 <= M - 1) ? __ldg(tab.phase + (size_t)(m + 1) * KP + ak) : make_double2(1.0, 0.0);
    }
    nl_core<N, R, T, CtaGroup, TM::TWT>(X, nullptr, smem + LY::TW, CtaGroup(), twt);
    const double wm = __ldg(tab.w + m);
#pragma unroll
    for (int o = 0; o < OMAX; ++o) {
      const int j = threadIdx.x + o * T;
      double2 cc[3], acc[3];
      tmem_ld3(tb + o * 24, cc);
      tmem_ld3(tb + o * 24 + 12, acc);
      if (j < Kc) {
        const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
        const int kf = full_index(kap, N);
        const double as = kap < 0 ? -GA[ak] : GA[ak];
        const double p = GP[ak], q = GQ[ak];
        double2 nn[3];
        get_output_eigen<N, R>(X, kf, (double)kap, as, p, q, nn);
        acc[0] = caxpy(wm, cmulc(nn[0], ph[o]), acc[0]);  // α=-1: e^{-iωτ}
        acc[1] = caxpy(wm, nn[1], acc[1]);                // α=0
        acc[2] = caxpy(wm, cmul(nn[2], ph[o]), acc[2]);   // α=+1: e^{+iωτ}
        if (m + 1 <= M - 1) {
          double2 c[3];
          c[0] = cmul(cc[0], phn[o]);
          c[1] = cc[1];
          c[2] = cmulc(cc[2], phn[o]);
          put_input_eigen<N, R>(X, kf, (double)kap, as, p, q, c);
        }
      }
      tmem_st3(tb + o * 24 + 12, acc);
      ph[o] = phn[o];
    }
    tmem_wait_st();
    __syncthreads();
  }
  // accumulator -> C[α][j] staging in X (all N-eval reads are done), then store
#pragma unroll
  for (int o = 0; o < OMAX; ++o) {
    const int j = threadIdx.x + o * T;
    double2 acc[3];
    tmem_ld3(tb + o * 24 + 12, acc);
    if (j < Kc) {
#pragma unroll
      for (int al = 0; al < 3; ++al) C[al * Kc + j] = acc[al];
    }
  }
  tmem_fence_before();
  __syncthreads();
  store_pair_prim<N, T>(C, tab.g, out + sA * L, (sB < n_states) ? out + sB * L : nullptr);
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc<TM::NCOL>(tslot);
  }
}



__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
  double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1234.5) out[0] = s;  // keep the chains alive
}


template <int N>
static cudaError_t launch_nl_n(const double* in, double* out, int S, const FineTab& tab, cudaStream_t st) {
  constexpr int R = fine_radix<N>(), T = core_threads<N, R>();
  auto kfn = k_nonlinear<N, R, T>;
  constexpr size_t sm = MiscLayout<N, R, T>::bytes;
  cudaError_t e = set_smem(kfn, sm);
  if (e != cudaSuccess) return e;
  kfn<<<(S + 1) / 2, T, sm, st>>>(in, out, S, tab);
  return cudaGetLastError();
}

#ifndef RSW_AVG_R512
#define RSW_AVG_R512 8  // radix of the batched N-bar at n = 512 (measurement knob)
#endif
template <int N>
static cudaError_t launch_avg_n(const double* in, double* out, int S, int M, const AvgTab& tab, cudaStream_t st) {
  constexpr int R = (N == 512) ? RSW_AVG_R512 : fine_radix<N>(), T = core_threads<N, R>();
  auto kfn = k_avg_states<N, R, T>;
  constexpr size_t sm = AvgLayout<N, R, T>::bytes;
  cudaError_t e = set_smem(kfn, sm);
  if (e != cudaSuccess) return e;
  kfn<<<(S + 1) / 2, T, sm, st>>>(in, out, S, M, tab);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Batched N̄ in triad form (P:1113-1118 with Alg.1's quadrature in the coefficients): a CTA
// takes B states, stages their eigen coordinates in the rotated frame (c'^α = c^α e^{-iαωτ_c}) in shared
// memory, and computes N̄_κ, κ = 0..K, for all of them.  A warp works on one κ at a time: lane
// (s, r) = (lane / RG, lane % RG) accumulates state s over the rows i ≡ r (mod RG) in ascending order
// (each coefficient load serves the warp's B states — RG distinct addresses per load, consecutive rows),
// a fixed xor tree over the RG lanes of a state sums them.  The coefficients (6.3 MB at n = 512) stream
// from L2; the per-state work is 60 DP instructions per (κ, κ1) row instead of M - 1 pseudo-spectral
// N-evals (C4: 4.7 vs 21.9 Mflop per state).
// ---------------------------------------------------------------------------------------------
#ifndef RSW_AVG_TRIAD_ASYNC
#define RSW_AVG_TRIAD_ASYNC 0  // 1: coefficients staged per warp with cp.async, TRIAD_STG chunks in flight (C4 2.11 ms vs 1.56 ms for the register prefetch: one row per lane per chunk costs more in waits and copies than it hides)
#endif
constexpr int TRIAD_STG = 4;  // chunk buffers per warp (TRIAD_STG - 1 chunks in flight)
template <int N, int B, int T = 256, int SG = 1>
struct AvgTriadLayout {  // Y[SG B][3][Kc] rotated eigen states, the frame rotation e^{iω_k τ_c}, per-warp chunk buffers
  static constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1, RG = 32 / B;
  static constexpr int Y = 0, RPH = Y + SG * B * 3 * Kc, WB = RPH + KP;
  static constexpr int WCH = 18 * RG / 2;  // double2 per chunk: 18 coefficients x RG rows
  static constexpr int D = WB + (RSW_AVG_TRIAD_ASYNC ? (T / 32) * TRIAD_STG * WCH : 0);
  static constexpr size_t bytes = sizeof(double2) * D;
};
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(sdst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NW>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(NW) : "memory"); }

#ifndef RSW_AVG_TRIAD_MINB
#define RSW_AVG_TRIAD_MINB 2  // two CTAs per SM (registers 162 -> 108): C4 1.83 -> 1.56 ms; 3 (80 registers) 4.2 ms
#endif
// SG state groups per CTA (RSW_AVG_TRIAD_SG): warp w serves group w / (T / 32 / SG); the groups walk the
// same κ sequence in step, so a coefficient row fetched from L2 by one group's warp is read by the
// others' from L1.
template <int N, int B, int T, int SG>
__global__ void __launch_bounds__(T, (RSW_AVG_TRIAD_MINB / SG > 0 ? RSW_AVG_TRIAD_MINB / SG : 1))
    k_avg_triad(const double* __restrict__ u_in, double* __restrict__ out, int n_states, const AvgTab tab) {
  using LY = AvgTriadLayout<N, B, T, SG>;
  constexpr int NWG = T / 32 / SG;  // warps per state group
  static_assert(NWG * SG * 32 == T, "k_avg_triad: T / 32 warps split evenly over SG state groups");
  constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1, NH = N / 2 + 1, RG = 32 / B;
  static_assert(B * RG == 32, "k_avg_triad: B states x RG row groups per warp");
  extern __shared__ double2 smem[];
  double2* Y = smem + LY::Y;
  double2* RPH = smem + LY::RPH;
  const int s0 = blockIdx.x * B * SG;
  for (int k = threadIdx.x; k <= K; k += T) RPH[k] = __ldg(tab.triad_ph + k);
  __syncthreads();
  // stage: primitive half spectra -> eigen coordinates of both signs of κ -> rotated frame
  for (int t = threadIdx.x; t < SG * B * Kc; t += T) {
    const int s = t / Kc, j = t - s * Kc, kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
    double2 c[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    if (s0 + s < n_states) {
      const double2* U = reinterpret_cast<const double2*>(u_in) + (size_t)(s0 + s) * 3 * NH;
      double2 z[3];
#pragma unroll
      for (int f = 0; f < 3; ++f) z[f] = kap < 0 ? cconj(__ldg(U + f * NH + ak)) : __ldg(U + f * NH + ak);
      const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
      to_eigen(as, __ldg(tab.g.p + ak), __ldg(tab.g.q + ak), z, c);
      const double2 r = RPH[ak];
      c[0] = cmul(c[0], r);
      c[2] = cmulc(c[2], r);
    }
#pragma unroll
    for (int al = 0; al < 3; ++al) Y[(s * 3 + al) * Kc + j] = c[al];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, sg = (int)(threadIdx.x >> 5) / NWG, sl = sg * B + lane / RG, r = lane % RG;
  const double2* Ys = Y + sl * 3 * Kc;
  for (int kap = (int)(threadIdx.x >> 5) % NWG; kap <= K; kap += NWG) {
    const int nk = triad_nk(kap, K);
    const double* Wb = tab.triad + (size_t)TRIAD_E * triad_rows_before(kap, K);
    double2 acc[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#if RSW_AVG_TRIAD_ASYNC
    // chunks of RG rows (row i = RG c + r): the warp copies chunk c + STG - 1 (18 RG doubles, 8-byte
    // cp.async: the rows of an entry are contiguous in the table but not 16-byte aligned) while it
    // computes chunk c from shared memory (layout [e][RG]: lane (s, r) reads entry e of its row)
    double* wbuf = reinterpret_cast<double*>(smem + LY::WB) + (size_t)(threadIdx.x >> 5) * TRIAD_STG * 18 * RG;
    const int nch = (nk + RG - 1) / RG;
    auto issue = [&](int c) {
      if (c < nch) {
        double* dst = wbuf + (size_t)(c % TRIAD_STG) * 18 * RG;
        for (int q = lane; q < 18 * RG; q += 32) {
          const int e = q / RG, rr = q % RG, i = c * RG + rr;
          if (i < nk) cp_async8(dst + q, Wb + (size_t)e * nk + i);
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int c = 0; c < TRIAD_STG - 1; ++c) issue(c);
    for (int c = 0; c < nch; ++c) {
      cp_async_wait<TRIAD_STG - 2>();
      __syncwarp();
      const int i = c * RG + r;
      if (i < nk) {
        const double* wc = wbuf + (size_t)(c % TRIAD_STG) * 18 * RG;
        double wv[18];
#pragma unroll
        for (int e = 0; e < 18; ++e) wv[e] = wc[e * RG + r];
        const int k1 = kap - K + i, k2 = K - i;
        const int j1 = k1 >= 0 ? k1 : k1 + Kc, j2 = k2 >= 0 ? k2 : k2 + Kc;
        const double2 am = Ys[j1], ap = Ys[2 * Kc + j1];
        double2 pr[6];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const double2 yb = Ys[b * Kc + j2];
          pr[b] = make_double2(fma(am.x, yb.x, -am.y * yb.y), fma(am.x, yb.y, am.y * yb.x));
          pr[3 + b] = make_double2(fma(ap.x, yb.x, -ap.y * yb.y), fma(ap.x, yb.y, ap.y * yb.x));
        }
#pragma unroll
        for (int g = 0; g < 3; ++g) {
#pragma unroll
          for (int ab2 = 0; ab2 < 6; ++ab2) {
            const double w = wv[g * 6 + ab2];
            if ((g == 1) == (ab2 % 3 == 1)) {
              acc[g].x = fma(w, pr[ab2].x, acc[g].x);
              acc[g].y = fma(w, pr[ab2].y, acc[g].y);
            } else {
              acc[g].x = fma(-w, pr[ab2].y, acc[g].x);
              acc[g].y = fma(w, pr[ab2].x, acc[g].y);
            }
          }
        }
      }
      __syncwarp();  // every lane is done with chunk c's buffer before it is refilled
      issue(c + TRIAD_STG - 1);
    }
    cp_async_wait<0>();
#else
    // the next row's coefficients (L2) are in flight while this row is computed
    double wn[18];
    if (r < nk)
#pragma unroll
      for (int e = 0; e < 18; ++e) wn[e] = __ldg(Wb + (size_t)e * nk + r);
    for (int i = r; i < nk; i += RG) {
      double wv[18];
#pragma unroll
      for (int e = 0; e < 18; ++e) wv[e] = wn[e];
      if (i + RG < nk)
#pragma unroll
        for (int e = 0; e < 18; ++e) wn[e] = __ldg(Wb + (size_t)e * nk + i + RG);
      const int k1 = kap - K + i, k2 = K - i;
      const int j1 = k1 >= 0 ? k1 : k1 + Kc, j2 = k2 >= 0 ? k2 : k2 + Kc;
      const double2 am = Ys[j1], ap = Ys[2 * Kc + j1];
      double2 pr[6];
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const double2 yb = Ys[b * Kc + j2];
        pr[b] = make_double2(fma(am.x, yb.x, -am.y * yb.y), fma(am.x, yb.y, am.y * yb.x));
        pr[3 + b] = make_double2(fma(ap.x, yb.x, -ap.y * yb.y), fma(ap.x, yb.y, ap.y * yb.x));
      }
#pragma unroll
      for (int g = 0; g < 3; ++g) {
#pragma unroll
        for (int ab2 = 0; ab2 < 6; ++ab2) {
          const double w = wv[g * 6 + ab2];
          if ((g == 1) == (ab2 % 3 == 1)) {
            acc[g].x = fma(w, pr[ab2].x, acc[g].x);
            acc[g].y = fma(w, pr[ab2].y, acc[g].y);
          } else {
            acc[g].x = fma(-w, pr[ab2].y, acc[g].x);
            acc[g].y = fma(w, pr[ab2].x, acc[g].y);
          }
        }
      }
    }
#endif
#pragma unroll
    for (int g = 0; g < 3; ++g)
      for (int m = RG / 2; m > 0; m >>= 1) {
        acc[g].x += __shfl_xor_sync(0xffffffffu, acc[g].x, m);
        acc[g].y += __shfl_xor_sync(0xffffffffu, acc[g].y, m);
      }
    if (r == 0 && s0 + sl < n_states) {  // back from the rotated frame (× e^{iγωτ_c}), to the primitive spectrum
      const double2 ph = RPH[kap];
      const double2 c[3] = {cmulc(acc[0], ph), acc[1], cmul(acc[2], ph)};
      double2 u[3];
      to_prim(__ldg(tab.g.a + kap), __ldg(tab.g.p + kap), __ldg(tab.g.q + kap), c, u);
      if (kap == 0) u[0].y = u[1].y = u[2].y = 0.0;
      double2* O = reinterpret_cast<double2*>(out) + (size_t)(s0 + sl) * 3 * NH;
#pragma unroll
      for (int f = 0; f < 3; ++f) O[f * NH + kap] = u[f];
    }
  }
  // modes K < k <= N/2 are zero
  for (int t = threadIdx.x; t < SG * B * 3 * (NH - KP); t += T) {
    const int s = t / (3 * (NH - KP)), q = t - s * 3 * (NH - KP), f = q / (NH - KP), k = KP + q % (NH - KP);
    if (s0 + s < n_states) reinterpret_cast<double2*>(out)[(size_t)(s0 + s) * 3 * NH + f * NH + k] = make_double2(0.0, 0.0);
  }
}

#ifndef RSW_AVG_TRIAD_SG
#define RSW_AVG_TRIAD_SG 1  // state groups per CTA (each of 256 threads, B states); 2 (one 512-thread CTA per SM, L1 reuse of the rows): C4 1.74 vs 1.56 ms, off
#endif
#ifndef RSW_AVG_TRIAD_B
#define RSW_AVG_TRIAD_B 4  // states per CTA of the batched triad N̄ (x 32/B row groups per warp); C4: 4 -> 3.44 ms, 8 -> 7.90 ms (1 CTA per SM)
#endif
template <int N>
static cudaError_t launch_avg_triad_n(const double* in, double* out, int S, const AvgTab& tab, cudaStream_t st) {
  constexpr int B = RSW_AVG_TRIAD_B, SG = RSW_AVG_TRIAD_SG, T = 256 * SG;
  auto kfn = k_avg_triad<N, B, T, SG>;
  constexpr size_t sm = AvgTriadLayout<N, B, T, SG>::bytes;
  cudaError_t e = set_smem(kfn, sm);
  if (e != cudaSuccess) return e;
  kfn<<<(S + B * SG - 1) / (B * SG), T, sm, st>>>(in, out, S, tab);
  return cudaGetLastError();
}

cudaError_t launch_nonlinear(int n, const double* in, double* out, int S, const FineTab& tab, cudaStream_t st) {
#define C(NN) launch_nl_n<NN>(in, out, S, tab, st)
  RSW_DISPATCH(n, C)
#undef C
}

cudaError_t launch_avg_states(int n, const double* in, double* out, int S, int M, const AvgTab& tab,
                              cudaStream_t st) {
  if (tab.triad) {  // triad form (n <= 512)
    switch (n) {
      case 16: return launch_avg_triad_n<16>(in, out, S, tab, st);
      case 32: return launch_avg_triad_n<32>(in, out, S, tab, st);
      case 64: return launch_avg_triad_n<64>(in, out, S, tab, st);
      case 128: return launch_avg_triad_n<128>(in, out, S, tab, st);
      case 256: return launch_avg_triad_n<256>(in, out, S, tab, st);
      case 512: return launch_avg_triad_n<512>(in, out, S, tab, st);
      default: return cudaErrorInvalidValue;
    }
  }
#define C(NN) launch_avg_n<NN>(in, out, S, M, tab, st)
  RSW_DISPATCH(n, C)
#undef C
}

// Layout check of input states (include/rsw.h STATE LAYOUT; R10, R16): one thread per half-spectrum
// entry, grid-stride; any violation raises a flag (bad[0]: mode k > n/3 non-zero, bad[1]: Im û_0 != 0).
__global__ void k_check_states(const double2* __restrict__ u, long long entries, int nh, int K, unsigned* bad) {
  unsigned hi = 0, im0 = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < entries; i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % nh);
    const double2 v = __ldg(u + i);
    if (k > K && (v.x != 0.0 || v.y != 0.0)) hi = 1;
    if (k == 0 && v.y != 0.0) im0 = 1;
  }
  if (__any_sync(0xffffffffu, hi) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
  if (__any_sync(0xffffffffu, im0) && (threadIdx.x & 31) == 0) atomicOr(bad + 1, 1u);
}

cudaError_t launch_check_states(int n, const double* u, int n_states, unsigned* bad, cudaStream_t st) {
  const int nh = n / 2 + 1;
  const long long entries = (long long)n_states * 3 * nh;
  const int blocks = (int)std::min<long long>((entries + 255) / 256, 148 * 8);
  k_check_states<<<blocks, 256, 0, st>>>(reinterpret_cast<const double2*>(u), entries, nh, n / 3, bad);
  return cudaGetLastError();
}

cudaError_t launch_dfma_peak(double* out, int blocks, int iters, cudaStream_t st) {
  k_dfma_peak<<<blocks, 256, 0, st>>>(out, iters);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// L2 die-homing probe (rsw_internal.h HomedArena).  One CTA per SM (cooperative launch,
// all co-resident).  Block 0 (the master) ping-pongs with every other block in turn — a value and a
// release flag each way, `rounds` round trips — through pages 0 and 1 of chunk 0 (opposite page
// parity): a pair on one die is ~2x faster through the page its die homes, a pair across the dies is
// slow through both, so the faster page tells the die of block x relative to the master and the
// parity the master's die homes.  Then, with the first same-die partner, pages (2r, 2r + 1) of every
// chunk at r = 0 and r = 200 give each chunk's constant and check the parity rule away from bit 0.
// Every spin gives up after ~2^20 polls (result -1), so a non-resident partner cannot hang the GPU.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned probe_ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void probe_st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ bool probe_wait(const unsigned* p, unsigned v) {
  for (int it = 0; it < (1 << 20); ++it)
    if (probe_ld_acq(p) == v) return true;
  return false;
}
// one use of page pg by a (master, partner) pair; sb: a sequence base unique to this use
__device__ long long probe_pingpong(char* pg, bool master, unsigned sb, int rounds) {
  unsigned* f1 = reinterpret_cast<unsigned*>(pg);
  unsigned* f2 = reinterpret_cast<unsigned*>(pg + 256);
  double* d1 = reinterpret_cast<double*>(pg + 128);
  double* d2 = reinterpret_cast<double*>(pg + 384);
  if (master) {
    if (!probe_wait(f2, sb)) return -1;
    double acc = 0.0;
    const long long t0 = clock64();
    for (int i = 1; i <= rounds; ++i) {
      *d1 = (double)i;
      probe_st_rel(f1, sb + 2u * i);
      if (!probe_wait(f2, sb + 2u * i + 1u)) return -1;
      acc += __ldcg(d2);
    }
    const long long t = (clock64() - t0) / rounds;
    return acc < 0.0 ? t + 1 : t;
  }
  probe_st_rel(f2, sb);
  for (int i = 1; i <= rounds; ++i) {
    if (!probe_wait(f1, sb + 2u * i)) return -1;
    *d2 = __ldcg(d1) + 1.0;
    probe_st_rel(f2, sb + 2u * i + 1u);
  }
  return 0;
}

__global__ void __launch_bounds__(32) k_die_probe(char* arena, int nch, unsigned* ctl, long long* res, int rounds) {
  extern __shared__ char keep_one_per_sm[];
  if (threadIdx.x != 0) return;
  keep_one_per_sm[0] = 0;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const int b = blockIdx.x, nb = gridDim.x;
  res[b] = smid;
  auto chunk_page = [&](int c, int v, int p) {  // page pairs r = 0, 8, 200 (the last two test bits 4 and 8)
    return arena + ((size_t)c << 21) + ((size_t)(2 * (v == 0 ? 0 : v == 1 ? 8 : 200) + p) << 12);
  };
  if (b == 0) {
    for (int x = 1; x < nb; ++x) {
      probe_st_rel(ctl + x, 1u);
      for (int p = 0; p < 2; ++p)
        res[nb + 2 * x + p] = probe_pingpong(arena + ((size_t)p << 12), true, ((unsigned)x << 12) + 1024u * p, rounds);
    }
    int y = -1;
    for (int x = 1; x < nb && y < 0; ++x) {
      const long long t0 = res[nb + 2 * x], t1 = res[nb + 2 * x + 1];
      if (t0 > 0 && t1 > 0 && 10 * min(t0, t1) < 7 * max(t0, t1)) y = x;
    }
    probe_st_rel(ctl + nb, y < 0 ? 0xffffffffu : (unsigned)y);
    if (y > 0)
      for (int c = 0; c < nch; ++c)
        for (int v = 0; v < 3; ++v)
          for (int p = 0; p < 2; ++p)
            res[3 * nb + 6 * c + 2 * v + p] = probe_pingpong(chunk_page(c, v, p), true, (1u << 28) + ((unsigned)(6 * c + 2 * v + p) << 10), rounds);
    return;
  }
  if (!probe_wait(ctl + b, 1u)) return;
  for (int p = 0; p < 2; ++p) probe_pingpong(arena + ((size_t)p << 12), false, ((unsigned)b << 12) + 1024u * p, rounds);
  unsigned y = 0;
  for (int it = 0; it < (1 << 22) && (y = probe_ld_acq(ctl + nb)) == 0u; ++it) {
  }
  if (y != (unsigned)b) return;
  for (int c = 0; c < nch; ++c)
    for (int v = 0; v < 3; ++v)
      for (int p = 0; p < 2; ++p) probe_pingpong(chunk_page(c, v, p), false, (1u << 28) + ((unsigned)(6 * c + 2 * v + p) << 10), rounds);
}

cudaError_t launch_die_probe(char* arena, int nch, unsigned* ctl, long long* res, int nb, int rounds, cudaStream_t st) {
  const size_t smem = 120 * 1024;  // one CTA per SM
  cudaError_t e = cudaFuncSetAttribute(k_die_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&arena, &nch, &ctl, &res, &rounds};
  return cudaLaunchCooperativeKernel((const void*)k_die_probe, dim3(nb), dim3(32), args, smem, st);
}

}  // namespace rsw
