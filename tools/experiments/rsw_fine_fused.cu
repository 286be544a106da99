// rsw_fine.cu — K1/K2, the fine propagator (the parfor of Alg.4): ETDRK4 (Cox–Matthews,
// cited P:1168-1169) or Strang (Alg.3, R7), every slice advanced independently, state
// resident on chip for all m steps.
//
// One CTA = one PAIR of slices packed into one complex field (rsw_device.cuh).  Each N(u) is two
// complex FFTs over the 3 fields with the mixed-radix Stockham sequence [RE, RM1, RM2, RE]:
//   forward  F1 (RE, NS=1) -> F2a (RM1, NS=RE) -> F2b (RM2, NS=RE·RM1) -> F3 (RE, NS=N/RE)
//   inverse  I1 (RE, NS=1) -> I2a, I2b -> I3 (RE, NS=N/RE)
// F3 stores, and I1 loads, exactly the index set {j + r N/RE} of butterfly j; so do I3 and F1.  So
// thread j runs, in registers and for all 3 fields,
//   * the SPECTRAL fused pass: F3 -> 1/N, derivative factors, eigenbasis change, the ETDRK4 stage
//     update of its modes k = j + r N/RE (state S0, S1, S2 in shared memory) -> next input -> I1;
//   * the PHYSICAL fused pass: I3 -> pointwise products v1²/2, v1 v2x, h v1 -> F1.
// Per N(u) the work buffer makes 6 shared-memory round trips (spectral, I2a, I2b, physical, F2a,
// F2b) instead of 8 Stockham passes plus separate product and spectral passes.  Thread j owns the same modes for
// the whole launch.
#include "rsw_internal.h"

namespace rsw {

template <int N>
struct FPlan;  // radix sequence [RE, RM1, RM2, RE] (RM = 1: no pass), threads T
template <> struct FPlan<16> { static constexpr int RE = 4, RM1 = 1, RM2 = 1, T = 32; };
template <> struct FPlan<32> { static constexpr int RE = 4, RM1 = 2, RM2 = 1, T = 32; };
template <> struct FPlan<64> { static constexpr int RE = 4, RM1 = 4, RM2 = 1, T = 32; };
template <> struct FPlan<128> { static constexpr int RE = 4, RM1 = 8, RM2 = 1, T = 64; };
template <> struct FPlan<256> { static constexpr int RE = 4, RM1 = 4, RM2 = 4, T = 64; };
template <> struct FPlan<512> { static constexpr int RE = 4, RM1 = 8, RM2 = 4, T = 128; };
template <> struct FPlan<1024> { static constexpr int RE = 4, RM1 = 8, RM2 = 8, T = 256; };

template <int N>
constexpr size_t fine2_smem() {
  return sizeof(double2) * (3 * WL<N>::NP + 3 * 3 * (2 * (N / 3) + 1));
}

// coefficient i of |κ| for eigen-row α: 0 E, 1 E2, 2 Q, 3 f1, 4 f2, 5 f3
struct Coef {
  const double2* cp;
  const double* c0;
  int stride;
  __device__ __forceinline__ double2 mul(int i, int alpha, int ak, double2 x) const {
    return dmul(alpha, __ldg(cp + i * stride + ak), __ldg(c0 + i * stride + ak), x);
  }
};

// MODE: 0 = prologue (input x = S1, then I1); 1 = F3 + stage update + I1; 2 = F3 + stage update
// (last stage of the last step, no next N-eval); 3 = linear-only stage update (N ≡ 0, no FFTs)
template <int N, int SCHEME, int MODE>
__device__ __forceinline__ void spectral_pass(double2* W, double2* S0, double2* S1, double2* S2, const FineTab& tab,
                                              const Coef& cf, int st, bool last_step, double h,
                                              const double2* twe) {
  constexpr int RE = FPlan<N>::RE, NI = N / RE, NP = WL<N>::NP, K = N / 3, Kc = 2 * K + 1;
  constexpr double invN = 1.0 / N;
  const int j = tid_x();
  double2 z[3][RE];
  if (MODE == 1 || MODE == 2) {
    if (j < NI) {
#pragma unroll
      for (int f = 0; f < 3; ++f)
#pragma unroll
        for (int r = 0; r < RE; ++r) z[f][r] = W[f * NP + pad(j + r * NI)];
    }
    __syncthreads();
  }
  if (j < NI) {
    if (MODE == 1 || MODE == 2) {
#pragma unroll
      for (int f = 0; f < 3; ++f) {  // F3: twiddle w^{rj}, DFT_RE (forward)
#pragma unroll
        for (int r = 1; r < RE; ++r) z[f][r] = cmul(z[f][r], __ldg(twe + r * j));
        dftR<RE, -1>(z[f]);
      }
    }
#pragma unroll
    for (int r = 0; r < RE; ++r) {
      const int k = j + r * NI;
      const int kap = (k <= N / 2) ? k : k - N;
      const int ak = kap < 0 ? -kap : kap;
      if (ak <= K && k != N / 2) {
        const int jj = kap >= 0 ? kap : kap + Kc;
        const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
        const double p = __ldg(tab.g.p + ak), q = __ldg(tab.g.q + ak);
        double2 nn[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
        if (MODE == 1 || MODE == 2) {
          const double2 Q0 = cscale(z[0][r], invN), Q1 = cscale(z[1][r], invN), Q2 = cscale(z[2][r], invN);
          double2 nh[3];
          nh[0] = cmulmi(cscale(Q0, (double)kap));  // -(1/2)∂x(v1²)·2/2: -iκ DFT(v1²/2)
          nh[1] = make_double2(-Q1.x, -Q1.y);       // -v1 ∂x v2
          nh[2] = cmulmi(cscale(Q2, (double)kap));  // -∂x(h v1)
          to_eigen(as, p, q, nh, nn);
        }
        double2 x[3];
#pragma unroll
        for (int al = 0; al < 3; ++al) {
          const int alpha = al - 1, e = al * Kc + jj;
          if (MODE == 0) {
            if (SCHEME == 1) S1[e] = cf.mul(1, alpha, ak, S1[e]);  // Strang: v = E2 c
            x[al] = S1[e];
          } else if (SCHEME == 0) {
            if (st == 0) {
              const double2 c = S1[e];
              const double2 e2c = cf.mul(1, alpha, ak, c);
              const double2 qn = cf.mul(2, alpha, ak, nn[al]);
              const double2 a = cadd(e2c, qn);
              S0[e] = e2c;
              S1[e] = cadd(cf.mul(0, alpha, ak, c), cf.mul(3, alpha, ak, nn[al]));
              S2[e] = csub(cf.mul(1, alpha, ak, a), qn);
              x[al] = a;
            } else if (st == 1) {
              x[al] = cadd(S0[e], cf.mul(2, alpha, ak, nn[al]));
              S1[e] = cadd(S1[e], cf.mul(4, alpha, ak, nn[al]));
            } else if (st == 2) {
              x[al] = cadd(S2[e], cscale(cf.mul(2, alpha, ak, nn[al]), 2.0));
              S1[e] = cadd(S1[e], cf.mul(4, alpha, ak, nn[al]));
            } else {
              const double2 c = cadd(S1[e], cf.mul(5, alpha, ak, nn[al]));
              S1[e] = c;
              x[al] = c;
            }
          } else {
            if (st == 0) {
              x[al] = caxpy(0.5 * h, nn[al], S1[e]);  // m = v + (h/2) N(v)
            } else {
              const double2 w = caxpy(h, nn[al], S1[e]);                 // w = v + h N(m)
              const double2 c = cf.mul(1, alpha, ak, w);                  // c+ = E2 w
              const double2 v = last_step ? c : cf.mul(1, alpha, ak, c);  // next v = E2 c+
              S1[e] = v;
              x[al] = v;
            }
          }
        }
        if (MODE == 0 || MODE == 1) {
          double2 u[3];
          to_prim(as, p, q, x, u);
          z[0][r] = u[0];
          z[1][r] = cmuli(cscale(u[1], (double)kap));  // iκ v̂2 -> ∂x v2 after the synthesis
          z[2][r] = u[2];
        }
      } else if (MODE == 0 || MODE == 1) {
        z[0][r] = z[1][r] = z[2][r] = make_double2(0.0, 0.0);  // 2/3 rule (R10)
      }
      asm volatile("" ::: "memory");  // keep the per-mode loads from being hoisted (register pressure)
    }
    if (MODE == 0 || MODE == 1) {
#pragma unroll
      for (int f = 0; f < 3; ++f) {  // I1: DFT_RE (inverse), NS = 1, stride-RE store
        dftR<RE, +1>(z[f]);
#pragma unroll
        for (int r = 0; r < RE; ++r) W[f * NP + pad(j * RE + r)] = z[f][r];
      }
    }
  }
  __syncthreads();
}

// I3 -> products -> F1 for the 3 fields of butterfly j
template <int N>
__device__ __forceinline__ void physical_pass(double2* W, const double2* twe) {
  constexpr int RE = FPlan<N>::RE, NI = N / RE, NP = WL<N>::NP;
  const int j = tid_x();
  double2 z[3][RE];
  if (j < NI) {
#pragma unroll
    for (int f = 0; f < 3; ++f)
#pragma unroll
      for (int r = 0; r < RE; ++r) z[f][r] = W[f * NP + pad(j + r * NI)];
  }
  __syncthreads();
  if (j < NI) {
#pragma unroll
    for (int f = 0; f < 3; ++f) {  // I3: twiddle conj(w^{rj}), DFT_RE (inverse) -> grid values
#pragma unroll
      for (int r = 1; r < RE; ++r) z[f][r] = cmulc(z[f][r], __ldg(twe + r * j));
      dftR<RE, +1>(z[f]);
    }
#pragma unroll
    for (int r = 0; r < RE; ++r) {  // products on the real / imaginary lanes (the two slices)
      const double2 v1 = z[0][r], v2x = z[1][r], hh = z[2][r];
      z[0][r] = make_double2(0.5 * v1.x * v1.x, 0.5 * v1.y * v1.y);
      z[1][r] = make_double2(v1.x * v2x.x, v1.y * v2x.y);
      z[2][r] = make_double2(hh.x * v1.x, hh.y * v1.y);
    }
#pragma unroll
    for (int f = 0; f < 3; ++f) {  // F1: DFT_RE (forward), NS = 1
      dftR<RE, -1>(z[f]);
#pragma unroll
      for (int r = 0; r < RE; ++r) W[f * NP + pad(j * RE + r)] = z[f][r];
    }
  }
  __syncthreads();
}

template <int N, int SCHEME, bool LIN>
__global__ void __launch_bounds__(FPlan<N>::T, 1) k_fine2(const double* u_in, double* u_out, int n_slices, int m_steps,
                                                       double h, const FineTab tab) {
  constexpr int T = FPlan<N>::T, RE = FPlan<N>::RE, RM1 = FPlan<N>::RM1, RM2 = FPlan<N>::RM2, NI = N / RE;
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  extern __shared__ double2 smem[];
  double2* W = smem;
  double2* S0 = W + 3 * WL<N>::NP;
  double2* S1 = S0 + 3 * Kc;
  double2* S2 = S1 + 3 * Kc;
  const int sA = 2 * blockIdx.x, sB = sA + 1;
  const size_t L = (size_t)3 * NH * 2;
  load_pair_eigen<N, T>(u_in + sA * L, (sB < n_slices) ? u_in + sB * L : nullptr, tab.g, S1);
  const double2* twe = tab.tw;  // edge-pass twiddles w^{rj} (L1-resident table)
  const Coef cf{tab.cp, tab.c0, K + 1};
  __syncthreads();

  if (LIN) {
    spectral_pass<N, SCHEME, 0>(W, S0, S1, S2, tab, cf, 0, false, h, twe);  // Strang: v = E2 c
    for (int step = 0; step < m_steps; ++step) {
      const int nst = (SCHEME == 0) ? 4 : 2;
      for (int st = 0; st < nst; ++st)
        spectral_pass<N, SCHEME, 3>(W, S0, S1, S2, tab, cf, st, step == m_steps - 1, h, twe);
    }
  } else {
    spectral_pass<N, SCHEME, 0>(W, S0, S1, S2, tab, cf, 0, false, h, twe);
    const int nst = (SCHEME == 0) ? 4 : 2;
    for (int step = 0; step < m_steps; ++step) {
      const bool last_step = (step == m_steps - 1);
      for (int st = 0; st < nst; ++st) {
        if constexpr (RM1 > 1) stockham_pass<N, T, RM1, RE, +1>(W, tab.tw);        // I2a
        if constexpr (RM2 > 1) stockham_pass<N, T, RM2, RE * RM1, +1>(W, tab.tw);  // I2b
        physical_pass<N>(W, twe);                                                  // I3, products, F1
        if constexpr (RM1 > 1) stockham_pass<N, T, RM1, RE, -1>(W, tab.tw);        // F2a
        if constexpr (RM2 > 1) stockham_pass<N, T, RM2, RE * RM1, -1>(W, tab.tw);  // F2b
        if (last_step && st == nst - 1)
          spectral_pass<N, SCHEME, 2>(W, S0, S1, S2, tab, cf, st, last_step, h, twe);
        else
          spectral_pass<N, SCHEME, 1>(W, S0, S1, S2, tab, cf, st, last_step, h, twe);
      }
    }
  }
  store_pair_prim<N, T>(S1, tab.g, u_out + sA * L, (sB < n_slices) ? u_out + sB * L : nullptr);
}

template <typename KernelT>
static cudaError_t set_smem2(KernelT k, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int N>
static cudaError_t launch_fine2_n(int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                                  const FineTab& tab, cudaStream_t st) {
  constexpr int T = FPlan<N>::T;
  const int grid = (S + 1) / 2;
  const size_t sm = fine2_smem<N>();
  cudaError_t e;
#define LAUNCH_FINE2(SC, LN)                                   \
  {                                                             \
    auto kfn = k_fine2<N, SC, LN>;                              \
    if ((e = set_smem2(kfn, sm)) != cudaSuccess) return e;      \
    kfn<<<grid, T, sm, st>>>(in, out, S, m, h, tab);            \
  }
  if (scheme == 0 && !lin) LAUNCH_FINE2(0, false)
  else if (scheme == 0 && lin) LAUNCH_FINE2(0, true)
  else if (scheme == 1 && !lin) LAUNCH_FINE2(1, false)
  else LAUNCH_FINE2(1, true)
#undef LAUNCH_FINE2
  return cudaGetLastError();
}

cudaError_t launch_fine(int n, int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                        const FineTab& tab, cudaStream_t st) {
  switch (n) {
    case 16: return launch_fine2_n<16>(scheme, lin, in, out, S, m, h, tab, st);
    case 32: return launch_fine2_n<32>(scheme, lin, in, out, S, m, h, tab, st);
    case 64: return launch_fine2_n<64>(scheme, lin, in, out, S, m, h, tab, st);
    case 128: return launch_fine2_n<128>(scheme, lin, in, out, S, m, h, tab, st);
    case 256: return launch_fine2_n<256>(scheme, lin, in, out, S, m, h, tab, st);
    case 512: return launch_fine2_n<512>(scheme, lin, in, out, S, m, h, tab, st);
    case 1024: return launch_fine2_n<1024>(scheme, lin, in, out, S, m, h, tab, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rsw
