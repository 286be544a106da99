// rsw_k_misc.cu — standalone N(u) (a1), batched averaged nonlinearity (a3) and the DFMA peak probe.
#include "rsw_blocks.cuh"

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
template <int N, int T>
__global__ void __launch_bounds__(T) k_nonlinear(const double* u_in, double* out, int n_states,
                                                 const FineTab tab) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  constexpr double invN = 1.0 / N;
  extern __shared__ double2 smem[];
  double2* W = smem;
  double2* C = W + 3 * WL<N>::NP;
  const int sA = 2 * blockIdx.x, sB = sA + 1;
  const size_t L = (size_t)3 * NH * 2;
  load_pair_eigen<N, T>(u_in + sA * L, (sB < n_states) ? u_in + sB * L : nullptr, tab.g, C);
  __syncthreads();
  prologue_from<N, T>(W, C, tab.g);
  __syncthreads();
  nl_physical<N, T, radix_for<N>()>(W, tab.tw);
  for (int j = threadIdx.x; j < Kc; j += T) {
    const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
    const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
    double2 nh[3], nn[3];
    get_output<N>(W, full_index(kap, N), (double)kap, invN, nh);
    to_eigen(as, __ldg(tab.g.p + ak), __ldg(tab.g.q + ak), nh, nn);
#pragma unroll
    for (int al = 0; al < 3; ++al) C[al * Kc + j] = nn[al];
  }
  __syncthreads();
  store_pair_prim<N, T>(C, tab.g, out + sA * L, (sB < n_states) ? out + sB * L : nullptr);
}

// ---------------------------------------------------------------------------------------------
// K3: averaged nonlinearity for pairs of independent states (same sample m for both):
//   acc = Σ_{m=1}^{M-1} w_m P+_m N(P-_m c), in ascending m; P±_m = diag(e^{±iατ_m ω}) (eigen).
// ---------------------------------------------------------------------------------------------

template <int N, int T>
__global__ void __launch_bounds__(T) k_avg_states(const double* u_in, double* out, int n_states, int M,
                                                  const AvgTab tab) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  constexpr double invN = 1.0 / N;
  extern __shared__ double2 smem[];
  double2* W = smem;
  double2* C = W + 3 * WL<N>::NP;
  double2* A = C + 3 * Kc;
  const int sA = 2 * blockIdx.x, sB = sA + 1;
  const size_t L = (size_t)3 * NH * 2;
  load_pair_eigen<N, T>(u_in + sA * L, (sB < n_states) ? u_in + sB * L : nullptr, tab.g, C);
  for (int i = threadIdx.x; i < 3 * Kc; i += T) A[i] = make_double2(0.0, 0.0);
  __syncthreads();
  // prologue for m = 1
  for (int m = 1; m <= M - 1; ++m) {
    if (m == 1) {
      for (int j = threadIdx.x; j < Kc; j += T) {
        const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
        const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
        const double2 ph = __ldg(tab.phase + (size_t)m * (K + 1) + ak);  // e^{iωτ_m}
        double2 c[3], u[3];
        c[0] = cmul(C[j], ph);            // α=-1: e^{+iωτ}
        c[1] = C[Kc + j];                 // α=0
        c[2] = cmulc(C[2 * Kc + j], ph);  // α=+1: e^{-iωτ}
        to_prim(as, __ldg(tab.g.p + ak), __ldg(tab.g.q + ak), c, u);
        put_input<N>(W, full_index(kap, N), (double)kap, u);
      }
      zero_tail<N, T>(W);
      __syncthreads();
    }
    nl_physical<N, T, radix_for<N>()>(W, tab.tw);
    const double wm = __ldg(tab.w + m);
    for (int j = threadIdx.x; j < Kc; j += T) {
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
      const int kf = full_index(kap, N);
      const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
      const double p = __ldg(tab.g.p + ak), q = __ldg(tab.g.q + ak);
      double2 nh[3], nn[3];
      get_output<N>(W, kf, (double)kap, invN, nh);
      to_eigen(as, p, q, nh, nn);
      const double2 ph = __ldg(tab.phase + (size_t)m * (K + 1) + ak);
      A[j] = caxpy(wm, cmulc(nn[0], ph), A[j]);               // α=-1: e^{-iωτ}
      A[Kc + j] = caxpy(wm, nn[1], A[Kc + j]);                // α=0
      A[2 * Kc + j] = caxpy(wm, cmul(nn[2], ph), A[2 * Kc + j]);  // α=+1: e^{+iωτ}
      if (m + 1 <= M - 1) {
        const double2 ph2 = __ldg(tab.phase + (size_t)(m + 1) * (K + 1) + ak);
        double2 c[3], u[3];
        c[0] = cmul(C[j], ph2);
        c[1] = C[Kc + j];
        c[2] = cmulc(C[2 * Kc + j], ph2);
        to_prim(as, p, q, c, u);
        put_input<N>(W, kf, (double)kap, u);
      }
    }
    zero_tail<N, T>(W);
    __syncthreads();
  }
  store_pair_prim<N, T>(A, tab.g, out + sA * L, (sB < n_states) ? out + sB * L : nullptr);
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
constexpr size_t nl_smem() { return sizeof(double2) * (3 * WL<N>::NP + 3 * (2 * (N / 3) + 1)); }
template <int N>
constexpr size_t avg_smem() { return sizeof(double2) * (3 * WL<N>::NP + 2 * 3 * (2 * (N / 3) + 1)); }


template <int N>
static cudaError_t launch_nl_n(const double* in, double* out, int S, const FineTab& tab, cudaStream_t st) {
  constexpr int T = threads_for<N>();
  auto kfn = k_nonlinear<N, T>;
  cudaError_t e = set_smem(kfn, nl_smem<N>());
  if (e != cudaSuccess) return e;
  kfn<<<(S + 1) / 2, T, nl_smem<N>(), st>>>(in, out, S, tab);
  return cudaGetLastError();
}


template <int N>
static cudaError_t launch_avg_n(const double* in, double* out, int S, int M, const AvgTab& tab, cudaStream_t st) {
  constexpr int T = threads_for<N>();
  auto kfn = k_avg_states<N, T>;
  cudaError_t e = set_smem(kfn, avg_smem<N>());
  if (e != cudaSuccess) return e;
  kfn<<<(S + 1) / 2, T, avg_smem<N>(), st>>>(in, out, S, M, tab);
  return cudaGetLastError();
}


cudaError_t launch_nonlinear(int n, const double* in, double* out, int S, const FineTab& tab, cudaStream_t st) {
#define C(NN) launch_nl_n<NN>(in, out, S, tab, st)
  RSW_DISPATCH(n, C)
#undef C
}

cudaError_t launch_avg_states(int n, const double* in, double* out, int S, int M, const AvgTab& tab,
                              cudaStream_t st) {
#define C(NN) launch_avg_n<NN>(in, out, S, M, tab, st)
  RSW_DISPATCH(n, C)
#undef C
}

cudaError_t launch_dfma_peak(double* out, int blocks, int iters, cudaStream_t st) {
  k_dfma_peak<<<blocks, 256, 0, st>>>(out, iters);
  return cudaGetLastError();
}

}  // namespace rsw
