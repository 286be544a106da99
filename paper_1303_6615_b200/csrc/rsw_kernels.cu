// rsw_kernels.cu — the hot-path kernels (sm_100a, fp64 CUDA cores; no tensor cores: the path is
// FFT + per-mode diagonal algebra, not a dense contraction).  See DESIGN.md §6 for the roofline of
// each kernel and rsw_device.cuh for the data layout.
#include "rsw_internal.h"
#include "rsw_device.cuh"

#include <cstdlib>

namespace rsw {

// FFT radix and CTA size, T = 3N/R (one radix-R butterfly of each field per thread), chosen from
// measurements on B200: large transforms (n >= 512) are shared-memory-traffic bound,
// so radix 16 (fewest passes) wins for the throughput kernels (C5 fine 5.6 -> 6.3 TFLOP/s, C4 N̄
// 6.5 -> 7.8); at n <= 256 the kernels are latency bound and radix 4 with more threads wins (C3 fine
// 5.4 TFLOP/s vs 4.0 at radix 16; C3 coarse stage 7.5 us vs 14.1).
template <int N>
#ifndef RSW_RADIX_FINE
#define RSW_RADIX_FINE 0
#endif
#ifndef RSW_RADIX_COARSE
#define RSW_RADIX_COARSE 0
#endif
__host__ __device__ constexpr int radix_for() { return RSW_RADIX_FINE ? RSW_RADIX_FINE : (N >= 512 ? 16 : 4); }
template <int N>
__host__ __device__ constexpr int threads_for() { return (3 * N / radix_for<N>()) > 96 ? (3 * N / radix_for<N>()) : 96; }
// register FFT core (nl_core): R values per thread, T = 3N/R threads (>= 32)
template <int N>
__host__ __device__ constexpr int fine_radix() { return N <= 32 ? 4 : N <= 256 ? 8 : 16; }  // palindromic
template <int N, int R>
__host__ __device__ constexpr int core_threads() { return (3 * (N / R) + 31) / 32 * 32; }
static int fine_radix_override() {
  static int r = -1;
  if (r < 0) {
    const char* e = getenv("RSW_FINE_RADIX");
    r = e ? atoi(e) : 0;
  }
  return r;
}
template <int N>
__host__ __device__ constexpr int coarse_radix() {  // palindromic; latency-bound (one pair per SM)
  return RSW_RADIX_COARSE ? RSW_RADIX_COARSE : (N <= 32 ? 4 : N <= 256 ? 8 : 16);
}
template <int N>
__host__ __device__ constexpr int coarse_threads() { return core_threads<N, coarse_radix<N>()>() > 192 ? core_threads<N, coarse_radix<N>()>() : 192; }

// ---------------------------------------------------------------------------------------------
// shared helpers: load a pair of half-spectrum states into packed eigen coordinates, and store
// ---------------------------------------------------------------------------------------------
template <int N, int T>
__device__ __forceinline__ void load_pair_eigen(const double* __restrict__ uA, const double* __restrict__ uB,
                                                const ModeGeom g, double2* C /*[3][Kc]*/) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  const double2* A = reinterpret_cast<const double2*>(uA);
  const double2* B = reinterpret_cast<const double2*>(uB);
  for (int j = threadIdx.x; j < Kc; j += T) {
    const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
    double2 z[3];
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double2 a = A[f * NH + ak];
      double2 b = B ? B[f * NH + ak] : make_double2(0.0, 0.0);
      if (kap < 0) {  // û(-κ) = conj(û(κ)) for real fields (R16)
        a = cconj(a);
        b = cconj(b);
      }
      z[f] = make_double2(a.x - b.y, a.y + b.x);  // a + i b
    }
    const double as = kap < 0 ? -__ldg(g.a + ak) : __ldg(g.a + ak);
    double2 c[3];
    to_eigen(as, __ldg(g.p + ak), __ldg(g.q + ak), z, c);
#pragma unroll
    for (int al = 0; al < 3; ++al) C[al * Kc + j] = c[al];
  }
}

// unpack Z = Û_A + i Û_B (primitive, from eigen C) and store both half spectra (modes > K -> 0)
template <int N, int T>
__device__ __forceinline__ void store_pair_prim(const double2* C, const ModeGeom g, double* __restrict__ oA,
                                                double* __restrict__ oB) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  double2* A = reinterpret_cast<double2*>(oA);
  double2* B = reinterpret_cast<double2*>(oB);
  for (int k = threadIdx.x; k < NH; k += T) {
    double2 ua[3], ub[3];
    if (k <= K) {
      const double a = __ldg(g.a + k), p = __ldg(g.p + k), q = __ldg(g.q + k);
      double2 cp[3], cm[3], zp[3], zm[3];
      const int jm = (k == 0) ? 0 : Kc - k;  // compact index of -κ
#pragma unroll
      for (int al = 0; al < 3; ++al) {
        cp[al] = C[al * Kc + k];
        cm[al] = C[al * Kc + jm];
      }
      to_prim(a, p, q, cp, zp);
      to_prim(-a, p, q, cm, zm);
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        const double2 zc = cconj(zm[f]);
        ua[f] = cscale(cadd(zp[f], zc), 0.5);
        ub[f] = cscale(cmulmi(csub(zp[f], zc)), 0.5);  // (Z - conj Z(-κ)) / (2i)
      }
      if (k == 0) {
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          ua[f].y = 0.0;
          ub[f].y = 0.0;
        }
      }
    } else {
#pragma unroll
      for (int f = 0; f < 3; ++f) ua[f] = ub[f] = make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      A[f * NH + k] = ua[f];
      if (B) B[f * NH + k] = ub[f];
    }
  }
}

// write prim(x) of every retained entry as the next N-eval input and zero the tail
template <int N, int T>
__device__ __forceinline__ void prologue_from(double2* W, const double2* X, const ModeGeom g) {
  constexpr int K = N / 3, Kc = 2 * K + 1;
  for (int j = threadIdx.x; j < Kc; j += T) {
    const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
    const double as = kap < 0 ? -__ldg(g.a + ak) : __ldg(g.a + ak);
    double2 c[3], u[3];
#pragma unroll
    for (int al = 0; al < 3; ++al) c[al] = X[al * Kc + j];
    to_prim(as, __ldg(g.p + ak), __ldg(g.q + ak), c, u);
    put_input<N>(W, full_index(kap, N), (double)kap, u);
  }
  zero_tail<N, T>(W);
}

// ---------------------------------------------------------------------------------------------
// K1/K2: fine propagator.  One CTA = one pair of slices, state resident in shared memory for all
// m steps; the only global traffic is one load and one store per slice.
//   ETDRK4 (Cox–Matthews), eigen-diagonal form with three persistent vectors S0, S1, S2:
//     stage 0 (n0 = N(c)):  S0 = E2 c;  S1 = E c + f1 n0;  a = S0 + Q n0;  S2 = E2 a - Q n0;  x = a
//     stage 1 (n1 = N(a)):  x = b = S0 + Q n1;  S1 += f2 n1
//     stage 2 (n2 = N(b)):  x = c' = S2 + 2 Q n2;  S1 += f2 n2
//     stage 3 (n3 = N(c')): S1 += f3 n3;  x = S1 (next state)
//   which is u+ = E u + f1 Nu + f2 (Na + Nb) + f3 Nc with a, b, c' as in Cox–Matthews.
//   Strang (Alg.3 + R7): v = E2 c;  m = v + (h/2) N(v);  w = v + h N(m);  c+ = E2 w.
// ---------------------------------------------------------------------------------------------
template <int N, int R, int T>
struct FineLayout {  // dynamic shared memory of k_fine (double2 units first, then doubles)
  static constexpr int K = N / 3, KP = K + 1;
  static constexpr int W = 0, Y = W + 3 * N, TW = Y + 3 * N, CP = TW + fft_tw_size<N, R>(), D = CP + 6 * KP;
  static constexpr int C0 = 0, GA = C0 + 6 * KP, GP = GA + KP, GQ = GP + KP, ND = GQ + KP;      // double offsets
  static constexpr size_t bytes = sizeof(double2) * D + sizeof(double) * ND;
  static constexpr int Kc = 2 * K + 1, OMAX = (Kc + T - 1) / T, NGRP = (T + 127) / 128;
  static constexpr int NCOL = tmem_cols_pow2<NGRP * OMAX * 36>();  // TMEM columns (S1, S0, S2 per mode slot)
};

template <int N, int R, int T, int SCHEME, bool LIN>
__global__ void __launch_bounds__(T) k_fine(const double* u_in, double* u_out, int n_slices, int m_steps,
                                            double h, const FineTab tab) {
  using LY = FineLayout<N, R, T>;
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1, KP = K + 1, OMAX = LY::OMAX;
  constexpr double invN = 1.0 / N;
  extern __shared__ double2 smem[];
  double2* W = smem + LY::W;   // N-eval input / output (natural order, padded)
  double2* Y = smem + LY::Y;   // ping-pong partner of the register FFT core
  double2* sTW = smem + LY::TW;
  double2* sCP = smem + LY::CP;
  double* sd = reinterpret_cast<double*>(smem + LY::D);
  double* sC0 = sd + LY::C0;
  double* sGA = sd + LY::GA;
  double* sGP = sd + LY::GP;
  double* sGQ = sd + LY::GQ;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<LY::NCOL>(&tslot);
  // per-configuration tables into shared memory (read every stage)
  fill_packed_twiddles<N, R, T>(sTW, tab.tw);
  for (int i = threadIdx.x; i < 6 * KP; i += T) {
    sCP[i] = __ldg(tab.cp + i);
    sC0[i] = __ldg(tab.c0 + i);
  }
  for (int i = threadIdx.x; i < KP; i += T) {
    sGA[i] = __ldg(tab.g.a + i);
    sGP[i] = __ldg(tab.g.p + i);
    sGQ[i] = __ldg(tab.g.q + i);
  }
  const int sA = 2 * blockIdx.x, sB = sA + 1;
  const size_t L = (size_t)3 * NH * 2;
  const double* inB = (sB < n_slices) ? u_in + sB * L : nullptr;
  load_pair_eigen<N, T>(u_in + sA * L, inB, tab.g, W);  // C[α][j] staged in W
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  // thread-private TMEM slot of mode slot o: columns o*36 + {S1: 0, S0: 12, S2: 24} + 4α
  const uint32_t tb = tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * OMAX * 36);
  double2 c0v[OMAX][3];
#pragma unroll
  for (int o = 0; o < OMAX; ++o) {
    const int j = threadIdx.x + o * T;
#pragma unroll
    for (int al = 0; al < 3; ++al) c0v[o][al] = (j < Kc) ? W[al * Kc + j] : make_double2(0.0, 0.0);
  }
  __syncthreads();  // C fully read before W receives the first N-eval input
#pragma unroll
  for (int o = 0; o < OMAX; ++o) {
    const int j = threadIdx.x + o * T;
    const int jj = j < Kc ? j : 0;
    const int kap = kappa_of(jj, K), ak = kap < 0 ? -kap : kap;
    if (SCHEME == 1) {  // Strang prologue: S1 = v = E2 c
#pragma unroll
      for (int al = 0; al < 3; ++al) c0v[o][al] = dmul(al - 1, sCP[1 * KP + ak], sC0[1 * KP + ak], c0v[o][al]);
    }
    tmem_st3(tb + o * 36, c0v[o]);
    if (!LIN && j < Kc) {
      const double as = kap < 0 ? -sGA[ak] : sGA[ak];
      double2 u[3];
      to_prim(as, sGP[ak], sGQ[ak], c0v[o], u);
      put_input_z<N>(W, full_index(kap, N), (double)kap, u);
    }
  }
  tmem_wait_st();
  __syncthreads();

  const int nst = (SCHEME == 0) ? 4 : 2;
  for (int step = 0; step < m_steps; ++step) {
    const bool last_step = (step == m_steps - 1);
    for (int st = 0; st < nst; ++st) {
      if (!LIN) nl_core<N, R, T>(W, Y, sTW);
      // epilogue (this stage's update) fused with the prologue of the next N-eval
#pragma unroll
      for (int o = 0; o < OMAX; ++o) {
        const int j = threadIdx.x + o * T;
        const bool valid = j < Kc;
        const int jj = valid ? j : 0;
        const int kap = kappa_of(jj, K), ak = kap < 0 ? -kap : kap;
        const int kf = full_index(kap, N);
        const uint32_t ts = tb + o * 36;
        double2 s1[3], s0[3], s2[3];
        tmem_ld3(ts, s1);                                            // S1 (every stage)
        if (SCHEME == 0 && st == 1) tmem_ld3(ts + 12, s0);           // S0 = E2 c
        if (SCHEME == 0 && st == 2) tmem_ld3(ts + 24, s2);           // S2 = E2 a - Q Nu
        const double as = kap < 0 ? -sGA[ak] : sGA[ak];
        const double p = sGP[ak], q = sGQ[ak];
        double2 nn[3];
        if (!LIN && valid) {
          double2 nh[3];
          get_output_z<N>(W, kf, (double)kap, invN, nh);
          to_eigen(as, p, q, nh, nn);
        } else {
#pragma unroll
          for (int al = 0; al < 3; ++al) nn[al] = make_double2(0.0, 0.0);
        }
        double2 x[3];
#pragma unroll
        for (int al = 0; al < 3; ++al) {
          const int alpha = al - 1;
          // coefficient i of |κ|: 0 E, 1 E2, 2 Q, 3 f1, 4 f2, 5 f3
#define CP(i) sCP[(i) * KP + ak]
#define C0(i) sC0[(i) * KP + ak]
          if (SCHEME == 0) {
            if (st == 0) {
              const double2 c = s1[al];
              const double2 e2c = dmul(alpha, CP(1), C0(1), c);
              const double2 qn = dmul(alpha, CP(2), C0(2), nn[al]);
              const double2 a = cadd(e2c, qn);
              s0[al] = e2c;
              s1[al] = cadd(dmul(alpha, CP(0), C0(0), c), dmul(alpha, CP(3), C0(3), nn[al]));
              s2[al] = csub(dmul(alpha, CP(1), C0(1), a), qn);
              x[al] = a;
            } else if (st == 1) {
              x[al] = cadd(s0[al], dmul(alpha, CP(2), C0(2), nn[al]));
              s1[al] = cadd(s1[al], dmul(alpha, CP(4), C0(4), nn[al]));
            } else if (st == 2) {
              x[al] = cadd(s2[al], cscale(dmul(alpha, CP(2), C0(2), nn[al]), 2.0));
              s1[al] = cadd(s1[al], dmul(alpha, CP(4), C0(4), nn[al]));
            } else {
              s1[al] = cadd(s1[al], dmul(alpha, CP(5), C0(5), nn[al]));
              x[al] = s1[al];
            }
          } else {
            if (st == 0) {
              x[al] = caxpy(0.5 * h, nn[al], s1[al]);  // m = v + (h/2) N(v)
            } else {
              const double2 w = caxpy(h, nn[al], s1[al]);                     // w = v + h N(m)
              const double2 c = dmul(alpha, CP(1), C0(1), w);                 // c+ = E2 w
              s1[al] = last_step ? c : dmul(alpha, CP(1), C0(1), c);          // next v = E2 c+
              x[al] = s1[al];
            }
          }
#undef CP
#undef C0
        }
        if (SCHEME == 0 || st == 1) tmem_st3(ts, s1);
        if (SCHEME == 0 && st == 0) {
          tmem_st3(ts + 12, s0);
          tmem_st3(ts + 24, s2);
        }
        if (!LIN && valid) {
          double2 u[3];
          to_prim(as, p, q, x, u);
          put_input_z<N>(W, kf, (double)kap, u);
        }
      }
      tmem_wait_st();
      __syncthreads();
    }
  }
  // final state S1 -> C[α][j] in Y (W may still hold the last stage's inputs), then store
#pragma unroll
  for (int o = 0; o < OMAX; ++o) {
    const int j = threadIdx.x + o * T;
    double2 s1[3];
    tmem_ld3(tb + o * 36, s1);
    if (j < Kc) {
#pragma unroll
      for (int al = 0; al < 3; ++al) Y[al * Kc + j] = s1[al];
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc<LY::NCOL>(tslot);
  }
  store_pair_prim<N, T>(Y, tab.g, u_out + sA * L, (sB < n_slices) ? u_out + sB * L : nullptr);
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

// ---------------------------------------------------------------------------------------------
// K4: the serial coarse sweep (Alg.4's serial loop P:583-587 over Alg.2 coarse steps) as ONE
// persistent cooperative kernel.  Per RK stage of slice n:
//   phase 1 (all CTAs, sample-parallel as Alg.1): CTA b evaluates its sample pairs
//     (m_A, m_B) = (2p+1, 2p+2), p = b, b+P, ..., packing the two rotated copies P-_m y of the
//     stage input into one complex field, and writes its partial Σ w_m P+_m N(P-_m y) to part[b];
//   grid barrier;
//   phase 2 (distributed over |κ|): CTA b owns |κ| ≡ b (mod P) and reduces part[0..P-1] for its 6
//     eigen entries (α, ±κ) in a fixed order, then applies the RK4 / midpoint stage update; at the
//     last stage also the D half step, the back-transform e^{-(ΔT/ε)L̂}, the parareal update
//     U_{n+1} = G + (F_n - G_n) with the residual partials (R12), and slice n+1's first input;
//   grid barrier.
// Cross-CTA data (y, part) is read with ld.global.cg (L2), never through the incoherent L1.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// grid barrier: monotone arrival counter, arrive with a gpu-scope release RMW, spin with
// gpu-scope acquire loads (1.2 us at 128-148 CTAs on B200, vs 2.2 us for a volatile-flag barrier;
// tools/micro/barrier_bench.cu).  `epoch` counts this CTA's barriers; the counter is zeroed by the
// host before the launch.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks, unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    const unsigned target = epoch * nblocks;
    while (ld_acquire_gpu(bar) < target) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Stage input through a triple-buffered shared array (replaces "owners write y -> grid barrier ->
// everyone loads y"): update phase u writes its owned entries of the next stage input into
// ybuf[u%3] (each entry once) and resets the same entries of ybuf[(u+2)%3] to the sentinel; the
// samples phase polls ybuf[u%3] until no entry holds the sentinel.  Safe without fences: each
// 8-byte half is single-copy atomic; the reset of ybuf[(u+2)%3] happens after every reader of it
// (samples phase u-1) passed the release/acquire grid barrier before update u, and it is ordered
// before any reader of ybuf[(u+2)%3] (samples phase u+2) by the grid barrier after samples u+1.
constexpr unsigned long long YIN_SENTINEL = 0x7FF4DEADBEEF0001ull;  // a signalling-NaN payload arithmetic never produces
__device__ __forceinline__ double2 ld_relaxed_v2(const double2* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_v2(double2* p, double2 v) {
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ bool is_sentinel(double x) { return (unsigned long long)__double_as_longlong(x) == YIN_SENTINEL; }
__device__ __forceinline__ double2 yin_sentinel() {
  const double s = __longlong_as_double((long long)YIN_SENTINEL);
  return make_double2(s, s);
}

template <int N, int R, int T>
__device__ __forceinline__ void coarse_samples_phase(const double2* y, double2* part, int M, const AvgTab& tab,
                                                     double2* X, double2* Y, const double2* TW, double2* C,
                                                     double2* A, const double2* PH, const double* SW,
                                                     const double* GA, const double* GP, const double* GQ,
                                                     unsigned long long* cyc = nullptr) {
#define STAMP(i) \
  if (cyc && threadIdx.x == 0) cyc[i] = clock64();
  STAMP(0)
  // PH: this CTA's phases e^{iωτ_m} for its first pair, [2][K+1] (null: load from the table);
  // SW: its weights w_mA, w_mB; GA/GP/GQ: geometry a, p, q per |κ| staged in shared memory
  constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1;
  constexpr double invN = 1.0 / N;
  // stage input from this CTA's inbox (y = inbox row): poll, keep, reset to the sentinel
  for (int i = threadIdx.x; i < 3 * Kc; i += T) {
    double2 v = ld_relaxed_v2(y + i);
    while (is_sentinel(v.x) || is_sentinel(v.y)) v = ld_relaxed_v2(y + i);
    C[i] = v;
    A[i] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int npairs = M / 2;  // samples 1..M-1 -> pairs (1,2), (3,4), ...; last B may be M (w=0)
  for (int pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
    const int mA = 2 * pr + 1, mB = 2 * pr + 2;
    const bool hasB = mB <= M - 1;
    const bool cached = PH && pr == (int)blockIdx.x;
    for (int j = threadIdx.x; j < Kc; j += T) {
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
      const double as = kap < 0 ? -GA[ak] : GA[ak];
      const double2 pA = cached ? PH[ak] : __ldg(tab.phase + (size_t)mA * KP + ak);
      const double2 pB = !hasB ? make_double2(1.0, 0.0) : (cached ? PH[KP + ak] : __ldg(tab.phase + (size_t)mB * KP + ak));
      double2 c[3], u[3];
      // packed eigen input: P-_{mA} y + i P-_{mB} y   (P-: α=-1 -> e^{+iωτ}, α=+1 -> e^{-iωτ})
      const double2 ym = C[j], y0 = C[Kc + j], yp = C[2 * Kc + j];
      const double2 bm = hasB ? cmul(ym, pB) : make_double2(0.0, 0.0);
      const double2 b0 = hasB ? y0 : make_double2(0.0, 0.0);
      const double2 bp = hasB ? cmulc(yp, pB) : make_double2(0.0, 0.0);
      c[0] = cadd(cmul(ym, pA), cmuli(bm));
      c[1] = cadd(y0, cmuli(b0));
      c[2] = cadd(cmulc(yp, pA), cmuli(bp));
      to_prim(as, GP[ak], GQ[ak], c, u);
      put_input_z<N>(X, full_index(kap, N), (double)kap, u);
    }
    __syncthreads();
    STAMP(1)
    nl_core<N, R, T>(X, Y, TW);
    STAMP(2)
    const double wA = cached ? SW[0] : __ldg(tab.w + mA), wB = hasB ? (cached ? SW[1] : __ldg(tab.w + mB)) : 0.0;
    for (int j = threadIdx.x; j < Kc; j += T) {
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
      const double as = kap < 0 ? -GA[ak] : GA[ak];
      const double p = GP[ak], q = GQ[ak];
      double2 zp[3], zm[3], na[3], nb[3], ea[3], eb[3];
      get_output_z<N>(X, full_index(kap, N), (double)kap, invN, zp);
      get_output_z<N>(X, full_index(-kap, N), (double)(-kap), invN, zm);
#pragma unroll
      for (int f = 0; f < 3; ++f) {  // unpack: N_A(κ) = (Z(κ) + conj Z(-κ))/2, N_B = (Z - conj Z(-κ))/(2i)
        const double2 zc = cconj(zm[f]);
        na[f] = cscale(cadd(zp[f], zc), 0.5);
        nb[f] = cscale(cmulmi(csub(zp[f], zc)), 0.5);
      }
      to_eigen(as, p, q, na, ea);
      to_eigen(as, p, q, nb, eb);
      const double2 pA = cached ? PH[ak] : __ldg(tab.phase + (size_t)mA * KP + ak);
      A[j] = caxpy(wA, cmulc(ea[0], pA), A[j]);  // P+: α=-1 -> e^{-iωτ}, α=+1 -> e^{+iωτ}
      A[Kc + j] = caxpy(wA, ea[1], A[Kc + j]);
      A[2 * Kc + j] = caxpy(wA, cmul(ea[2], pA), A[2 * Kc + j]);
      if (hasB) {
        const double2 pB = cached ? PH[KP + ak] : __ldg(tab.phase + (size_t)mB * KP + ak);
        A[j] = caxpy(wB, cmulc(eb[0], pB), A[j]);
        A[Kc + j] = caxpy(wB, eb[1], A[Kc + j]);
        A[2 * Kc + j] = caxpy(wB, cmul(eb[2], pB), A[2 * Kc + j]);
      }
    }
    __syncthreads();  // all mirror reads of X done before the next prologue overwrites it
    STAMP(3)
  }
  double2* P = part + (size_t)blockIdx.x * 3 * Kc;
  for (int i = threadIdx.x; i < 3 * Kc; i += T) P[i] = A[i];
  STAMP(4)
#undef STAMP
}

// phase 2 of one RK stage, thread-parallel over the CTA's owned modes |κ| = b + o P (o < NOWN):
// items i = o*6 + e, entries e = (α, +κ) for e < 3, (α, -κ) for e >= 3.  The stage base v and the RK
// accumulator ks of owned modes live in this CTA's shared memory for the whole sweep; the stage
// input y is published to global memory for the samples phase of every CTA.
template <int N, int NOWN, int T>
__device__ __forceinline__ void push_stage_input(const CoarseArgs& ca, const double2* yv, const int* yidx, unsigned u) {
  constexpr int Kc3 = 3 * (2 * (N / 3) + 1);
  __syncthreads();
  if (threadIdx.x < NOWN * 6 && yidx[threadIdx.x] >= 0) {
    st_relaxed_v2(ca.yin + (size_t)(u % 3) * Kc3 + yidx[threadIdx.x], yv[threadIdx.x]);
    st_relaxed_v2(ca.yin + (size_t)((u + 2) % 3) * Kc3 + yidx[threadIdx.x], yin_sentinel());
  }
}

template <int N, int T, int NOWN>
__device__ __forceinline__ void coarse_update_phase(const CoarseArgs& ca, int stage, int n, double2* Vs,
                                                    double2* KSs, double2* kk, double2* un_s, double* nd_s,
                                                    double2* red_buf, double2* yv, int* yidx, unsigned ucount) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1, NW = T / 32;
  const int P = gridDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t Ls = (size_t)3 * NH;
  const double dT = ca.dT;
  auto entry = [&](int o, int e, int& ak, int& al, int& j) {
    ak = blockIdx.x + o * P;
    al = e % 3;
    j = (e < 3) ? ak : ((ak == 0) ? 0 : Kc - ak);
  };
  const bool last = (ca.scheme == 0) ? (stage == 4) : (stage == 2);
  // prefetch the finalize operands (F_n, old G_n, old U_{n+1}) before the reduction's L2 round trip
  double2 pf_F = make_double2(0.0, 0.0), pf_G = make_double2(0.0, 0.0), pf_U = make_double2(0.0, 0.0);
  if (stage > 0 && last && threadIdx.x < NOWN * 3) {
    const int o = threadIdx.x / 3, f = threadIdx.x % 3, ak = blockIdx.x + o * P;
    if (ak <= K) {
      if (ca.F) pf_F = __ldcg(reinterpret_cast<const double2*>(ca.F) + (size_t)n * Ls + f * NH + ak);
      pf_G = reinterpret_cast<const double2*>(ca.G)[(size_t)n * Ls + f * NH + ak];
      pf_U = reinterpret_cast<const double2*>(ca.U)[(size_t)(n + 1) * Ls + f * NH + ak];
    }
  }
  if (stage > 0) {
    // deterministic reduction of the partials: TQ threads per item issue all their loads at once,
    // then a fixed-order tree in shared memory
    constexpr int ITEMS = NOWN * 6;
    constexpr int TQ0 = T / ITEMS;
    constexpr int TQ = TQ0 >= 32 ? 32 : TQ0 >= 16 ? 16 : TQ0 >= 8 ? 8 : TQ0 >= 4 ? 4 : TQ0 >= 2 ? 2 : 1;
    double2* rd = reinterpret_cast<double2*>(red_buf);
    const int it = threadIdx.x / TQ, qd = threadIdx.x % TQ;
    if (it < ITEMS) {
      int ak, al, j;
      entry(it / 6, it % 6, ak, al, j);
      double2 sacc = make_double2(0.0, 0.0);
      if (ak <= K)
        for (int b = qd; b < ca.nparts; b += TQ) sacc = cadd(sacc, __ldcg(ca.part + (size_t)b * 3 * Kc + al * Kc + j));
      rd[threadIdx.x] = sacc;
    }
    __syncthreads();
#pragma unroll
    for (int w = TQ / 2; w > 0; w >>= 1) {
      if (it < ITEMS && qd < w) rd[threadIdx.x] = cadd(rd[threadIdx.x], rd[threadIdx.x + w]);
      __syncthreads();
    }
    if (it < ITEMS && qd == 0) kk[it] = rd[threadIdx.x];
    __syncthreads();
    if (threadIdx.x < NOWN * 6) {
      int ak, al, j;
      const int it = threadIdx.x;
      entry(it / 6, it % 6, ak, al, j);
      if (ak <= K && !(ak == 0 && it % 6 >= 3)) {
        const double2 k = kk[it];
        double2& V = Vs[it];
        double2& KS = KSs[it];
        double2* Y = yv + it;
        yidx[it] = last ? -1 : al * Kc + j;
        if (ca.scheme == 0) {  // classical RK4 (R6): (k1 + 2k2 + 2k3 + k4) accumulated in this order
          if (stage == 1) {
            KS = k;
            *Y = caxpy(0.5 * dT, k, V);
          } else if (stage == 2) {
            KS = caxpy(2.0, k, KS);
            *Y = caxpy(0.5 * dT, k, V);
          } else if (stage == 3) {
            KS = caxpy(2.0, k, KS);
            *Y = caxpy(dT, k, V);
          } else {
            KS = cadd(KS, k);
            V = caxpy(dT / 6.0, KS, V);
          }
        } else {  // midpoint (Alg.2, R7): v + ΔT N̄(v + ΔT/2 N̄(v))
          if (stage == 1) *Y = caxpy(0.5 * dT, k, V);
          else V = caxpy(dT, k, V);
        }
      } else {
        yidx[it] = -1;
      }
    }
    if (!last) {
      push_stage_input<N, NOWN, T>(ca, yv, yidx, ucount);
      return;
    }
    __syncthreads();
    // finalize: D half step, back-transform, primitive G, parareal update (thread per (o, f))
    if (threadIdx.x < NOWN * 3) {
      const int o = threadIdx.x / 3, f = threadIdx.x % 3, ak = blockIdx.x + o * P;
      if (ak <= K) {
        const double a = __ldg(ca.g.a + ak), p = __ldg(ca.g.p + ak), q = __ldg(ca.g.q + ak);
        const double dh = __ldg(ca.dhalf + ak);
        const double2 bt = __ldg(ca.back + ak);  // e^{-iωΔT/ε}: α=+1 entry of e^{-(ΔT/ε)L̂} (R3)
        double2 cg[3], G[3];
#pragma unroll
        for (int al = 0; al < 3; ++al) {
          const double2 c = cscale(Vs[o * 6 + al], dh);  // e^{(ΔT/2) D̂} (Alg.2)
          cg[al] = (al == 1) ? c : (al == 2 ? cmul(c, bt) : cmulc(c, bt));
        }
        to_prim(a, p, q, cg, G);
        double2 g = G[f];
        if (ak == 0) g.y = 0.0;
        double2* Gst = reinterpret_cast<double2*>(ca.G) + (size_t)n * Ls + f * NH + ak;
        double2* Uo = reinterpret_cast<double2*>(ca.U) + (size_t)(n + 1) * Ls + f * NH + ak;
        double2 un = g;
        if (ca.F) un = cadd(g, csub(pf_F, pf_G));  // U^k_{n+1} = G(U^k_n) + (F_n - G_n)
        const double2 d = csub(un, pf_U);
        const double wk = (ak == 0 || 2 * ak == N) ? 1.0 : 2.0;
        nd_s[threadIdx.x * 2] = wk * (d.x * d.x + d.y * d.y);
        nd_s[threadIdx.x * 2 + 1] = wk * (un.x * un.x + un.y * un.y);
        *Gst = g;
        *Uo = un;
        un_s[threadIdx.x] = un;
        if (ak == K)  // modes K < k <= N/2 stay zero
          for (int k = K + 1; k < NH; ++k) {
            Uo[k - K] = make_double2(0.0, 0.0);
            Gst[k - K] = make_double2(0.0, 0.0);
          }
      }
    }
    __syncthreads();
    if (ca.rparts && threadIdx.x < NOWN) {
      const int ak = blockIdx.x + threadIdx.x * P;
      if (ak <= K) {
        const double* t = nd_s + threadIdx.x * 6;
        ca.rparts[((size_t)n * (K + 1) + ak) * 2 + 0] = t[0] + t[2] + t[4];
        ca.rparts[((size_t)n * (K + 1) + ak) * 2 + 1] = t[1] + t[3] + t[5];
      }
    }
    if (n + 1 >= ca.n_end) return;  // no next slice
  } else {
    // stage 0: load U_0 of owned modes
    if (threadIdx.x < NOWN * 3) {
      const int o = threadIdx.x / 3, f = threadIdx.x % 3, ak = blockIdx.x + o * P;
      if (ak <= K) un_s[threadIdx.x] = reinterpret_cast<const double2*>(ca.U)[(size_t)n * Ls + f * NH + ak];
    }
    __syncthreads();
  }
  // first stage input of the next slice: v = e^{ΔT D̂/2} u (Alg.2), eigen, both signs of κ
  if (threadIdx.x < NOWN * 6) {
    int ak, al, j;
    const int it = threadIdx.x, o = it / 6, e = it % 6;
    entry(o, e, ak, al, j);
    if (ak <= K && !(ak == 0 && e >= 3)) {
      const double a = __ldg(ca.g.a + ak), p = __ldg(ca.g.p + ak), q = __ldg(ca.g.q + ak);
      double2 u[3], c[3];
#pragma unroll
      for (int f = 0; f < 3; ++f) u[f] = (e < 3) ? un_s[o * 3 + f] : cconj(un_s[o * 3 + f]);
      to_eigen(e < 3 ? a : -a, p, q, u, c);
      const double2 v = cscale(c[al], __ldg(ca.dhalf + ak));
      Vs[it] = v;
      yv[it] = v;
      yidx[it] = al * Kc + j;
    } else {
      yidx[it] = -1;
    }
  }
  push_stage_input<N, NOWN, T>(ca, yv, yidx, ucount);
  __syncthreads();
}

template <int N, int R, int T, int NOWN>
struct CoarseLayout {  // dynamic shared memory of k_coarse_sweep (double2 units, then doubles)
  static constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1, NR = (T > NOWN * 6 ? T : NOWN * 6);
  static constexpr int X = 0, Y = X + 3 * N, TW = Y + 3 * N, C = TW + fft_tw_size<N, R>(), A = C + 3 * Kc,
                       VS = A + 3 * Kc, KS = VS + NOWN * 6, KK = KS + NOWN * 6, UN = KK + NOWN * 6,
                       RDB = UN + NOWN * 3, PH = RDB + T, YV = PH + 2 * KP, D = YV + NOWN * 6;
  static constexpr int RED = 0, GA = RED + NR, GP = GA + KP, GQ = GP + KP, SW = GQ + KP, YI = SW + 2,
                       ND = YI + NOWN * 6;  // YI: int entry indices stored in double slots
  static constexpr size_t bytes = sizeof(double2) * D + sizeof(double) * ND;
};

template <int N, int R, int T, int NOWN>
__global__ void __launch_bounds__(T) k_coarse_sweep(const CoarseArgs ca, const AvgTab tab, int M, unsigned* bar,
                                                    double* r_out) {
  using LY = CoarseLayout<N, R, T, NOWN>;
  constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1;
  extern __shared__ double2 smem[];
  double2* X = smem + LY::X;
  double2* Y = smem + LY::Y;
  double2* TW = smem + LY::TW;
  double2* C = smem + LY::C;
  double2* A = smem + LY::A;
  double2* Vs = smem + LY::VS;    // [NOWN*6]
  double2* KSs = smem + LY::KS;   // [NOWN*6]
  double2* kk = smem + LY::KK;    // [NOWN*6]
  double2* un_s = smem + LY::UN;  // [NOWN*3]
  double2* rdb = smem + LY::RDB;  // [T]
  double2* PH = smem + LY::PH;    // [2][K+1]
  double* sd = reinterpret_cast<double*>(smem + LY::D);
  double* red = sd + LY::RED;     // [max(T, NOWN*6)]
  double* GA = sd + LY::GA;       // [K+1] each
  double* GP = sd + LY::GP;
  double* GQ = sd + LY::GQ;
  double* SW = sd + LY::SW;       // [2]
  // per-CTA constants for the whole sweep: geometry, twiddles, and the phases / weights of this
  // CTA's sample pair
  fill_packed_twiddles<N, R, T>(TW, tab.tw);
  for (int k = threadIdx.x; k <= K; k += T) {
    GA[k] = __ldg(tab.g.a + k);
    GP[k] = __ldg(tab.g.p + k);
    GQ[k] = __ldg(tab.g.q + k);
  }
  const bool one_pair = (int)gridDim.x >= M / 2;
  if (one_pair && (int)blockIdx.x < M / 2) {
    const int mA = 2 * blockIdx.x + 1, mB = 2 * blockIdx.x + 2;
    for (int k = threadIdx.x; k <= K; k += T) {
      PH[k] = __ldg(tab.phase + (size_t)mA * KP + k);
      PH[KP + k] = __ldg(tab.phase + (size_t)mB * KP + k);
    }
    if (threadIdx.x == 0) {
      SW[0] = __ldg(tab.w + mA);
      SW[1] = mB <= M - 1 ? __ldg(tab.w + mB) : 0.0;
    }
  }
  __syncthreads();
  const double2* PHc = one_pair ? PH : nullptr;
  double2* yv = smem + LY::YV;
  int* yidx = reinterpret_cast<int*>(sd + LY::YI);
  const unsigned P = gridDim.x;
  constexpr int Kc3 = 3 * Kc;
  const int nst = ca.scheme == 0 ? 4 : 2;
  unsigned epoch = 0, ucount = 0;
  const bool prof = ca.prof && blockIdx.x == 0;
  int ps = 0;
  // the three stage-input buffers start empty (sentinel) before anyone writes
  for (int i = blockIdx.x * T + threadIdx.x; i < 3 * Kc3; i += P * T) st_relaxed_v2(ca.yin + i, yin_sentinel());
  grid_barrier(bar, P, epoch);
  coarse_update_phase<N, T, NOWN>(ca, 0, 0, Vs, KSs, kk, un_s, red, rdb, yv, yidx, ucount);  // slice 0: v = e^{ΔT D̂/2} U_0
  for (int n = 0; n < ca.n_end; ++n) {
    for (int st = 1; st <= nst; ++st) {
      if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 0] = gtimer();
      const double2* inbox = ca.yin + (size_t)(ucount % 3) * Kc3;
      coarse_samples_phase<N, R, T>(inbox, const_cast<double2*>(ca.part), M, tab, X, Y, TW, C, A, PHc, SW, GA, GP, GQ,
                                    (prof && ps == 8) ? ca.prof + 256 : nullptr);
      if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 1] = gtimer();
      grid_barrier(bar, P, epoch);
      if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 2] = gtimer();
      ++ucount;
      coarse_update_phase<N, T, NOWN>(ca, st, n, Vs, KSs, kk, un_s, red, rdb, yv, yidx, ucount);
      if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 3] = gtimer();
      ++ps;
    }
  }
  grid_barrier(bar, P, epoch);  // every slice's U, G and residual partials are written
  if (r_out && blockIdx.x == 0) {  // r_k = max_n sqrt(Σ num / Σ den) over slices (fixed order)
    double mx = 0.0;
    bool bad = false;
    for (int s = threadIdx.x; s < ca.n_end; s += T) {
      double num = 0.0, den = 0.0;
      for (int k = 0; k <= K; ++k) {
        num += __ldcg(ca.rparts + ((size_t)s * (K + 1) + k) * 2);
        den += __ldcg(ca.rparts + ((size_t)s * (K + 1) + k) * 2 + 1);
      }
      const double r = sqrt(num / den);
      if (!(r == r) || isinf(r)) bad = true;
      mx = fmax(mx, r);
    }
    double* rr = red;
    rr[threadIdx.x] = bad ? __longlong_as_double(0x7ff8000000000000LL) : mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      bool nan = false;
      for (int t = 0; t < T; ++t) {
        if (rr[t] != rr[t]) nan = true;
        m = fmax(m, rr[t]);
      }
      *r_out = nan ? __longlong_as_double(0x7ff8000000000000LL) : m;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Standard parareal (NEXT-1): the coarse solver is ONE Strang step of size ΔT on the
// full equation (Alg.3 with m = 1).  The serial sweep is a single CTA: per slice one Strang step
// (2 N-evals, the state in the real lane of the packed pair), the parareal update
// U_{n+1} = G + (F_n - G_n), G_n <- G, and the per-slice residual; r_k = max_n at the end.
// ---------------------------------------------------------------------------------------------
template <int N, int T>
__global__ void __launch_bounds__(T) k_strang_sweep(const FineTab tab, double h, double* U, double* G,
                                                     const double* F, double* Gnew, int S, double* r_out) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  constexpr double invN = 1.0 / N;
  extern __shared__ double2 smem[];
  double2* W = smem;
  double2* S1 = W + 3 * WL<N>::NP;
  __shared__ double red[2][T];
  __shared__ double rmax;
  if (threadIdx.x == 0) rmax = 0.0;
  const size_t L = (size_t)3 * NH * 2;
  for (int n = 0; n < S; ++n) {
    load_pair_eigen<N, T>(U + (size_t)n * L, nullptr, tab.g, S1);
    __syncthreads();
    for (int j = threadIdx.x; j < Kc; j += T) {  // v = E2 c
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
#pragma unroll
      for (int al = 0; al < 3; ++al)
        S1[al * Kc + j] = dmul(al - 1, __ldg(tab.cp + 1 * (K + 1) + ak), __ldg(tab.c0 + 1 * (K + 1) + ak),
                               S1[al * Kc + j]);
    }
    __syncthreads();
    prologue_from<N, T>(W, S1, tab.g);
    __syncthreads();
    for (int st = 0; st < 2; ++st) {
      nl_physical<N, T, radix_for<N>()>(W, tab.tw);
      for (int j = threadIdx.x; j < Kc; j += T) {
        const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
        const int kf = full_index(kap, N);
        const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
        const double p = __ldg(tab.g.p + ak), q = __ldg(tab.g.q + ak);
        double2 nh[3], nn[3], x[3];
        get_output<N>(W, kf, (double)kap, invN, nh);
        to_eigen(as, p, q, nh, nn);
#pragma unroll
        for (int al = 0; al < 3; ++al) {
          const int e = al * Kc + j;
          if (st == 0) {
            x[al] = caxpy(0.5 * h, nn[al], S1[e]);  // midpoint input v + (h/2) N(v)
          } else {
            const double2 w = caxpy(h, nn[al], S1[e]);  // w = v + h N(mid)
            S1[e] = dmul(al - 1, __ldg(tab.cp + 1 * (K + 1) + ak), __ldg(tab.c0 + 1 * (K + 1) + ak), w);
          }
        }
        if (st == 0) {
          double2 u[3];
          to_prim(as, p, q, x, u);
          put_input<N>(W, kf, (double)kap, u);
        }
      }
      if (st == 0) zero_tail<N, T>(W);
      __syncthreads();
    }
    store_pair_prim<N, T>(S1, tab.g, Gnew, nullptr);
    __syncthreads();
    // parareal update and residual (R12) over the half spectrum
    const double2* gn = reinterpret_cast<const double2*>(Gnew);
    double2* Go = reinterpret_cast<double2*>(G) + (size_t)n * 3 * NH;
    double2* Uo = reinterpret_cast<double2*>(U) + (size_t)(n + 1) * 3 * NH;
    const double2* Fn = F ? reinterpret_cast<const double2*>(F) + (size_t)n * 3 * NH : nullptr;
    double num = 0.0, den = 0.0;
    for (int i = threadIdx.x; i < 3 * NH; i += T) {
      const int k = i % NH;
      const double2 g = gn[i];
      const double2 un = Fn ? cadd(g, csub(Fn[i], Go[i])) : g;
      const double2 d = csub(un, Uo[i]);
      const double wk = (k == 0 || 2 * k == N) ? 1.0 : 2.0;
      num += wk * (d.x * d.x + d.y * d.y);
      den += wk * (un.x * un.x + un.y * un.y);
      Go[i] = g;
      Uo[i] = un;
    }
    red[0][threadIdx.x] = num;
    red[1][threadIdx.x] = den;
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0;
      for (int t = 0; t < T; ++t) {
        a += red[0][t];
        b += red[1][t];
      }
      const double r = sqrt(a / b);
      rmax = (r != r || rmax != rmax) ? __longlong_as_double(0x7ff8000000000000LL) : fmax(rmax, r);
    }
    __syncthreads();
  }
  if (r_out && threadIdx.x == 0) *r_out = rmax;
}

// M0: DFMA peak probe — independent FMA chains, every SM
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

// ---------------------------------------------------------------------------------------------
// launch wrappers (host side of this translation unit)
// ---------------------------------------------------------------------------------------------


template <int N>
constexpr size_t nl_smem() { return sizeof(double2) * (3 * WL<N>::NP + 3 * (2 * (N / 3) + 1)); }
template <int N>
constexpr size_t avg_smem() { return sizeof(double2) * (3 * WL<N>::NP + 2 * 3 * (2 * (N / 3) + 1)); }

template <typename KernelT>
static cudaError_t set_smem(KernelT k, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
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
  else LAUNCH_FINE(1, true)
#undef LAUNCH_FINE
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_fine_n(int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                                 const FineTab& tab, cudaStream_t st) {
  const int r = fine_radix_override();
  if constexpr (N == 256) {  // measured alternatives (RSW_FINE_RADIX, benchmarking only)
    if (r == 4) return launch_fine_nr<N, 4>(scheme, lin, in, out, S, m, h, tab, st);
    if (r == 16) return launch_fine_nr<N, 16>(scheme, lin, in, out, S, m, h, tab, st);
  }
  if constexpr (N == 1024) {
    if (r == 4) return launch_fine_nr<N, 4>(scheme, lin, in, out, S, m, h, tab, st);
    if (r == 32) return launch_fine_nr<N, 32>(scheme, lin, in, out, S, m, h, tab, st);
  }
  return launch_fine_nr<N, fine_radix<N>()>(scheme, lin, in, out, S, m, h, tab, st);
}

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

static int coarse_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RSW_COARSE_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int N, int NOWN, int R = coarse_radix<N>(), int T = coarse_threads<N>()>
static cudaError_t launch_coarse_sweep_nown(const CoarseArgs& ca, const AvgTab& tab, int M, unsigned* bar,
                                            double* r_out, int grid, cudaStream_t st) {
  if constexpr (N == 256 && R == coarse_radix<N>() && T == coarse_threads<N>()) {  // measured alternatives
    const int v = coarse_variant();
    if (v == 1) return launch_coarse_sweep_nown<N, NOWN, 8, 96>(ca, tab, M, bar, r_out, grid, st);
    if (v == 2) return launch_coarse_sweep_nown<N, NOWN, 4, 192>(ca, tab, M, bar, r_out, grid, st);
    if (v == 3) return launch_coarse_sweep_nown<N, NOWN, 16, 192>(ca, tab, M, bar, r_out, grid, st);
    if (v == 4) return launch_coarse_sweep_nown<N, NOWN, 8, 256>(ca, tab, M, bar, r_out, grid, st);
    if (v == 5) return launch_coarse_sweep_nown<N, NOWN, 4, 256>(ca, tab, M, bar, r_out, grid, st);
  }
  auto kfn = k_coarse_sweep<N, R, T, NOWN>;
  const size_t sm = CoarseLayout<N, R, T, NOWN>::bytes;
  cudaError_t e = set_smem(kfn, sm);
  if (e != cudaSuccess) return e;
  int dev, sms, per_sm;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, T, sm)) != cudaSuccess) return e;
  if (grid > per_sm * sms) return cudaErrorCooperativeLaunchTooLarge;
  CoarseArgs c2 = ca;
  c2.nparts = grid;
  if ((e = cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st)) != cudaSuccess) return e;
  void* args[] = {(void*)&c2, (void*)&tab, (void*)&M, (void*)&bar, (void*)&r_out};
  return cudaLaunchCooperativeKernel((const void*)kfn, dim3(grid), dim3(T), args, sm, st);
}

template <int N>
static cudaError_t launch_coarse_sweep_n(const CoarseArgs& ca, const AvgTab& tab, int M, unsigned* bar,
                                         double* r_out, int* grid_used, cudaStream_t st) {
  int dev, sms;
  cudaError_t e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  constexpr int K = N / 3;
  // one sample pair per CTA, but enough CTAs that each owns <= 16 modes in the update phase;
  // at most one CTA per SM (co-residency of the cooperative launch)
  int grid = M / 2;
  if (grid < (K + 1 + 15) / 16) grid = (K + 1 + 15) / 16;
  if (grid > sms) grid = sms;
  if (grid > ca.nparts) grid = ca.nparts;
  if (grid < 1) grid = 1;
  const int nown = (K + 1 + grid - 1) / grid;  // owned modes per CTA in the update phase
  if (grid_used) *grid_used = grid;
  if (nown <= 1) return launch_coarse_sweep_nown<N, 1>(ca, tab, M, bar, r_out, grid, st);
  if (nown <= 2) return launch_coarse_sweep_nown<N, 2>(ca, tab, M, bar, r_out, grid, st);
  if (nown <= 4) return launch_coarse_sweep_nown<N, 4>(ca, tab, M, bar, r_out, grid, st);
  if (nown <= 8) return launch_coarse_sweep_nown<N, 8>(ca, tab, M, bar, r_out, grid, st);
  if (nown <= 16) return launch_coarse_sweep_nown<N, 16>(ca, tab, M, bar, r_out, grid, st);
  return cudaErrorInvalidConfiguration;
}

template <int N>
static cudaError_t launch_strang_sweep_n(const FineTab& tab, double h, double* U, double* G, const double* F,
                                         double* Gnew, int S, double* r_out, cudaStream_t st) {
  constexpr int T = threads_for<N>();
  auto kfn = k_strang_sweep<N, T>;
  const size_t sm = nl_smem<N>();
  cudaError_t e = set_smem(kfn, sm);
  if (e != cudaSuccess) return e;
  kfn<<<1, T, sm, st>>>(tab, h, U, G, F, Gnew, S, r_out);
  return cudaGetLastError();
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

cudaError_t launch_fine(int n, int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                        const FineTab& tab, cudaStream_t st) {
#define C(NN) launch_fine_n<NN>(scheme, lin, in, out, S, m, h, tab, st)
  RSW_DISPATCH(n, C)
#undef C
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
cudaError_t launch_coarse_sweep(int n, const CoarseArgs& ca, const AvgTab& tab, int M, unsigned* bar, double* r_out,
                                int* grid_used, cudaStream_t st) {
#define C(NN) launch_coarse_sweep_n<NN>(ca, tab, M, bar, r_out, grid_used, st)
  RSW_DISPATCH(n, C)
#undef C
}
cudaError_t launch_strang_sweep(int n, const FineTab& tab, double h, double* U, double* G, const double* F,
                                double* Gnew, int S, double* r_out, cudaStream_t st) {
#define C(NN) launch_strang_sweep_n<NN>(tab, h, U, G, F, Gnew, S, r_out, st)
  RSW_DISPATCH(n, C)
#undef C
}
cudaError_t launch_dfma_peak(double* out, int blocks, int iters, cudaStream_t st) {
  k_dfma_peak<<<blocks, 256, 0, st>>>(out, iters);
  return cudaGetLastError();
}

}  // namespace rsw
