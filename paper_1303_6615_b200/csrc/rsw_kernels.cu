// rsw_kernels.cu — the hot-path kernels (sm_100a, fp64 CUDA cores; no tensor cores: the path is
// FFT + per-mode diagonal algebra, not a dense contraction).  See DESIGN.md §6 for the roofline of
// each kernel and rsw_device.cuh for the data layout.
#include "rsw_internal.h"
#include "rsw_device.cuh"

namespace rsw {

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
    put_input(W, N, full_index(kap, N), (double)kap, u);
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
template <int N, int T, int SCHEME, bool LIN>
__global__ void __launch_bounds__(T) k_fine(const double* u_in, double* u_out, int n_slices, int m_steps,
                                            double h, const FineTab tab) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  constexpr double invN = 1.0 / N;
  extern __shared__ double2 smem[];
  double2* W = smem;
  double2* S0 = W + 3 * N;
  double2* S1 = S0 + 3 * Kc;
  double2* S2 = S1 + 3 * Kc;
  const int sA = 2 * blockIdx.x, sB = sA + 1;
  const size_t L = (size_t)3 * NH * 2;
  const double* inB = (sB < n_slices) ? u_in + sB * L : nullptr;
  load_pair_eigen<N, T>(u_in + sA * L, inB, tab.g, S1);
  __syncthreads();

  if (SCHEME == 1) {  // Strang prologue: S1 = v = E2 c
    for (int j = threadIdx.x; j < Kc; j += T) {
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
#pragma unroll
      for (int al = 0; al < 3; ++al)
        S1[al * Kc + j] = dmul(al - 1, __ldg(tab.cp + 1 * (K + 1) + ak), __ldg(tab.c0 + 1 * (K + 1) + ak),
                               S1[al * Kc + j]);
    }
    __syncthreads();
  }
  if (!LIN) {
    prologue_from<N, T>(W, S1, tab.g);
    __syncthreads();
  }

  const int nst = (SCHEME == 0) ? 4 : 2;
  for (int step = 0; step < m_steps; ++step) {
    const bool last_step = (step == m_steps - 1);
    for (int st = 0; st < nst; ++st) {
      if (!LIN) nl_physical<N, T>(W, tab.tw);
      // epilogue (this stage's update) fused with the prologue of the next N-eval
      for (int j = threadIdx.x; j < Kc; j += T) {
        const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
        const int kf = full_index(kap, N);
        const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
        const double p = __ldg(tab.g.p + ak), q = __ldg(tab.g.q + ak);
        double2 nn[3];
        if (!LIN) {
          double2 nh[3];
          get_output(W, N, kf, (double)kap, invN, nh);
          to_eigen(as, p, q, nh, nn);
        } else {
#pragma unroll
          for (int al = 0; al < 3; ++al) nn[al] = make_double2(0.0, 0.0);
        }
        double2 x[3];
#pragma unroll
        for (int al = 0; al < 3; ++al) {
          const int alpha = al - 1, e = al * Kc + j;
          // coefficient i of |κ|: 0 E, 1 E2, 2 Q, 3 f1, 4 f2, 5 f3
#define CP(i) __ldg(tab.cp + (i) * (K + 1) + ak)
#define C0(i) __ldg(tab.c0 + (i) * (K + 1) + ak)
          if (SCHEME == 0) {
            if (st == 0) {
              const double2 c = S1[e];
              const double2 e2c = dmul(alpha, CP(1), C0(1), c);
              const double2 qn = dmul(alpha, CP(2), C0(2), nn[al]);
              const double2 a = cadd(e2c, qn);
              S0[e] = e2c;
              S1[e] = cadd(dmul(alpha, CP(0), C0(0), c), dmul(alpha, CP(3), C0(3), nn[al]));
              S2[e] = csub(dmul(alpha, CP(1), C0(1), a), qn);
              x[al] = a;
            } else if (st == 1) {
              x[al] = cadd(S0[e], dmul(alpha, CP(2), C0(2), nn[al]));
              S1[e] = cadd(S1[e], dmul(alpha, CP(4), C0(4), nn[al]));
            } else if (st == 2) {
              x[al] = cadd(S2[e], cscale(dmul(alpha, CP(2), C0(2), nn[al]), 2.0));
              S1[e] = cadd(S1[e], dmul(alpha, CP(4), C0(4), nn[al]));
            } else {
              const double2 c = cadd(S1[e], dmul(alpha, CP(5), C0(5), nn[al]));
              S1[e] = c;
              x[al] = c;
            }
          } else {
            if (st == 0) {
              x[al] = caxpy(0.5 * h, nn[al], S1[e]);  // m = v + (h/2) N(v)
            } else {
              const double2 w = caxpy(h, nn[al], S1[e]);          // w = v + h N(m)
              const double2 c = dmul(alpha, CP(1), C0(1), w);      // c+ = E2 w
              const double2 v = last_step ? c : dmul(alpha, CP(1), C0(1), c);  // next v = E2 c+
              S1[e] = v;
              x[al] = v;
            }
          }
#undef CP
#undef C0
        }
        if (!LIN) {
          double2 u[3];
          to_prim(as, p, q, x, u);
          put_input(W, N, kf, (double)kap, u);
        }
      }
      if (!LIN) zero_tail<N, T>(W);
      __syncthreads();
    }
  }
  store_pair_prim<N, T>(S1, tab.g, u_out + sA * L, (sB < n_slices) ? u_out + sB * L : nullptr);
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
  double2* C = W + 3 * N;
  const int sA = 2 * blockIdx.x, sB = sA + 1;
  const size_t L = (size_t)3 * NH * 2;
  load_pair_eigen<N, T>(u_in + sA * L, (sB < n_states) ? u_in + sB * L : nullptr, tab.g, C);
  __syncthreads();
  prologue_from<N, T>(W, C, tab.g);
  __syncthreads();
  nl_physical<N, T>(W, tab.tw);
  for (int j = threadIdx.x; j < Kc; j += T) {
    const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
    const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
    double2 nh[3], nn[3];
    get_output(W, N, full_index(kap, N), (double)kap, invN, nh);
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
  double2* C = W + 3 * N;
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
        put_input(W, N, full_index(kap, N), (double)kap, u);
      }
      zero_tail<N, T>(W);
      __syncthreads();
    }
    nl_physical<N, T>(W, tab.tw);
    const double wm = __ldg(tab.w + m);
    for (int j = threadIdx.x; j < Kc; j += T) {
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
      const int kf = full_index(kap, N);
      const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
      const double p = __ldg(tab.g.p + ak), q = __ldg(tab.g.q + ak);
      double2 nh[3], nn[3];
      get_output(W, N, kf, (double)kap, invN, nh);
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
        put_input(W, N, kf, (double)kap, u);
      }
    }
    zero_tail<N, T>(W);
    __syncthreads();
  }
  store_pair_prim<N, T>(A, tab.g, out + sA * L, (sB < n_states) ? out + sB * L : nullptr);
}

// ---------------------------------------------------------------------------------------------
// K4 (coarse step, one state): samples kernel.  CTA b evaluates the sample pairs
// (m_A, m_B) = (2p+1, 2p+2), p = b, b + gridDim.x, ..., packing the two rotated copies of the
// same state y into one complex field, and writes its partial sum (eigen, signed κ) to part[b].
// ---------------------------------------------------------------------------------------------
template <int N, int T>
__global__ void __launch_bounds__(T) k_coarse_samples(const double2* __restrict__ y, double2* __restrict__ part,
                                                      int M, const AvgTab tab) {
  constexpr int K = N / 3, Kc = 2 * K + 1;
  constexpr double invN = 1.0 / N;
  extern __shared__ double2 smem[];
  double2* W = smem;
  double2* C = W + 3 * N;
  double2* A = C + 3 * Kc;
  for (int i = threadIdx.x; i < 3 * Kc; i += T) {
    C[i] = y[i];
    A[i] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int npairs = M / 2;  // samples 1..M-1 -> pairs (1,2), (3,4), ...; last B may be M (w=0)
  for (int pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
    const int mA = 2 * pr + 1, mB = 2 * pr + 2;
    const bool hasB = mB <= M - 1;
    for (int j = threadIdx.x; j < Kc; j += T) {
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
      const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
      const double2 pA = __ldg(tab.phase + (size_t)mA * (K + 1) + ak);
      const double2 pB = hasB ? __ldg(tab.phase + (size_t)mB * (K + 1) + ak) : make_double2(1.0, 0.0);
      double2 c[3], u[3];
      // packed eigen input: P-_{mA} y + i P-_{mB} y
      const double2 ym = C[j], y0 = C[Kc + j], yp = C[2 * Kc + j];
      double2 bm = hasB ? cmul(ym, pB) : make_double2(0.0, 0.0);
      double2 b0 = hasB ? y0 : make_double2(0.0, 0.0);
      double2 bp = hasB ? cmulc(yp, pB) : make_double2(0.0, 0.0);
      c[0] = cadd(cmul(ym, pA), cmuli(bm));
      c[1] = cadd(y0, cmuli(b0));
      c[2] = cadd(cmulc(yp, pA), cmuli(bp));
      to_prim(as, __ldg(tab.g.p + ak), __ldg(tab.g.q + ak), c, u);
      put_input(W, N, full_index(kap, N), (double)kap, u);
    }
    zero_tail<N, T>(W);
    __syncthreads();
    nl_physical<N, T>(W, tab.tw);
    const double wA = __ldg(tab.w + mA), wB = hasB ? __ldg(tab.w + mB) : 0.0;
    for (int j = threadIdx.x; j < Kc; j += T) {
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
      const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
      const double p = __ldg(tab.g.p + ak), q = __ldg(tab.g.q + ak);
      double2 zp[3], zm[3], na[3], nb[3], ea[3], eb[3];
      get_output(W, N, full_index(kap, N), (double)kap, invN, zp);
      get_output(W, N, full_index(-kap, N), (double)(-kap), invN, zm);
#pragma unroll
      for (int f = 0; f < 3; ++f) {  // unpack: N_A(κ) = (Z(κ) + conj Z(-κ))/2, N_B = (Z - conj Z(-κ))/(2i)
        const double2 zc = cconj(zm[f]);
        na[f] = cscale(cadd(zp[f], zc), 0.5);
        nb[f] = cscale(cmulmi(csub(zp[f], zc)), 0.5);
      }
      to_eigen(as, p, q, na, ea);
      to_eigen(as, p, q, nb, eb);
      const double2 pA = __ldg(tab.phase + (size_t)mA * (K + 1) + ak);
      A[j] = caxpy(wA, cmulc(ea[0], pA), A[j]);
      A[Kc + j] = caxpy(wA, ea[1], A[Kc + j]);
      A[2 * Kc + j] = caxpy(wA, cmul(ea[2], pA), A[2 * Kc + j]);
      if (hasB) {
        const double2 pB = __ldg(tab.phase + (size_t)mB * (K + 1) + ak);
        A[j] = caxpy(wB, cmulc(eb[0], pB), A[j]);
        A[Kc + j] = caxpy(wB, eb[1], A[Kc + j]);
        A[2 * Kc + j] = caxpy(wB, cmul(eb[2], pB), A[2 * Kc + j]);
      }
    }
    __syncthreads();  // all mirror reads of W done before the next prologue overwrites it
  }
  double2* P = part + (size_t)blockIdx.x * 3 * Kc;
  for (int i = threadIdx.x; i < 3 * Kc; i += T) P[i] = A[i];
}

// ---------------------------------------------------------------------------------------------
// K4 (coarse step, one state): combine kernel.  One CTA per |κ| (handles κ and -κ, 6 eigen
// entries): deterministic sum of the partials, the RK4 / midpoint stage logic of Alg.2, and at
// the last stage the D half step, the back-transform e^{-(ΔT/ε)L̂}, the parareal update
// U_{n+1} = G + (F_n - G_n) (Eq. HMM parareal iteration), the residual partials (R12), and the
// first stage input of slice n+1.
//   mode: 0 = init from U[n] (no partials), 1..4 = RK stage s done, with `final` set on the last.
// ---------------------------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(128) k_coarse_combine(CoarseArgs ca, int stage, int n) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  const int ak = blockIdx.x;  // |κ|
  const int jp = ak, jm = (ak == 0) ? 0 : Kc - ak;
  const int ne = (ak == 0) ? 3 : 6;  // entries handled: (α, +κ) and (α, -κ)
  __shared__ double2 red[6][128];
  double2 ksum[6];
#pragma unroll
  for (int e = 0; e < 6; ++e) ksum[e] = make_double2(0.0, 0.0);
  if (stage > 0) {
    for (int b = threadIdx.x; b < ca.nparts; b += 128) {
      const double2* P = ca.part + (size_t)b * 3 * Kc;
#pragma unroll
      for (int e = 0; e < 6; ++e) {
        if (e < ne) {
          const int al = e % 3, j = (e < 3) ? jp : jm;
          ksum[e] = cadd(ksum[e], P[al * Kc + j]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) red[e][threadIdx.x] = ksum[e];
    __syncthreads();
    for (int s = 64; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
#pragma unroll
        for (int e = 0; e < 6; ++e) red[e][threadIdx.x] = cadd(red[e][threadIdx.x], red[e][threadIdx.x + s]);
      }
      __syncthreads();
    }
  }
  if (threadIdx.x != 0) return;
  const double a = ca.g.a[ak], p = ca.g.p[ak], q = ca.g.q[ak];
  const double dT = ca.dT;
  double2* V = ca.v;   // [3][Kc] stage base v (after the first D half step)
  double2* KS = ca.ks; // [3][Kc] RK accumulator
  double2* Y = ca.y;   // [3][Kc] next stage input
  const size_t Ls = (size_t)3 * NH;  // complex entries per half-spectrum state
  bool finalize = false;
  for (int e = 0; e < ne; ++e) {
    const int al = e % 3, j = (e < 3) ? jp : jm, idx = al * Kc + j;
    const double2 kk = red[e][0];
    if (stage == 0) break;
    if (ca.scheme == 0) {  // RK4
      if (stage == 1) {
        KS[idx] = kk;
        Y[idx] = caxpy(0.5 * dT, kk, V[idx]);
      } else if (stage == 2) {
        KS[idx] = caxpy(2.0, kk, KS[idx]);
        Y[idx] = caxpy(0.5 * dT, kk, V[idx]);
      } else if (stage == 3) {
        KS[idx] = caxpy(2.0, kk, KS[idx]);
        Y[idx] = caxpy(dT, kk, V[idx]);
      } else {
        KS[idx] = cadd(KS[idx], kk);
        V[idx] = caxpy(dT / 6.0, KS[idx], V[idx]);
        finalize = true;
      }
    } else {  // midpoint: v + ΔT N̄(v + ΔT/2 N̄(v))
      if (stage == 1) {
        Y[idx] = caxpy(0.5 * dT, kk, V[idx]);
      } else {
        V[idx] = caxpy(dT, kk, V[idx]);
        finalize = true;
      }
    }
  }
  if (stage == 0 || finalize) {
    const double dh = ca.dhalf[ak];
    const double2 bt = ca.back[ak];  // e^{-iω ΔT/ε}  (α=+1 entry of e^{-(ΔT/ε)L̂})
    const double2* Uin = reinterpret_cast<const double2*>(ca.U) + (size_t)n * Ls;
    double2* Uout = reinterpret_cast<double2*>(ca.U) + (size_t)(n + 1) * Ls;
    double2 unew[3];
    if (finalize) {
      // D half step, back-transform, primitive G at +κ
      double2 cg[3], G[3];
#pragma unroll
      for (int al = 0; al < 3; ++al) {
        double2 c = cscale(V[al * Kc + jp], dh);
        cg[al] = (al == 1) ? c : (al == 2 ? cmul(c, bt) : cmulc(c, bt));
      }
      to_prim(a, p, q, cg, G);
      if (ak == 0) {
#pragma unroll
        for (int f = 0; f < 3; ++f) G[f].y = 0.0;
      }
      double2* Gst = reinterpret_cast<double2*>(ca.G) + (size_t)n * Ls;
      double num = 0.0, den = 0.0;
      const double wk = (ak == 0 || 2 * ak == N) ? 1.0 : 2.0;
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        double2 un;
        if (ca.F) {
          const double2 Fv = reinterpret_cast<const double2*>(ca.F)[(size_t)n * Ls + f * NH + ak];
          un = cadd(G[f], csub(Fv, Gst[f * NH + ak]));
        } else {
          un = G[f];
        }
        const double2 uo = Uout[f * NH + ak];
        const double2 d = csub(un, uo);
        num += wk * (d.x * d.x + d.y * d.y);
        den += wk * (un.x * un.x + un.y * un.y);
        Gst[f * NH + ak] = G[f];
        Uout[f * NH + ak] = un;
        unew[f] = un;
      }
      if (ca.rparts) {
        ca.rparts[((size_t)n * (K + 1) + ak) * 2 + 0] = num;
        ca.rparts[((size_t)n * (K + 1) + ak) * 2 + 1] = den;
      }
      if (ak == K) {  // modes K < k <= N/2 stay zero
        for (int k = K + 1; k < NH; ++k)
          for (int f = 0; f < 3; ++f) {
            Uout[f * NH + k] = make_double2(0.0, 0.0);
            Gst[f * NH + k] = make_double2(0.0, 0.0);
          }
      }
      if (n + 1 >= ca.n_end) return;  // no next slice
    } else {
#pragma unroll
      for (int f = 0; f < 3; ++f) unew[f] = Uin[f * NH + ak];
    }
    // first stage input of the next slice: v = e^{ΔT D̂/2} u (eigen, both signs of κ)
    double2 cpos[3], cneg[3], uneg[3];
#pragma unroll
    for (int f = 0; f < 3; ++f) uneg[f] = cconj(unew[f]);
    to_eigen(a, p, q, unew, cpos);
    to_eigen(-a, p, q, uneg, cneg);
#pragma unroll
    for (int al = 0; al < 3; ++al) {
      const double2 vp = cscale(cpos[al], dh), vn = cscale(cneg[al], dh);
      V[al * Kc + jp] = vp;
      Y[al * Kc + jp] = vp;
      if (ak > 0) {
        V[al * Kc + jm] = vn;
        Y[al * Kc + jm] = vn;
      }
    }
  }
}

// residual r_k = max_n sqrt(Σ_κ num / Σ_κ den)  (fixed order; one CTA)
__global__ void __launch_bounds__(256) k_resid_max(const double* rparts, int S, int Kp1, double* r_out,
                                                   double* per_slice) {
  __shared__ double red[256];
  double mx = 0.0;
  bool bad = false;
  for (int n = threadIdx.x; n < S; n += 256) {
    double num = 0.0, den = 0.0;
    for (int k = 0; k < Kp1; ++k) {
      num += rparts[((size_t)n * Kp1 + k) * 2];
      den += rparts[((size_t)n * Kp1 + k) * 2 + 1];
    }
    const double r = sqrt(num / den);
    if (per_slice) per_slice[n] = r;
    if (!(r == r) || isinf(r)) bad = true;
    mx = fmax(mx, r);
  }
  red[threadIdx.x] = bad ? __longlong_as_double(0x7ff8000000000000LL) : mx;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double a = red[threadIdx.x], b = red[threadIdx.x + s];
      red[threadIdx.x] = (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000LL) : fmax(a, b);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *r_out = red[0];
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
constexpr int threads_for() { return (3 * N / 8) > 96 ? (3 * N / 8) : 96; }

template <int N>
constexpr size_t fine_smem() { return sizeof(double2) * (3 * N + 3 * 3 * (2 * (N / 3) + 1)); }
template <int N>
constexpr size_t nl_smem() { return sizeof(double2) * (3 * N + 3 * (2 * (N / 3) + 1)); }
template <int N>
constexpr size_t avg_smem() { return sizeof(double2) * (3 * N + 2 * 3 * (2 * (N / 3) + 1)); }

template <typename KernelT>
static cudaError_t set_smem(KernelT k, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int N>
static cudaError_t launch_fine_n(int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                                 const FineTab& tab, cudaStream_t st) {
  constexpr int T = threads_for<N>();
  const int grid = (S + 1) / 2;
  const size_t sm = fine_smem<N>();
  cudaError_t e;
#define LAUNCH_FINE(SC, LN)                                                  \
  {                                                                           \
    auto kfn = k_fine<N, T, SC, LN>;                                          \
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

template <int N>
static cudaError_t launch_coarse_samples_n(const double2* y, double2* part, int nparts, int M, const AvgTab& tab,
                                           cudaStream_t st) {
  constexpr int T = threads_for<N>();
  auto kfn = k_coarse_samples<N, T>;
  cudaError_t e = set_smem(kfn, avg_smem<N>());
  if (e != cudaSuccess) return e;
  kfn<<<nparts, T, avg_smem<N>(), st>>>(y, part, M, tab);
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_coarse_combine_n(const CoarseArgs& ca, int stage, int n, cudaStream_t st) {
  k_coarse_combine<N><<<N / 3 + 1, 128, 0, st>>>(ca, stage, n);
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
cudaError_t launch_coarse_samples(int n, const double2* y, double2* part, int nparts, int M, const AvgTab& tab,
                                  cudaStream_t st) {
#define C(NN) launch_coarse_samples_n<NN>(y, part, nparts, M, tab, st)
  RSW_DISPATCH(n, C)
#undef C
}
cudaError_t launch_coarse_combine(int n, const CoarseArgs& ca, int stage, int slice, cudaStream_t st) {
#define C(NN) launch_coarse_combine_n<NN>(ca, stage, slice, st)
  RSW_DISPATCH(n, C)
#undef C
}
cudaError_t launch_resid_max(const double* rparts, int S, int Kp1, double* r_out, double* per_slice,
                             cudaStream_t st) {
  k_resid_max<<<1, 256, 0, st>>>(rparts, S, Kp1, r_out, per_slice);
  return cudaGetLastError();
}
cudaError_t launch_dfma_peak(double* out, int blocks, int iters, cudaStream_t st) {
  k_dfma_peak<<<blocks, 256, 0, st>>>(out, iters);
  return cudaGetLastError();
}

}  // namespace rsw
