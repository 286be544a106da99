// rsw_device.cuh — device building blocks of the B200 hot path (sm_100a, fp64 CUDA cores).
//
// Layout conventions used by every kernel:
//  * One CTA advances a PAIR of real states (slices, states or quadrature samples) packed into ONE
//    complex field:  z = u_A + i u_B.  Every operator on the path is real-preserving (its symbol
//    at -κ is the conjugate of the symbol at κ), so it can be applied to the packed full
//    spectrum Z_κ = Û_A(κ) + i Û_B(κ) directly; only the physical-space products act on the real
//    and imaginary lanes separately.  Two real N-point transforms thus cost one complex N-point
//    FFT, with no real-FFT post-processing.
//  * Spectral state: compact signed wavenumbers j = 0..Kc-1, Kc = 2K+1, K = floor(N/3) (R10):
//    κ(j) = j for j <= K, j - Kc otherwise.  Eigen coordinates c_α(κ), α = -1, 0, +1 stored
//    [α+1][j], in the closed-form eigenbasis of L̂(κ).
//  * Work buffer W: double2[3][N] (fields v1, v2, h) — full spectrum or physical grid.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rsw {

// ---------------------------------------------------------------------------------------------
// complex arithmetic on double2
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cmuli(double2 a) { return make_double2(-a.y, a.x); }   // i a
__device__ __forceinline__ double2 cmulmi(double2 a) { return make_double2(a.y, -a.x); }  // -i a
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {               // a*b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 caxpy(double s, double2 a, double2 c) {  // s*a + c
  return make_double2(fma(s, a.x, c.x), fma(s, a.y, c.y));
}
// multiply by the diagonal coefficient of eigen-row α: α=+1 -> C, α=-1 -> conj(C), α=0 -> real c0
__device__ __forceinline__ double2 dmul(int alpha, double2 C, double c0, double2 x) {
  return alpha == 0 ? cscale(x, c0) : (alpha > 0 ? cmul(C, x) : cmulc(x, C));
}

// ---------------------------------------------------------------------------------------------
// small DFT butterflies, sign SIGN: X_q = Σ_r v_r e^{SIGN 2πi rq/R}
// ---------------------------------------------------------------------------------------------
template <int SIGN>
__device__ __forceinline__ double2 rot90(double2 a) {  // a * (SIGN i)
  return SIGN > 0 ? cmuli(a) : cmulmi(a);
}

template <int SIGN>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int SIGN>
__device__ __forceinline__ void dft4(double2& v0, double2& v1, double2& v2, double2& v3) {
  double2 t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = rot90<SIGN>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v2 = csub(t0, t2);
  v1 = cadd(t1, t3);
  v3 = csub(t1, t3);
}

template <int SIGN>
__device__ __forceinline__ void dft8(double2* v) {
  const double s = 0.70710678118654752440084436210485;  // 1/sqrt(2)
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<SIGN>(e0, e1, e2, e3);
  dft4<SIGN>(o0, o1, o2, o3);
  // w8^q = e^{SIGN 2πi q/8}: q=1: s(1 + SIGN i), q=2: SIGN i, q=3: s(-1 + SIGN i)
  double2 t1 = make_double2(s * (o1.x - SIGN * o1.y), s * (o1.y + SIGN * o1.x));
  double2 t2 = rot90<SIGN>(o2);
  double2 t3 = make_double2(s * (-o3.x - SIGN * o3.y), s * (-o3.y + SIGN * o3.x));
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, t1);
  v[5] = csub(e1, t1);
  v[2] = cadd(e2, t2);
  v[6] = csub(e2, t2);
  v[3] = cadd(e3, t3);
  v[7] = csub(e3, t3);
}

template <int SIGN>
__device__ __forceinline__ void dft16(double2* v) {
  // radix-2 split of two 8-point DFTs: X_q = E_q + w16^q O_q, X_{q+8} = E_q - w16^q O_q
  const double c1 = 0.92387953251128675612818318939678829, s1 = 0.38268343236508977172845998403039887;
  const double h = 0.70710678118654752440084436210485;
  double2 e[8], o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    e[i] = v[2 * i];
    o[i] = v[2 * i + 1];
  }
  dft8<SIGN>(e);
  dft8<SIGN>(o);
  const double2 w[8] = {make_double2(1.0, 0.0),      make_double2(c1, SIGN * s1),  make_double2(h, SIGN * h),
                        make_double2(s1, SIGN * c1), make_double2(0.0, SIGN * 1.0), make_double2(-s1, SIGN * c1),
                        make_double2(-h, SIGN * h),  make_double2(-c1, SIGN * s1)};
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    double2 t;
    if (q == 0) t = o[0];
    else if (q == 4) t = rot90<SIGN>(o[4]);
    else t = cmul(o[q], w[q]);
    v[q] = cadd(e[q], t);
    v[q + 8] = csub(e[q], t);
  }
}

template <int R, int SIGN>
__device__ __forceinline__ void dftR(double2* v) {
  if constexpr (R == 2) dft2<SIGN>(v[0], v[1]);
  else if constexpr (R == 4) dft4<SIGN>(v[0], v[1], v[2], v[3]);
  else if constexpr (R == 8) dft8<SIGN>(v);
  else dft16<SIGN>(v);
}

// ---------------------------------------------------------------------------------------------
// Padded work-buffer layout: element i of a field lives at i + i/8, field stride NP = N + N/8.
// Every access pattern of the path (Stockham loads, the stride-R stores of the first pass,
// grid-point and mode loops) is then free of shared-memory bank conflicts for 16-byte elements.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ int pad(int i) { return i + (i >> 3); }
template <int N>
struct WL {
  static constexpr int NP = N + N / 8;
};

// ---------------------------------------------------------------------------------------------
// Stockham autosort FFT over the 3 fields of W (in place: load all, barrier, compute, store).
// Pass with radix R after NS = product of previous radices (natural order in and out):
//   for j in [0, N/R): k = j mod NS; v_r = W[j + r N/R] * w^{r k N/(NS R)}; DFT_R;
//                      W[(j/NS) NS R + k + r NS] = v_r.
// tw[m] = e^{-2πi m/N} (forward, SIGN=-1); the inverse (SIGN=+1) uses conj(tw).
// ---------------------------------------------------------------------------------------------
template <int N, int T, int R, int NS, int SIGN>
__device__ __forceinline__ void stockham_pass(double2* W, const double2* __restrict__ tw) {
  constexpr int NB = 3 * (N / R);  // butterflies over the 3 fields
  constexpr int BPT = (NB + T - 1) / T;
  double2 v[BPT][R];
#pragma unroll
  for (int i = 0; i < BPT; ++i) {
    const int b = threadIdx.x + i * T;
    if (NB % T == 0 || b < NB) {
      const int f = b / (N / R), j = b % (N / R);
      const double2* in = W + f * WL<N>::NP;
#pragma unroll
      for (int r = 0; r < R; ++r) v[i][r] = in[pad(j + r * (N / R))];
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < BPT; ++i) {
    const int b = threadIdx.x + i * T;
    if (NB % T == 0 || b < NB) {
      const int f = b / (N / R), j = b % (N / R);
      const int k = j % NS;
      if constexpr (NS > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const double2 w = __ldg(tw + r * k * (N / (NS * R)));
          v[i][r] = SIGN < 0 ? cmul(v[i][r], w) : cmulc(v[i][r], w);
        }
      }
      dftR<R, SIGN>(v[i]);
      double2* out = W + f * WL<N>::NP;
      const int base = (j / NS) * NS * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) out[pad(base + r * NS)] = v[i][r];
    }
  }
  __syncthreads();
}

// RMAX: largest radix (8: fewer shared-memory passes, best for throughput; 4: twice the threads,
// best for latency-bound launches such as the serial coarse sweep)
template <int N, int T, int SIGN, int RMAX, int NS = 1>
__device__ __forceinline__ void fft3(double2* W, const double2* __restrict__ tw) {
  if constexpr (NS < N) {
    constexpr int rem = N / NS;
    constexpr int R = (rem % RMAX == 0) ? RMAX : rem;
    stockham_pass<N, T, R, NS, SIGN>(W, tw);
    fft3<N, T, SIGN, RMAX, NS * R>(W, tw);
  }
}

// ---------------------------------------------------------------------------------------------
// Closed-form eigenbasis of L̂(κ) = [[0,-1,ia],[1,0,0],[ia,0,0]], a = κ/√F:
//   r^- = (-iω, 1, ia)/(√2ω),  r^0 = (0, ia, 1)/ω,  r^+ = (iω, 1, ia)/(√2ω),  ω = √(1+a²),
//   L̂ r^α = iαω r^α.  Per |κ| the host stores a, p = 1/(√2ω), q = 1/ω.
// ---------------------------------------------------------------------------------------------
struct ModeGeom {
  const double* a;  // |κ|/√F, |κ| = 0..K
  const double* p;  // 1/(√2 ω)
  const double* q;  // 1/ω
};

__device__ __forceinline__ int kappa_of(int j, int K) { return j <= K ? j : j - (2 * K + 1); }

// primitive (u0,u1,u2) -> eigen (c-, c0, c+) : c = R^H u
__device__ __forceinline__ void to_eigen(double as, double p, double q, const double2* u, double2* c) {
  const double s = 0.70710678118654752440084436210485;
  double2 t = cscale(csub(u[1], cmuli(cscale(u[2], as))), p);  // p (u1 - i a u2)
  double2 isu0 = cmuli(cscale(u[0], s));                          // i s u0
  c[0] = cadd(t, isu0);                                           // c-
  c[2] = csub(t, isu0);                                           // c+
  c[1] = cscale(csub(u[2], cmuli(cscale(u[1], as))), q);          // q (u2 - i a u1)
}

// eigen -> primitive : u = R c
__device__ __forceinline__ void to_prim(double as, double p, double q, const double2* c, double2* u) {
  const double s = 0.70710678118654752440084436210485;
  double2 d = csub(c[2], c[0]), e = cadd(c[2], c[0]);
  u[0] = cmuli(cscale(d, s));
  double2 pe = cscale(e, p), qc0 = cscale(c[1], q);
  u[1] = cadd(pe, cmuli(cscale(qc0, as)));
  u[2] = cadd(qc0, cmuli(cscale(pe, as)));
}

// ---------------------------------------------------------------------------------------------
// N(u) on the packed work buffer W (3 fields, full spectrum in, full spectrum out, unscaled):
//   in:  W[0] = v̂1, W[1] = iκ v̂2, W[2] = ĥ  (prepared by the caller's prologue)
//   out: W[f] = N * DFT(q_f),  q = (v1²/2, v1 v2x, h v1)   (products per real/imag lane)
// The caller's epilogue applies 1/N, the derivative factors (-iκ, -1, -iκ) and the 2/3 mask:
//   N(u) = -(∂x(v1²/2), v1 ∂x v2, ∂x(h v1))   (P:1090-1094 with R1; v1 v1x = ∂x(v1²/2))
// ---------------------------------------------------------------------------------------------
template <int N, int T, int RMAX>
__device__ __forceinline__ void nl_physical(double2* W, const double2* __restrict__ tw) {
  fft3<N, T, +1, RMAX>(W, tw);  // synthesis: u(x_n) = Σ_κ Z_κ e^{iκ x_n}
  constexpr int NP = WL<N>::NP;
  for (int n = threadIdx.x; n < N; n += T) {
    const int i = pad(n);
    const double2 v1 = W[i], v2x = W[NP + i], h = W[2 * NP + i];
    W[i] = make_double2(0.5 * v1.x * v1.x, 0.5 * v1.y * v1.y);
    W[NP + i] = make_double2(v1.x * v2x.x, v1.y * v2x.y);
    W[2 * NP + i] = make_double2(h.x * v1.x, h.y * v1.y);
  }
  __syncthreads();
  fft3<N, T, -1, RMAX>(W, tw);  // analysis (unnormalised)
}

// prologue helper: write prim(x) of entry j into W as the N-eval input (v1, iκ v2, h)
template <int N>
__device__ __forceinline__ void put_input(double2* W, int k_full, double kap, const double2* u) {
  constexpr int NP = WL<N>::NP;
  const int i = pad(k_full);
  W[i] = u[0];
  W[NP + i] = cmuli(cscale(u[1], kap));
  W[2 * NP + i] = u[2];
}

// epilogue helper: read the N-eval output of entry k_full, return N̂ (primitive)
template <int N>
__device__ __forceinline__ void get_output(const double2* W, int k_full, double kap, double invN, double2* nh) {
  constexpr int NP = WL<N>::NP;
  const int i = pad(k_full);
  const double2 Q0 = cscale(W[i], invN), Q1 = cscale(W[NP + i], invN), Q2 = cscale(W[2 * NP + i], invN);
  nh[0] = cmulmi(cscale(Q0, kap));  // -iκ Q0
  nh[1] = make_double2(-Q1.x, -Q1.y);
  nh[2] = cmulmi(cscale(Q2, kap));  // -iκ Q2
}

// zero the non-retained full-spectrum entries K < k < N-K of the 3 fields
template <int N, int T>
__device__ __forceinline__ void zero_tail(double2* W) {
  constexpr int K = N / 3, NZ = N - (2 * K + 1);
  for (int i = threadIdx.x; i < 3 * NZ; i += T) {
    const int f = i / NZ, k = K + 1 + i % NZ;
    W[f * WL<N>::NP + pad(k)] = make_double2(0.0, 0.0);
  }
}

__device__ __forceinline__ int full_index(int kap, int N) { return kap >= 0 ? kap : kap + N; }

}  // namespace rsw
