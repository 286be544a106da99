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
//  * Work buffer W: nl_core's padded buffer (fields v1, v2, h at stride N + N/R, then the v1 copy) —
//    full spectrum or physical grid (digit-reversed order between the transforms).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rsw {

// Debug build only (-DRSW_PHASE_PROF, e.g. tools/build_variant.py): cycles of the N-eval phases seen by
// thread 0 of CTA 0 (0 = between N-evals, i.e. the epilogue, 1 = inverse FFT, 2 = products and the
// first analysis pass, 3 = the other analysis passes), printed per launch by k_fine.
#ifdef RSW_PHASE_PROF
static __device__ unsigned long long g_phase[8];
#define RSW_PHASE(i)                                                 \
  do {                                                               \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                       \
      const unsigned long long c_ = clock64();                       \
      if (g_phase[7]) g_phase[i] += c_ - g_phase[7];                 \
      g_phase[7] = c_;                                               \
    }                                                                \
  } while (0)
#else
#define RSW_PHASE(i) \
  do {               \
  } while (0)
#endif

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

// e ± o·w for a compile-time twiddle w = (c, σ) in FMA form (6 DP instructions instead of a complex
// multiply plus two complex adds): o·w = f·u with u = o + i (σ/c) o, f = c when |c| >= |σ|, or
// u = (c/σ) o + i o, f = σ otherwise (the ratio is <= 1 in magnitude), then e ± f u by FMAs.
template <int SIGN>
__device__ __forceinline__ void tw_butterfly(double2& lo, double2& hi, const double2 e, const double2 o, const double c,
                                             const double sg) {
  const bool cf = (c >= 0 ? c : -c) >= (sg >= 0 ? sg : -sg);
  double2 u;
  double f;
  if (cf) {
    const double r = sg / c;
    u = make_double2(fma(-r, o.y, o.x), fma(r, o.x, o.y));
    f = c;
  } else {
    const double r = c / sg;
    u = make_double2(fma(r, o.x, -o.y), fma(r, o.y, o.x));
    f = sg;
  }
  lo = make_double2(fma(f, u.x, e.x), fma(f, u.y, e.y));
  hi = make_double2(fma(-f, u.x, e.x), fma(-f, u.y, e.y));
}

template <int SIGN>
__device__ __forceinline__ void dft8(double2* v) {
  const double s = 0.70710678118654752440084436210485;  // 1/sqrt(2)
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<SIGN>(e0, e1, e2, e3);
  dft4<SIGN>(o0, o1, o2, o3);
  // w8^q = e^{SIGN 2πi q/8}: q=1: s(1 + SIGN i), q=2: SIGN i, q=3: s(-1 + SIGN i); the factor s is
  // applied by the FMAs of the output pair
  const double2 u1 = make_double2(o1.x - SIGN * o1.y, o1.y + SIGN * o1.x);
  const double2 u3 = make_double2(-o3.x - SIGN * o3.y, -o3.y + SIGN * o3.x);
  const double2 t2 = rot90<SIGN>(o2);
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = make_double2(fma(s, u1.x, e1.x), fma(s, u1.y, e1.y));
  v[5] = make_double2(fma(-s, u1.x, e1.x), fma(-s, u1.y, e1.y));
  v[2] = cadd(e2, t2);
  v[6] = csub(e2, t2);
  v[3] = make_double2(fma(s, u3.x, e3.x), fma(s, u3.y, e3.y));
  v[7] = make_double2(fma(-s, u3.x, e3.x), fma(-s, u3.y, e3.y));
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
  // w16^q = (cos, SIGN sin)(2π q/16)
  const double cs[8] = {1.0, c1, h, s1, 0.0, -s1, -h, -c1};
  const double sn[8] = {0.0, s1, h, c1, 1.0, c1, h, s1};
  v[0] = cadd(e[0], o[0]);
  v[8] = csub(e[0], o[0]);
  {
    const double2 t = rot90<SIGN>(o[4]);
    v[4] = cadd(e[4], t);
    v[12] = csub(e[4], t);
  }
#pragma unroll
  for (int q = 1; q < 8; ++q)
    if (q != 4) tw_butterfly<SIGN>(v[q], v[q + 8], e[q], o[q], cs[q], SIGN * sn[q]);
}

template <int SIGN>
__device__ __forceinline__ void dft32(double2* v) {
  // radix-2 split of two 16-point DFTs: X_q = E_q + w32^q O_q, X_{q+16} = E_q - w32^q O_q
  double2 e[16], o[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    e[i] = v[2 * i];
    o[i] = v[2 * i + 1];
  }
  dft16<SIGN>(e);
  dft16<SIGN>(o);
  // cos / sin (2π q/32), q = 0..8
  const double c[9] = {1.0,
                       0.98078528040323044912618223613424,
                       0.92387953251128675612818318939679,
                       0.83146961230254523707878837761791,
                       0.70710678118654752440084436210485,
                       0.55557023301960222474283081394853,
                       0.38268343236508977172845998403040,
                       0.19509032201612826784828486847702,
                       0.0};
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    double2 t;
    if (q == 0) t = o[0];
    else if (q == 8) t = rot90<SIGN>(o[8]);
    else {
      // w32^q = e^{SIGN 2πi q/32} = (cos, SIGN sin); for q > 8 use cos(θ) = -sin(θ - π/2) symmetry
      const double cr = q <= 8 ? c[q] : -c[16 - q];
      const double si = q <= 8 ? c[8 - q] : c[q - 8];
      t = cmul(o[q], make_double2(cr, SIGN * si));
    }
    v[q] = cadd(e[q], t);
    v[q + 16] = csub(e[q], t);
  }
}

template <int R, int SIGN>
__device__ __forceinline__ void dftR(double2* v) {
  if constexpr (R == 2) dft2<SIGN>(v[0], v[1]);
  else if constexpr (R == 4) dft4<SIGN>(v[0], v[1], v[2], v[3]);
  else if constexpr (R == 8) dft8<SIGN>(v);
  else if constexpr (R == 16) dft16<SIGN>(v);
  else dft32<SIGN>(v);
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

// thread-group policies: the whole CTA, or a warp-aligned group of a CTA with its own named barrier
// fbar(): first of three named barriers the FFT core may use per field (0: none, use the group barrier)
struct CtaGroup {
  __device__ __forceinline__ int base() const { return 0; }
  __device__ __forceinline__ int tid() const { return threadIdx.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  __device__ __forceinline__ bool sync_or(bool p) const { return __syncthreads_or(p) != 0; }
  __device__ __forceinline__ int fbar() const { return 1; }  // ids 1..3 (kernels whose whole CTA is one group)
  __device__ __forceinline__ int ftid() const { return threadIdx.x; }
};
struct NamedGroup {
  int b0, id, nthr;  // first thread, barrier id (1..15), thread count (multiple of 32)
  int fb = 0;        // per-field barrier ids fb..fb+2, or 0
  int wsw = 0;       // FFT roles with the group's warps 2 and 3 exchanged (ftid)
  __device__ __forceinline__ int base() const { return b0; }
  __device__ __forceinline__ int tid() const { return threadIdx.x - b0; }
  // thread index of the FFT core's (field, column) roles: tid(), or with warps 2 and 3 exchanged, which
  // moves the third field's warp to the SM sub-partition the group would otherwise leave without FFT work
  // (warp w issues on sub-partition w mod 4; used by the pipelined schedule's fine group, whose CTA
  // neighbours are the coarse parts)
  __device__ __forceinline__ int ftid() const {
    const int t = tid();
    return (wsw && (t >> 6) == 1) ? (t ^ 32) : t;
  }
  __device__ __forceinline__ void sync() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthr) : "memory"); }
  // barrier that also ORs a predicate over the group's threads
  __device__ __forceinline__ bool sync_or(bool p) const {
    unsigned r;
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n bar.red.or.pred q, %2, %3, q;\n selp.u32 %0, 1, 0, q;\n}"
        : "=r"(r)
        : "r"((unsigned)p), "r"(id), "r"(nthr)
        : "memory");
    return r != 0;
  }
  __device__ __forceinline__ int fbar() const { return fb; }
};

// Padded storage of the FFT buffers: element e of a field lives at fpad(e) = e + e / R (one pad slot
// per R elements), fields FS = N + N/R apart; nl_core's buffer is X[3 FS] followed by V[FS].  The
// pad is conflict-free for every pass of the plans below at R >= 8 (quarter-warp of 8 threads on 8
// distinct 16-byte bank groups; tools/fft_model.py) and it is additive over disjoint bit fields:
// a butterfly's elements e0 + d s have e0 and d s in disjoint bits, so fpad(e0 + d s) =
// fpad(e0) + fpad(d s) — one base register per butterfly plus compile-time immediate offsets.
template <int R>
__host__ __device__ __forceinline__ constexpr int fpad(int e) {
  return e + (e >> (R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : R == 16 ? 4 : 5));
}
template <int N, int R>
__host__ __device__ constexpr int fft_fs() { return N + N / R; }
template <int N, int R>
__host__ __device__ constexpr int nl_buf() { return 4 * fft_fs<N, R>(); }  // X (3 fields) + V

// ---------------------------------------------------------------------------------------------
// In-place mixed-radix FFT core (nl_core).  Plan for (N, R): pass 0 has radix rem = N / R^a when
// N is not a power of R, every other pass radix R (1024 = 4.16.16, 512 = 2.16.16, 256 = 16.16 at
// R = 16).  Pass p works on blocks of length L_p = N / (r_0 ... r_{p-1}) with stride d_p = L_p / r_p:
// butterfly b = (block, k1) = divmod(b, d_p) owns the elements block·L_p + k1 + d_p·s, s < r_p.
//  * synthesis (inverse transform, sign +): decimation in frequency (Gentleman–Sande) — r-point DFT,
//    then the twiddles ω_L^{s k1} — written back to the positions it was read from.  The grid
//    values come out in digit-reversed order, which the pointwise products do not care about;
//  * analysis (forward transform, sign −): the conjugate transpose, passes in reverse order —
//    twiddles e^{-2πi s k1/L} on the inputs, then the r-point DFT, again in place — which returns
//    the natural spectral order.  No reordering pass is ever needed.
// Because a butterfly writes back exactly the elements it read, a pass needs no barrier between its
// loads and its stores: ONE barrier per pass and a single buffer of 3N values (plus N for the v1
// copy of the products).  Thread t of the group owns field f = t / (N/R) and column j = t mod (N/R);
// its butterflies in a pass of radix r are b = j + i N/R, i < R/r.  Storage: the padded layout fpad
// (below), conflict-free for every pass of these plans at R >= 8.
// ---------------------------------------------------------------------------------------------
template <int N, int R>
__host__ __device__ constexpr int fft_npass() {
  int a = 0, x = 1;
  while (x * R <= N) {
    x *= R;
    ++a;
  }
  return (N / x > 1) ? a + 1 : a;
}
template <int N, int R>
__host__ __device__ constexpr int fft_rad(int p) {
  int x = 1;
  while (x * R <= N) x *= R;
  return (N / x > 1 && p == 0) ? N / x : R;
}
template <int N, int R>
__host__ __device__ constexpr int fft_len(int p) {  // block length L_p
  int L = N;
  for (int q = 0; q < p; ++q) L /= fft_rad<N, R>(q);
  return L;
}
// Twiddles of pass p: radix >= 8 passes of the large transforms (N >= 512) read every power from a
// full table TW[off_p + (s-1) d_p + k1] = e^{-2πi s k1 / L_p}, s = 1..r-1 (exact table values, one
// shared-memory load per twiddle instead of forming the 15 powers of a radix-16 butterfly in
// registers: ~60 DP instructions per butterfly, ~20% of the transform); the other passes store the
// bases e^{-2πi k1 / L_p} only and form the powers in registers (small radices, or the latency-bound
// small transforms, where the product chain was measured faster than the loads).
#ifndef RSW_TW_FULL_MIN_N
#define RSW_TW_FULL_MIN_N 512  // smallest transform whose radix >= 8 passes keep a full twiddle table
#endif
template <int N, int R>
__host__ __device__ constexpr bool fft_tw_full(int p) { return N >= RSW_TW_FULL_MIN_N && fft_rad<N, R>(p) >= 8; }
template <int N, int R>
__host__ __device__ constexpr int fft_tw_len(int p) {  // table entries of pass p (last pass: none)
  return (p >= fft_npass<N, R>() - 1) ? 0
         : (fft_tw_full<N, R>(p) ? (fft_rad<N, R>(p) - 1) : 1) * (fft_len<N, R>(p) / fft_rad<N, R>(p));
}
template <int N, int R>
__host__ __device__ constexpr int fft_tw_off(int p) {  // offset of pass p's twiddles
  int o = 0;
  for (int q = 0; q < p; ++q) o += fft_tw_len<N, R>(q);
  return o;
}
// size of the twiddle table for the passes p < m-1 (the last pass has d = 1 and no twiddles)
template <int N, int R>
__host__ __device__ constexpr int fft_tw_size() { return fft_tw_off<N, R>(fft_npass<N, R>() - 1) > 0 ? fft_tw_off<N, R>(fft_npass<N, R>() - 1) : 1; }

// Twiddle source of pass p for a kernel's policy TWT (only passes with a full table differ):
//   0 = powers formed in registers from the base (the s = 1 row of the full table),
//   1 = the full shared-memory table,
//   2 = the full table copied once into the thread's own TMEM lane (passes of radix R: each thread has
//       ONE butterfly there, so its r-1 twiddles are fixed for the whole kernel) — loaded with
//       tcgen05.ld, which takes those reads off the shared-memory pipe (the binding resource of the
//       n = 1024 fine kernel: 81% of peak wavefronts with the smem table, 72% with register powers).
template <int N, int R, int TWT>
__host__ __device__ constexpr int fft_tw_src(int p) {
  return (p >= fft_npass<N, R>() - 1 || !fft_tw_full<N, R>(p)) ? 0
         : (TWT == 2 && fft_rad<N, R>(p) == R) ? 2 : (TWT == 0 ? 0 : 1);
}
// TMEM columns of pass p's twiddles (chunks of 3 complex = 12 columns) and their total
template <int N, int R>
__host__ __device__ constexpr int fft_tw_tcol(int p) {
  int o = 0;
  for (int q = 0; q < p; ++q)
    if (fft_tw_src<N, R, 2>(q) == 2) o += (fft_rad<N, R>(q) + 1) / 3 * 12;
  return o;
}
template <int N, int R>
__host__ __device__ constexpr int fft_tw_tcols() { return fft_tw_tcol<N, R>(fft_npass<N, R>()); }

// fill the twiddle table from the plain table tw[m] = e^{-2πi m/N} (threads t0, t0 + T, ...)
template <int N, int R, int T>
__device__ __forceinline__ void fill_packed_twiddles(double2* TW, const double2* __restrict__ tw, int t0 = -1, int nthr = T) {
  constexpr int m = fft_npass<N, R>();
  for (int i = (t0 < 0 ? (int)threadIdx.x : t0); i < fft_tw_off<N, R>(m - 1); i += nthr) {
    int p = 0;
    while (p < m - 2 && i >= fft_tw_off<N, R>(p + 1)) ++p;
    const int li = i - fft_tw_off<N, R>(p), L = fft_len<N, R>(p), d = L / fft_rad<N, R>(p);
    const int sk = fft_tw_full<N, R>(p) ? (li / d + 1) * (li % d) : li;  // s k1 (< L)
    TW[i] = __ldg(tw + sk * (N / L));
  }
}

__device__ __forceinline__ double2 csqr(double2 a) {  // a^2
  return make_double2(fma(a.x, a.x, -a.y * a.y), (a.x + a.x) * a.y);
}

// v[s] *= w^s (CONJ: conj(w)^s), s = 1..r-1, for a twiddle base w read from the shared table; the
// powers are formed in registers as they are needed (w^2 = w·w, w^3 = w^2·w, w^4 = (w^2)^2, ...,
// w^{8+s} = w^8·w^s: at most 5 roundings deep, error ≲ 5 ulp): the shared-memory pipe is the binding
// resource of the FFT core (ncu, n = 1024: 80% of peak wavefronts, twiddle loads ~23% of them),
// while the FP64 pipe has room.
// v[s] *= TWs[(s-1) d] (CONJ: its conjugate), s = 1..r-1: full-table twiddles of one butterfly
template <int r, bool CONJ>
__device__ __forceinline__ void apply_twiddles_tab(double2* v, const double2* TWs, int d) {
#pragma unroll
  for (int s = 1; s < r; ++s) v[s] = CONJ ? cmulc(v[s], TWs[(s - 1) * d]) : cmul(v[s], TWs[(s - 1) * d]);
}

// TMEM twiddles: chunk c of a pass's slot holds s = 3c+1 .. 3c+3 (12 columns); loads are issued one
// chunk ahead of their use.  The wait names the chunk's registers as in/out operands, so no use of
// them can be scheduled before the asynchronous load completed.
__device__ __forceinline__ void tmem_ld12_issue(uint32_t ta, uint32_t (&r)[12]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(ta)
      : "memory");
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
               : "r"(ta + 8)
               : "memory");
}
__device__ __forceinline__ void tmem_wait12(uint32_t (&r)[12]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11])
               :
               : "memory");
}
template <int r, bool CONJ>
__device__ __forceinline__ void apply_twiddles_tmem(double2* v, uint32_t ta) {
  constexpr int NCH = (r + 1) / 3;  // chunks covering s = 1..r-1
  uint32_t ca[12], cb[12];
  tmem_ld12_issue(ta, ca);
  tmem_wait12(ca);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    uint32_t(&cur)[12] = (c & 1) ? cb : ca;
    uint32_t(&nxt)[12] = (c & 1) ? ca : cb;
    if (c + 1 < NCH) tmem_ld12_issue(ta + 12 * (c + 1), nxt);
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int sidx = 3 * c + 1 + u;
      if (sidx < r) {
        const double2 w = make_double2(__hiloint2double(cur[4 * u + 1], cur[4 * u]), __hiloint2double(cur[4 * u + 3], cur[4 * u + 2]));
        v[sidx] = CONJ ? cmulc(v[sidx], w) : cmul(v[sidx], w);
      }
    }
    if (c + 1 < NCH) tmem_wait12(nxt);
  }
}

template <int r, bool CONJ>
__device__ __forceinline__ void apply_twiddles(double2* v, const double2 w1) {
#define TWM(s, w) v[s] = CONJ ? cmulc(v[s], w) : cmul(v[s], w)
  if constexpr (r >= 2) TWM(1, w1);
  if constexpr (r >= 4) {
    const double2 w2 = csqr(w1), w3 = cmul(w2, w1);
    TWM(2, w2);
    TWM(3, w3);
    if constexpr (r >= 8) {
      const double2 w4 = csqr(w2), w5 = cmul(w4, w1), w6 = csqr(w3), w7 = cmul(w4, w3);
      TWM(4, w4);
      TWM(5, w5);
      TWM(6, w6);
      TWM(7, w7);
      if constexpr (r >= 16) {
        const double2 w8 = csqr(w4);
        const double2 ws[8] = {make_double2(1.0, 0.0), w1, w2, w3, w4, w5, w6, w7};
        TWM(8, w8);
#pragma unroll
        for (int s = 9; s < 16; ++s) TWM(s, cmul(w8, ws[s - 8]));
        static_assert(r <= 16, "apply_twiddles: radix <= 16");
      }
    }
  }
#undef TWM
}

template <int N, int R, int p>
__device__ __forceinline__ int fft_elem0(int b) {  // first element of butterfly b in pass p
  constexpr int L = fft_len<N, R>(p), d = L / fft_rad<N, R>(p);
  return (b / d) * L + (b % d);
}

// Synchronisation between two passes of the SAME field: every pass touches only its own field's
// buffer, so when a field's N/R threads lie inside one warp (N/R divides 32) a warp barrier orders the
// passes; otherwise the group barrier.  Called by every thread of the group (also the inactive ones,
// which may share a warp with active ones), so __syncwarp always sees the full warp.
// Fields spanning several whole warps (N/R = 64, 128) synchronise on a named barrier of their own
// N/R threads when the group provides per-field barrier ids (the three fields then run their passes
// independently); the threads outside the three fields (act = false) skip it.
template <int N, int R, class GRP>
__device__ __forceinline__ void pass_sync(const GRP& grp, int f = 0, bool act = true) {
  constexpr int NJ = N / R;
  if constexpr (NJ <= 32 && 32 % NJ == 0) {
    __syncwarp();
  } else if constexpr (NJ % 32 == 0) {
    if (grp.fbar() > 0) {
      if (act) asm volatile("bar.sync %0, %1;" ::"r"(grp.fbar() + f), "r"(NJ) : "memory");
    } else {
      grp.sync();
    }
  } else {
    grp.sync();
  }
}

// synthesis passes p..m-1 of field buffer Xf (sign +); the last pass leaves its outputs in v
template <int N, int R, int p, int TWT, class GRP>
__device__ __forceinline__ void core_inverse(double2 (&v)[R], double2* Xf, int j, bool act, const double2* TW,
                                             uint32_t twt, const GRP& grp, int f) {
  constexpr int m = fft_npass<N, R>(), r = fft_rad<N, R>(p), L = fft_len<N, R>(p), d = L / r, NJ = N / R;
  constexpr int K = N / 3;
  if (act) {
#pragma unroll
    for (int i = 0; i < R / r; ++i) {
      const int b = j + i * NJ, e0 = fft_elem0<N, R, p>(b);
      const double2* xb = Xf + fpad<R>(e0);
#pragma unroll
      for (int s = 0; s < r; ++s) {
        const int e = e0 + d * s;
        if constexpr (p == 0) v[i * r + s] = (e <= K || e >= N - K) ? xb[fpad<R>(d * s)] : make_double2(0.0, 0.0);  // R10
        else v[i * r + s] = xb[fpad<R>(d * s)];
      }
      dftR<r, +1>(&v[i * r]);
      if constexpr (p < m - 1) {
        if constexpr (fft_tw_src<N, R, TWT>(p) == 2) apply_twiddles_tmem<r, true>(&v[i * r], twt + fft_tw_tcol<N, R>(p));
        else if constexpr (fft_tw_src<N, R, TWT>(p) == 1)
          apply_twiddles_tab<r, true>(&v[i * r], TW + fft_tw_off<N, R>(p) + (b % d), d);
        else apply_twiddles<r, true>(&v[i * r], TW[fft_tw_off<N, R>(p) + (b % d)]);  // ω_L^{+s k1}
#pragma unroll
        for (int s = 0; s < r; ++s) Xf[fpad<R>(e0) + fpad<R>(d * s)] = v[i * r + s];
      }
    }
  }
  if constexpr (p < m - 1) {
    pass_sync<N, R>(grp, f, act);
    core_inverse<N, R, p + 1, TWT>(v, Xf, j, act, TW, twt, grp, f);
  }
}

// analysis passes p, p-1, ..., 0 (sign -); pass 0 stores the retained modes only
template <int N, int R, int p, int TWT, class GRP>
__device__ __forceinline__ void core_forward(double2 (&v)[R], double2* Xf, int j, bool act, const double2* TW,
                                             uint32_t twt, const GRP& grp, int f) {
  if constexpr (p >= 0) {
    constexpr int r = fft_rad<N, R>(p), L = fft_len<N, R>(p), d = L / r, NJ = N / R;
    constexpr int K = N / 3;
    if (act) {
#pragma unroll
      for (int i = 0; i < R / r; ++i) {
        const int b = j + i * NJ, e0 = fft_elem0<N, R, p>(b);
        double2* xb = Xf + fpad<R>(e0);
#pragma unroll
        for (int s = 0; s < r; ++s) v[i * r + s] = xb[fpad<R>(d * s)];
        if constexpr (fft_tw_src<N, R, TWT>(p) == 2) apply_twiddles_tmem<r, false>(&v[i * r], twt + fft_tw_tcol<N, R>(p));
        else if constexpr (fft_tw_src<N, R, TWT>(p) == 1)
          apply_twiddles_tab<r, false>(&v[i * r], TW + fft_tw_off<N, R>(p) + (b % d), d);
        else apply_twiddles<r, false>(&v[i * r], TW[fft_tw_off<N, R>(p) + (b % d)]);  // e^{-2πi s k1/L}
        dftR<r, -1>(&v[i * r]);
#pragma unroll
        for (int s = 0; s < r; ++s) {
          const int e = e0 + d * s;
          if (p > 0 || e <= K || e >= N - K) xb[fpad<R>(d * s)] = v[i * r + s];
        }
      }
    }
    if constexpr (p > 0) pass_sync<N, R>(grp, f, act);  // the next pass reads this field only
    else grp.sync();                                     // exit: the caller reads every field
    core_forward<N, R, p - 1, TWT>(v, Xf, j, act, TW, twt, grp, f);
  }
}

// N(u) core on the packed pair: X = double2[nl_buf<N, R>()] — fields (v1, i κ v2, h) at f FS in the
// padded layout, then V (the v1 copy) at 3 FS — holds the retained spectra of (v1, iκ v2, h) on entry
// and the retained spectra of (v1²/2, v1 v2x, h v1) (unnormalised) on exit.  The second argument is
// unused (kept for the callers' layouts, which reserve >= nl_buf entries from X).  Group barriers: the
// v1 copy before the products and the exit; between passes of a field a warp barrier when the field
// lies in one warp (N/R <= 32: n <= 256), else a group barrier (2m in all).  TWT: twiddle policy (fft_tw_src); with TWT = 2, twt is the
// thread's TMEM address of its twiddle slots (lane quarter + column base, filled by tw_tmem_fill).
template <int N, int R, int T, class GRP = CtaGroup, int TWT = 0>
__device__ __forceinline__ void nl_core(double2* X, double2* /*unused*/, const double2* TW, const GRP& grp = GRP(),
                                        uint32_t twt = 0) {
  static_assert(T >= 3 * (N / R), "nl_core: T must cover 3 N/R field-columns");
  constexpr int m = fft_npass<N, R>(), NJ = N / R, K = N / 3;
  constexpr int rl = fft_rad<N, R>(m - 1), Ll = fft_len<N, R>(m - 1), dl = Ll / rl;
  static_assert(dl == 1 && rl == R, "nl_core: the last pass must have radix R and stride 1");
  const int t = grp.ftid();
  const int f = t / NJ, j = t % NJ;
  const bool act = t < 3 * NJ;
  constexpr int FS = fft_fs<N, R>();
  double2* Xf = X + (act ? f : 0) * FS;
  double2* V = X + 3 * FS + fpad<R>(j * R);
  double2 v[R];
  RSW_PHASE(0);
  core_inverse<N, R, 0, TWT>(v, Xf, j, act, TW, twt, grp, f);
  RSW_PHASE(1);
  // grid products (R1, R10): the last synthesis pass left the grid values of positions j R + s in
  // registers; v1 is shared with the v2x / h threads through V
  if (act && f == 0) {
#pragma unroll
    for (int s = 0; s < R; ++s) V[fpad<R>(s)] = v[s];
  }
  grp.sync();
  if (act) {
    if (f == 0) {
#pragma unroll
      for (int s = 0; s < R; ++s) v[s] = make_double2(0.5 * v[s].x * v[s].x, 0.5 * v[s].y * v[s].y);
    } else {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const double2 v1 = V[fpad<R>(s)];
        v[s] = make_double2(v1.x * v[s].x, v1.y * v[s].y);
      }
    }
    // analysis pass m-1: stride 1, no twiddles, operands already in registers
    dftR<R, -1>(v);
    double2* xb = Xf + fpad<R>(j * R);
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int e = j * R + s;
      if (m > 1 || e <= K || e >= N - K) xb[fpad<R>(s)] = v[s];
    }
  }
  if constexpr (m > 1) pass_sync<N, R>(grp, f, act);  // analysis pass m-1 wrote its own field only
  else grp.sync();
  RSW_PHASE(2);
  core_forward<N, R, m - 2, TWT>(v, Xf, j, act, TW, twt, grp, f);
  RSW_PHASE(3);
}

// N-eval input / output of one retained entry in the padded layout of nl_core
template <int N, int R>
__device__ __forceinline__ void put_input_z(double2* X, int k_full, double kap, const double2* u) {
  constexpr int FS = fft_fs<N, R>();
  const int i = fpad<R>(k_full);
  X[i] = u[0];
  X[FS + i] = cmuli(cscale(u[1], kap));
  X[2 * FS + i] = u[2];
}
template <int N, int R>
__device__ __forceinline__ void get_output_z(const double2* X, int k_full, double kap, double invN, double2* nh) {
  constexpr int FS = fft_fs<N, R>();
  const int i = fpad<R>(k_full);
  const double2 Q0 = cscale(X[i], invN), Q1 = cscale(X[FS + i], invN), Q2 = cscale(X[2 * FS + i], invN);
  nh[0] = cmulmi(cscale(Q0, kap));  // -iκ Q0
  nh[1] = make_double2(-Q1.x, -Q1.y);
  nh[2] = cmulmi(cscale(Q2, kap));  // -iκ Q2
}

// The same two maps fused with the eigenbasis change (per mode: 14 DP instructions plus 4-5
// scalar products instead of ~32 / ~20): the FFT output of a retained entry straight into eigen
// coordinates, nn = R^H diag(-iκ, -1, -iκ) Z / N, i.e. (with as = κ/√F, s = 1/√2)
//   c∓ = -(p/N)(Z1 + as κ Z2) ± (s κ/N) Z0,   c0 = -i (q/N)(κ Z2 - as Z1);
// and an eigen state into the FFT input, (u0, iκ u1, u2) with u = R c, i.e. with d = c+ - c-,
// e = c+ + c-:  X0 = i s d,  X1 = iκ p e - κ as q c0,  X2 = q c0 + i as p e.
// the map on raw (unnormalised) FFT outputs X0..X2 of one entry, with the normalisation `scale` (1/N,
// or 1/(2N) for the unpacked half-sums of the coarse sample pairs)
__device__ __forceinline__ void eigen_from_raw(const double2 X0, const double2 X1, const double2 X2, double kap,
                                               double as, double p, double q, double scale, double2* nn) {
  const double ak = as * kap, sk = 0.70710678118654752440084436210485 * scale * kap, pn = p * scale, qn = q * scale;
  const double2 T = make_double2(fma(ak, X2.x, X1.x), fma(ak, X2.y, X1.y));
  const double2 A = make_double2(sk * X0.x, sk * X0.y);
  nn[0] = make_double2(fma(-pn, T.x, A.x), fma(-pn, T.y, A.y));
  nn[2] = make_double2(fma(-pn, T.x, -A.x), fma(-pn, T.y, -A.y));
  const double2 W = make_double2(fma(kap, X2.x, -as * X1.x), fma(kap, X2.y, -as * X1.y));
  nn[1] = make_double2(qn * W.y, -qn * W.x);
}
template <int N, int R>
__device__ __forceinline__ void get_output_eigen(const double2* X, int k_full, double kap, double as, double p,
                                                 double q, double2* nn) {
  constexpr int FS = fft_fs<N, R>();
  const int i = fpad<R>(k_full);
  eigen_from_raw(X[i], X[FS + i], X[2 * FS + i], kap, as, p, q, 1.0 / N, nn);
}
template <int N, int R>
__device__ __forceinline__ void put_input_eigen(double2* X, int k_full, double kap, double as, double p, double q,
                                                const double2* c) {
  constexpr int FS = fft_fs<N, R>();
  constexpr double s = 0.70710678118654752440084436210485;
  const int i = fpad<R>(k_full);
  const double2 d = csub(c[2], c[0]), e = cadd(c[2], c[0]);
  const double kp = kap * p, kaq = kap * as * q, ap = as * p;
  X[i] = make_double2(-s * d.y, s * d.x);
  X[FS + i] = make_double2(fma(-kp, e.y, -kaq * c[1].x), fma(kp, e.x, -kaq * c[1].y));
  X[2 * FS + i] = make_double2(fma(q, c[1].x, -ap * e.y), fma(q, c[1].y, ap * e.x));
}

// ---------------------------------------------------------------------------------------------
// Tensor memory (TMEM, 512 columns x 128 lanes x 32 bit per SM) used as thread-private storage
// for the per-mode integrator state: a warp reaches the 32 lanes 32 (warp % 4) .. +31 of its
// quarter, each thread its own lane, so a (lane, column range) slot is private to one thread.
// This frees the shared memory the state would take (98 KB per CTA at n = 1024) for the
// coefficient / twiddle tables.  Shape 32x32b: thread i of the warp moves consecutive 32-bit
// columns of lane base + i.  All tcgen05 ops below are warp-collective (.sync.aligned).
// ---------------------------------------------------------------------------------------------
template <int C>
__host__ __device__ constexpr int tmem_cols_pow2() {
  return C <= 32 ? 32 : C <= 64 ? 64 : C <= 128 ? 128 : C <= 256 ? 256 : 512;
}
template <int NCOL>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {  // by one whole warp
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(slot);
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s), "n"(NCOL) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOL>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // by the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOL) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// one complex double = 4 columns; load / store 3 complex (12 columns) starting at taddr
__device__ __forceinline__ void tmem_ld3(uint32_t taddr, double2 (&x)[3]) {
  uint32_t r[12];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
               : "r"(taddr + 8)
               : "memory");
  tmem_wait_ld();
#pragma unroll
  for (int a = 0; a < 3; ++a)
    x[a] = make_double2(__hiloint2double(r[4 * a + 1], r[4 * a]), __hiloint2double(r[4 * a + 3], r[4 * a + 2]));
}
// two 3-complex slots with ONE wait (the second load's latency overlaps the first's)
__device__ __forceinline__ void tmem_ld3x2(uint32_t ta, double2 (&x)[3], uint32_t tb, double2 (&y)[3]) {
  uint32_t r[12], q[12];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(ta)
      : "memory");
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
               : "r"(ta + 8)
               : "memory");
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7])
      : "r"(tb)
      : "memory");
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11])
               : "r"(tb + 8)
               : "memory");
  tmem_wait_ld();
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    x[a] = make_double2(__hiloint2double(r[4 * a + 1], r[4 * a]), __hiloint2double(r[4 * a + 3], r[4 * a + 2]));
    y[a] = make_double2(__hiloint2double(q[4 * a + 1], q[4 * a]), __hiloint2double(q[4 * a + 3], q[4 * a + 2]));
  }
}
__device__ __forceinline__ void tmem_st3(uint32_t taddr, const double2 (&x)[3]) {
  uint32_t r[12];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    r[4 * a] = __double2loint(x[a].x);
    r[4 * a + 1] = __double2hiint(x[a].x);
    r[4 * a + 2] = __double2loint(x[a].y);
    r[4 * a + 3] = __double2hiint(x[a].y);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr + 8), "r"(r[8]),
               "r"(r[9]), "r"(r[10]), "r"(r[11])
               : "memory");
}

// Copy this thread's TMEM-sourced twiddles (fft_tw_src == 2: radix-R passes, one butterfly b = j per
// thread) from the staged shared-memory table into its own TMEM lane at twt.  Warp-collective: every
// thread of the warp calls it.  Warps sharing a lane quarter write their lanes with the same values
// in the layouts used (k1 = j mod d depends on the lane only, or on a column half the quarter fixes).
template <int N, int R, int TWT>
__device__ __forceinline__ void tw_tmem_fill(const double2* TW, uint32_t twt, int t) {
  if constexpr (TWT == 2) {
    constexpr int m = fft_npass<N, R>(), NJ = N / R;
    const int j = t % NJ;
#pragma unroll
    for (int p = 0; p < m - 1; ++p) {
      if (fft_tw_src<N, R, 2>(p) == 2) {
        const int r = fft_rad<N, R>(p), d = fft_len<N, R>(p) / r, k1 = j % d;
        for (int c = 0; c < (r + 1) / 3; ++c) {
          double2 w[3];
#pragma unroll
          for (int u = 0; u < 3; ++u) {
            const int sidx = 3 * c + 1 + u;
            w[u] = sidx < r ? TW[fft_tw_off<N, R>(p) + (sidx - 1) * d + k1] : make_double2(0.0, 0.0);
          }
          tmem_st3(twt + fft_tw_tcol<N, R>(p) + 12 * c, w);
        }
      }
    }
  }
}

__device__ __forceinline__ int full_index(int kap, int N) { return kap >= 0 ? kap : kap + N; }

}  // namespace rsw
