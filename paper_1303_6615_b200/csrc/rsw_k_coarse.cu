// rsw_k_coarse.cu — the persistent cooperative coarse sweep (a3-a5) and the Strang-coarse serial sweep (NEXT-1).
#include "rsw_blocks.cuh"

#include <algorithm>
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


// Kernel argument of one sweep: the placement, the die the sweep runs on (-1: ranks = blocks) and the
// participating CTA count P
struct SweepRun {
  SweepPlace pl;
  int die, P;
  size_t wsm;  // triad sweeps: shared-memory bytes of the owned-block copy (0: read the global table)
};

// TRIAD: N̄ in triad form (rsw_blocks.cuh triad_stage_phase): each CTA keeps the coefficient blocks of its
// owned modes in shared memory (after the layout's LY::bytes), a stage is poll -> owned N̄ -> update with
// no grid barrier (stage-input ring of TRIAD_NB buffers)
// (triad sweeps at n >= 512: two 256-thread CTAs per SM, so registers are capped at 128)
template <int N, int R, int T, int NOWN, bool TRIAD = false>
__global__ void __launch_bounds__(T, (TRIAD && N >= 512) ? 2 : 1) k_coarse_sweep(const CoarseArgs ca, const AvgTab tab, int M, const SweepRun sr,
                                                    double* r_out) {
  using LY = CoarseLayout<N, R, T, NOWN, 1, 1, TRIAD>;
  constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1;
  extern __shared__ double2 smem[];
  __shared__ int s_rank;
  if (threadIdx.x == 0) {  // rank: the block index, or (die placement) a ticket among the die's CTAs
    int r = (int)blockIdx.x;
    if (sr.die >= 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      const int d = smid < 192 ? (int)((sr.pl.diemask[smid >> 6] >> (smid & 63)) & 1ull) : 0;
      r = (d == sr.die) ? (int)atomicAdd(sr.pl.ticket, 1u) : -1;
      if (r >= sr.P) r = -1;
    }
    s_rank = r;
  }
  __syncthreads();
  const int rank = s_rank;
  if (rank < 0) return;  // not part of this sweep (other die, or a surplus CTA)
  HomedArena ha = sr.pl.arena[sr.die > 0 ? 1 : 0];
  ha.flat = sr.die < 0 ? 1 : 0;
  unsigned* bar = reinterpret_cast<unsigned*>(homed_page(ha, sr.pl.bpage));
  const HomedX ax{ha, sr.pl.ypage, sr.pl.ppage};
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
  // CTA's sample pair (TRIAD: the coefficient blocks of the owned modes)
  // (after the layout and the triad's owned constants; null: read the global table)
  double* Wl = sr.wsm ? reinterpret_cast<double*>(smem + (LY::bytes + sizeof(double) * NOWN * 8 + 15) / 16) : nullptr;
  // TRIAD: owned-mode constants after the double slots, frame rotation in the (unused) phase slots
  double* gsm = TRIAD ? reinterpret_cast<double*>(smem + LY::D) + LY::ND : nullptr;
  if constexpr (TRIAD) {
    if (Wl) triad_stage_table<N, NOWN>(tab.triad, Wl, rank, sr.P, threadIdx.x, T);
    owned_consts<N, NOWN>(ca, tab.triad_ph, gsm, smem + LY::PH, rank, sr.P, threadIdx.x, T);
  }
  else fill_packed_twiddles<N, R, T>(TW, tab.tw);
  for (int k = threadIdx.x; k <= K; k += T) {
    GA[k] = __ldg(tab.g.a + k);
    GP[k] = __ldg(tab.g.p + k);
    GQ[k] = __ldg(tab.g.q + k);
  }
  const unsigned P = (unsigned)sr.P;
  const bool one_pair = (int)P >= M / 2;
  if (!TRIAD && one_pair && rank < M / 2) {
    const int mA = 2 * rank + 1, mB = 2 * rank + 2;
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
  constexpr int Kc3 = 3 * Kc;
  const int nst = ca.scheme == 0 ? 4 : 2;
  unsigned epoch = 0, ucount = 0;
  const bool prof = ca.prof && rank == 0;
  int ps = 0;
  // the three stage-input buffers start empty (sentinel) before anyone writes
  constexpr int NB = TRIAD ? TRIAD_NB : 3;
  for (int i = rank * T + threadIdx.x; i < NB * Kc3; i += P * T) st_relaxed_v2(ax.y(i), yin_sentinel());
  grid_barrier(bar, P, epoch);
  coarse_update_phase<N, T, NOWN, CtaGroup, HomedX, TRIAD>(ca, ax, 0, 0, Vs, KSs, kk, un_s, red, rdb, yv, yidx, ucount,
                                                           rank, (int)P, CtaGroup(), nullptr, gsm);  // slice 0: v = e^{ΔT D̂/2} U_0
  for (int n = 0; n < ca.n_end; ++n) {
    if constexpr (TRIAD) {
      for (int st = 1; st <= nst; ++st) {
        if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 0] = gtimer();
        triad_stage_phase<N, T, NOWN, CtaGroup, HomedX>(ax, (size_t)(ucount % NB) * Kc3, Wl, tab.triad, smem + LY::PH, C, A, kk, rank, (int)P,
                                                        CtaGroup(), nullptr, 0, nullptr, nullptr, nullptr,
                                                        (prof && ps == 8) ? ca.prof + 256 : nullptr);
        if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 1] = ca.prof[ps * 4 + 2] = gtimer();
        ++ucount;
        coarse_update_phase<N, T, NOWN, CtaGroup, HomedX, TRIAD>(ca, ax, st, n, Vs, KSs, kk, un_s, red, rdb, yv, yidx,
                                                                 ucount, rank, (int)P, CtaGroup(), nullptr, gsm);
        if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 3] = gtimer();
        ++ps;
      }
    } else {
    for (int st = 1; st <= nst; ++st) {
      if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 0] = gtimer();
      coarse_samples_phase<N, R, T>(ax, (size_t)(ucount % 3) * Kc3, M, tab, X, Y, TW, C, A, PHc, SW, GA, GP, GQ,
                                    (prof && ps == 8) ? ca.prof + 256 : nullptr, rank, (int)P);
      if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 1] = gtimer();
      grid_barrier(bar, P, epoch);
      if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 2] = gtimer();
      ++ucount;
      coarse_update_phase<N, T, NOWN, CtaGroup, HomedX>(ca, ax, st, n, Vs, KSs, kk, un_s, red, rdb, yv, yidx, ucount, rank, (int)P, CtaGroup(),
                                      (prof && (ps == 9 || ps == 11)) ? ca.prof + (ps == 9 ? 300 : 320) : nullptr);
      if (prof && threadIdx.x == 0 && ps < 64) ca.prof[ps * 4 + 3] = gtimer();
      ++ps;
    }
    }  // !TRIAD
  }
  grid_barrier(bar, P, epoch);  // every slice's U, G and residual partials are written
  if (r_out && rank == 0) {  // r_k = max_n sqrt(Σ num / Σ den) over slices (fixed order)
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
template <int N, int R, int T>
__global__ void __launch_bounds__(T) k_strang_sweep(const FineTab tab, double h, double* U, double* G,
                                                     const double* F, double* Gnew, int S, double* r_out) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  constexpr double invN = 1.0 / N;
  extern __shared__ double2 smem[];
  double2* W = smem;              // nl_core X (padded layout)
  double2* Yb = W + 3 * N;        // nl_core Y
  double2* TW = Yb + 3 * N;       // packed twiddles
  double2* S1 = TW + fft_tw_size<N, R>();
  fill_packed_twiddles<N, R, T>(TW, tab.tw);
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
    for (int j = threadIdx.x; j < Kc; j += T) {  // first N-eval input: prim(v)
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
      double2 c[3], u[3];
#pragma unroll
      for (int al = 0; al < 3; ++al) c[al] = S1[al * Kc + j];
      to_prim(kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak), __ldg(tab.g.p + ak), __ldg(tab.g.q + ak), c, u);
      put_input_z<N, R>(W, full_index(kap, N), (double)kap, u);
    }
    __syncthreads();
    for (int st = 0; st < 2; ++st) {
      nl_core<N, R, T>(W, Yb, TW);
      for (int j = threadIdx.x; j < Kc; j += T) {
        const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
        const int kf = full_index(kap, N);
        const double as = kap < 0 ? -__ldg(tab.g.a + ak) : __ldg(tab.g.a + ak);
        const double p = __ldg(tab.g.p + ak), q = __ldg(tab.g.q + ak);
        double2 nh[3], nn[3], x[3];
        get_output_z<N, R>(W, kf, (double)kap, invN, nh);
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
          put_input_z<N, R>(W, kf, (double)kap, u);
        }
      }
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

template <int N, int NOWN, bool TRIAD = false, int R = coarse_radix<N>(), int T = coarse_threads<N>()>
static cudaError_t launch_coarse_sweep_nown(const CoarseArgs& ca, const AvgTab& tab, int M, const SweepPlace& pl,
                                            double* r_out, int grid, bool on_die, int* die_used, cudaStream_t st) {
  auto kfn = k_coarse_sweep<N, R, T, NOWN, TRIAD>;
  int dev, sms, per_sm;
  cudaError_t e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  SweepRun sr{pl, -1, grid, 0};
  size_t sm = CoarseLayout<N, R, T, NOWN, 1, 1, TRIAD>::bytes + (TRIAD ? sizeof(double) * NOWN * 8 : 0);  // (+ owned constants)
  if (TRIAD) {  // + the largest owned-block copy of the coefficient table, when it fits
    size_t mx = 0;
    for (int r = 0; r < grid; ++r) mx = std::max(mx, triad_local_entries(N / 3, r, grid, NOWN));
    int optin = 0;
    if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
    const size_t sw = (sm + 15) / 16 * 16 + sizeof(double) * mx;
    if (sw <= (size_t)optin) {
      sm = sw;
      sr.wsm = sizeof(double) * mx;
    }
  }
  int launch = grid;
  if (on_die) {  // on the die with more SMs; one CTA per SM on every SM (the others exit at once)
    sr.die = pl.die_n[1] > pl.die_n[0] ? 1 : 0;
    launch = sms;
    if (sm < 120 * 1024) sm = 120 * 1024;  // > half an SM's shared memory: exactly one CTA per SM
  }
  if ((e = set_smem(kfn, sm)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, T, sm)) != cudaSuccess) return e;
  if (launch > per_sm * sms) return cudaErrorCooperativeLaunchTooLarge;
  if (on_die && per_sm != 1) return cudaErrorInvalidConfiguration;
  if (die_used) *die_used = sr.die;
  CoarseArgs c2 = ca;
  // the barrier counter (its arena page) and the die ticket start at zero
  HomedArena ha = pl.arena[sr.die > 0 ? 1 : 0];
  ha.flat = sr.die < 0 ? 1 : 0;
  char* bpage = homed_page(ha, pl.bpage);
  if ((e = cudaMemsetAsync(bpage, 0, 4096, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(pl.ticket, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
  void* args[] = {(void*)&c2, (void*)&tab, (void*)&M, (void*)&sr, (void*)&r_out};
  return cudaLaunchCooperativeKernel((const void*)kfn, dim3(launch), dim3(T), args, sm, st);
}

template <int N>
static cudaError_t launch_coarse_sweep_n(const CoarseArgs& ca, const AvgTab& tab, int M, const SweepPlace& pl,
                                         double* r_out, int* grid_used, int* die_used, cudaStream_t st) {
  int dev, sms;
  cudaError_t e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  constexpr int K = N / 3;
  // one sample pair per CTA, but enough CTAs that each owns <= 16 modes in the update phase;
  // at most one CTA per SM (co-residency of the cooperative launch).  Triad form: two owned modes per
  // CTA (one warp per half of a mode's rows)
  const bool triad = tab.triad != nullptr;
  int grid = triad ? (K + 2) / 2 : M / 2;
  if (grid < (K + 1 + 15) / 16) grid = (K + 1 + 15) / 16;
  if (grid > sms) grid = sms;
  if (grid < 1) grid = 1;
  // die placement when the sweep fits on one die
  const bool on_die = pl.die_ok && grid <= std::max(pl.die_n[0], pl.die_n[1]) && !getenv("RSW_NO_DIE_AWARE");
  if (die_used) *die_used = -1;
  const int nown = (K + 1 + grid - 1) / grid;  // owned modes per CTA in the update phase
  if (grid_used) *grid_used = grid;
  if constexpr (N >= 512) {
    // n >= 512: the coefficients come from L2 and a mode has up to 683 rows: two owned modes per 256-thread
    // CTA (four warps each), (K+2)/2 CTAs, two per SM (C5: 171 CTAs instead of 148 with 3 modes each)
    if (triad && !getenv("RSW_TRIAD_WIDE_OFF")) {
      const int g2 = (K + 2) / 2;
      if (grid_used) *grid_used = g2;
      return launch_coarse_sweep_nown<N, 2, true, coarse_radix<N>(), 256>(ca, tab, M, pl, r_out, g2, false, die_used, st);
    }
  }
  if (triad) {
    if (nown <= 1) return launch_coarse_sweep_nown<N, 1, true>(ca, tab, M, pl, r_out, grid, on_die, die_used, st);
    if (nown <= 2) return launch_coarse_sweep_nown<N, 2, true>(ca, tab, M, pl, r_out, grid, on_die, die_used, st);
    if (nown <= 4) return launch_coarse_sweep_nown<N, 4, true>(ca, tab, M, pl, r_out, grid, on_die, die_used, st);
    return cudaErrorInvalidConfiguration;
  }
#define L_(NO) launch_coarse_sweep_nown<N, NO>(ca, tab, M, pl, r_out, grid, on_die, die_used, st)
  if (nown <= 1) return L_(1);
  if (nown <= 2) return L_(2);
  if (nown <= 4) return L_(4);
  if (nown <= 8) return L_(8);
  if (nown <= 16) return L_(16);
#undef L_
  return cudaErrorInvalidConfiguration;
}

unsigned sweep_pages(int n, int M) {
  const unsigned Kc3 = 3u * (2u * (unsigned)(n / 3) + 1u), pairs = (unsigned)std::max(M / 2, 1);
  return 1u + yin_pages(n) + (pairs * Kc3 + 255u) / 256u;
}

template <int N>
static cudaError_t launch_strang_sweep_n(const FineTab& tab, double h, double* U, double* G, const double* F,
                                         double* Gnew, int S, double* r_out, cudaStream_t st) {
  constexpr int R = fine_radix<N>(), T = core_threads<N, R>() > 96 ? core_threads<N, R>() : 96;
  auto kfn = k_strang_sweep<N, R, T>;
  constexpr size_t sm = sizeof(double2) * (6 * N + fft_tw_size<N, R>() + 3 * (2 * (N / 3) + 1));
  cudaError_t e = set_smem(kfn, sm);
  if (e != cudaSuccess) return e;
  kfn<<<1, T, sm, st>>>(tab, h, U, G, F, Gnew, S, r_out);
  return cudaGetLastError();
}


cudaError_t launch_coarse_sweep(int n, const CoarseArgs& ca, const AvgTab& tab, int M, const SweepPlace& pl,
                                double* r_out, int* grid_used, int* die_used, cudaStream_t st) {
#define C(NN) launch_coarse_sweep_n<NN>(ca, tab, M, pl, r_out, grid_used, die_used, st)
  RSW_DISPATCH(n, C)
#undef C
}

cudaError_t launch_strang_sweep(int n, const FineTab& tab, double h, double* U, double* G, const double* F,
                                double* Gnew, int S, double* r_out, cudaStream_t st) {
#define C(NN) launch_strang_sweep_n<NN>(tab, h, U, G, F, Gnew, S, r_out, st)
  RSW_DISPATCH(n, C)
#undef C
}

}  // namespace rsw
