// rsw_pipeline.cuh — pipelined parareal as ONE persistent cooperative kernel.
//
// The bulk-synchronous schedule (rsw_capi.cu) runs, per iteration, the fine sweep over every slice
// and then the serial coarse sweep; the GPU is almost idle during the sweep (one sample pair per
// SM, a latency-bound chain of 4S stages).  The data dependencies of the iteration (Eq. "HMM parareal
// iteration" P:428-430, Alg.4) are finer than that:
//     F(U^k_n)        needs U^k_n only                       (sweep k, slice n-1)
//     U^k_{n+1}      = G(U^k_n) + F(U^{k-1}_n) - G(U^{k-1}_n)  needs sweep k at slice n, the fine
//                     solve of U^{k-1}_n and sweep k-1 at slice n
// so sweep k can trail sweep k-1 by one fine-slice latency, and the fine solves fill the SMs the
// sweeps leave idle (P:433-438 notes the slices "can be computed as soon as" their input exists).
// The values computed are exactly those of the bulk schedule (same kernels' arithmetic, same fixed
// reduction orders), so the iterates, residuals and iteration counts are bitwise identical.
//
// Roles (by arrival ticket; 2 CTAs per SM, all co-resident):
//   * NG coarse groups of GC CTAs: group g runs sweeps k = g, g+NG, ... (rsw_blocks.cuh phases with a
//     group-local barrier counter and stage-input buffers); after every slice each CTA bumps
//     prog[k] (release); the finalize of slice n waits for doneF[k-1][n/2] and prog[k-1] (acquire).
//   * fine workers: NPG thread groups per CTA (named barriers), each claims the lowest-iteration
//     ready pair task (k, p) (slices 2p, 2p+1 of U^k; ready when prog[k] covers them), runs the
//     fine pair integrator (state in TMEM), writes F^k and sets doneF[k][p] (release).
// Stop rule (tol > 0): the group that finishes sweep k computes r_k; the first r_k < tol (or a
// divergence) lowers stopk; later sweeps abort at their next group barrier (the abort travels in
// the barrier counter, so every CTA of a group takes the same decision) and no more fine tasks of
// iterations >= stopk are claimed.  Every wait is bounded: it gives up after ~4 s without any progress
// anywhere in the kernel (heartbeat counter; watchdog flag).
#pragma once
#include "rsw_blocks.cuh"

#include <cstdio>

#ifndef RSW_PIPE_COARSE_THREADS
#define RSW_PIPE_COARSE_THREADS 288  // coarse sub-CTA: three 96-thread parts evaluate three sample pairs at once
#endif
#ifndef RSW_PIPE_FINE_TMUL
#define RSW_PIPE_FINE_TMUL 2  // threads per fine group = TMUL x 3N/R
#endif
#ifndef RSW_PIPE_FINE_WSWAP
#define RSW_PIPE_FINE_WSWAP 1  // fine FFT fields on warps 0, 1, 3 (NamedGroup::wsw)
#endif
#ifndef RSW_PIPE_REUSE_COARSE
#define RSW_PIPE_REUSE_COARSE 0  // 1: a coarse CTA whose sweeps are done runs an extra fine group (C3: 34.2 -> 34.4 ms, not kept)
#endif
#ifndef RSW_PIPE_COARSE_LOW
#define RSW_PIPE_COARSE_LOW 0  // 1: coarse sub-CTA on the low warps, fine groups on the high ones
#endif
#ifndef RSW_PIPE_CLAIM
#define RSW_PIPE_CLAIM 1  // fine-task claim order: 0 lowest iteration first, 1 oldest ready task first
#endif
#ifndef RSW_PIPE_FINE_GROUPS
#define RSW_PIPE_FINE_GROUPS 1  // fine worker groups per CTA (two slowed the sweeps on C3)
#endif
// triad sweeps: the coarse sub-CTA needs 2 warps per owned mode, and the fine throughput
// sets the pace once the chain is short — so fewer coarse threads and more fine groups per CTA
#ifndef RSW_PIPE_TRIAD_TC
#define RSW_PIPE_TRIAD_TC 288  // 128 (2 fine groups beside it): C3 29.6-34.4 ms; 128 (1 group): 27.6-27.9; 288: 25.6-26.5
#endif
#ifndef RSW_PIPE_TRIAD_NPG
#define RSW_PIPE_TRIAD_NPG 1
#endif
#ifndef RSW_PIPE_TRIAD_TMUL
#define RSW_PIPE_TRIAD_TMUL 2  // threads of the fine group beside a triad coarse sub-CTA = TMUL x 3N/R
#endif
#ifndef RSW_PIPE_TRIAD_XMUL
#define RSW_PIPE_TRIAD_XMUL 2  // ... and of the second fine group of a CTA without a coarse role (on the coarse threads)
#endif

namespace rsw {

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
constexpr unsigned ABORT_BIT = 1u << 28;

// group barrier over P CTAs (their coarse sub-CTAs `grp`) on counter `bar`; rank 0 may raise the abort
// bit, which every CTA of the group observes on the same barrier (or the one before it, where
// nothing else is left to do)
template <class GRP>
__device__ __forceinline__ bool group_barrier(unsigned* bar, unsigned P, unsigned& epoch, bool raise, unsigned* wd,
                                              const unsigned* hb, unsigned* s_flag, const GRP& grp) {
  grp.sync();
  if (grp.tid() == 0) {
    ++epoch;
    red_release_add(bar, raise ? ABORT_BIT + 1 : 1);
    const unsigned target = epoch * P;
    unsigned v = ld_acquire_gpu(bar);
    Watch w = watch_start(hb);
    for (unsigned it = 0; v < target && !(v & ABORT_BIT); ++it) {
      if ((it & 63) == 63 && watchdog_expired(w, wd, hb)) {
        v = ABORT_BIT;
        break;
      }
      if (RSW_POLL_SLEEP_NS > 0) __nanosleep(RSW_POLL_SLEEP_NS);
      v = ld_acquire_gpu(bar);
    }
    *s_flag = (v & ABORT_BIT) ? 1u : 0u;
  }
  grp.sync();
  return *s_flag != 0;
}

// CTA = NPG fine groups of TG threads (threads [0, NPG TG), named barriers 1..NPG) + one coarse
// sub-CTA (the TC highest threads, named barrier 15; the warp arbiter prefers high warp ids, so the
// latency-critical sweep wins issue slots over the throughput-bound fine solves).  The tcgen05
// allocation limits a cooperative launch to one CTA per SM, so the roles are warp-specialized inside
// the CTA rather than spread over CTAs.
// smallest radix whose FFT core fits in `threads` threads
template <int N>
__host__ __device__ constexpr int radix_for_threads(int threads) {
  return (3 * (N / 4) <= threads) ? 4 : (3 * (N / 8) <= threads) ? 8 : (3 * (N / 16) <= threads) ? 16 : 32;
}
template <int N, int TC, int NPC, int RC0>
__host__ __device__ constexpr int pipe_split() {  // sample pairs a coarse sub-CTA evaluates concurrently
  // parts must be whole warps (named-barrier thread counts) and must run the bulk sweep's radix RC0
  // (another radix rounds differently: the schedules would no longer agree bitwise)
  return (NPC >= 4 && (TC / 4) % 32 == 0 && 3 * (N / RC0) <= TC / 4 && TC / 4 < TC / 3 - 31) ? 4
       : (NPC >= 3 && (TC / 3) % 32 == 0 && 3 * (N / RC0) <= TC / 3) ? 3
       : (NPC >= 2 && (TC / 2) % 32 == 0 && 3 * (N / RC0) <= TC / 2) ? 2 : 1;
}

// coarse sub-CTA region of the triad sweeps (no FFT buffers, twiddles or sample phases): the stage input
// C, the half-sums HP, the owned entries' state, and the double / int slots; the coefficient blocks
// follow the whole layout (runtime size, PipeArgs::wsm)
template <int N, int T, int NOWN>
struct TriadCoarseLayout {
  static constexpr int K = N / 3, Kc = 2 * K + 1, NR = (T > NOWN * 6 ? T : NOWN * 6);
  static constexpr int C = 0, HP = C + 3 * Kc, VS = HP + NOWN * 6, KS = VS + NOWN * 6, KK = KS + NOWN * 6,
                       UN = KK + NOWN * 6, YV = UN + NOWN * 3, RPH = YV + NOWN * 6, PRE = RPH + K + 1,
                       D = PRE + NOWN * 9;
  static constexpr int RED = 0, YI = RED + NR, GS = YI + NOWN * 6, POK = GS + NOWN * 8, ND = POK + NOWN * 3;
  static constexpr size_t bytes = sizeof(double2) * D + sizeof(double) * ND;
};

template <int N, int RC0, int TC, int NOWN, int NPC, int RF, int TG, int NPG, bool TRIAD = false>
struct PipeLayout {
  static constexpr int SPLIT = pipe_split<N, TC, NPC, RC0>();
  static constexpr int RC = RC0;
  using CL = CoarseLayout<N, RC, TC, NOWN, NPC, SPLIT>;
  using TL = TriadCoarseLayout<N, TC, NOWN>;
  static constexpr int K = N / 3, KP = K + 1;
  // coarse region: the coarse sub-CTA's layout, or (CTAs without a coarse role) TC/TG extra fine groups' X/Y
  // second fine groups on the coarse threads of CTAs without a coarse role: TGX threads each
  static constexpr int TGX = TRIAD ? RSW_PIPE_TRIAD_XMUL * core_threads<N, RF>() : TG;
  static constexpr int XG = TC / TGX;
  static constexpr size_t CB_ = TRIAD ? TL::bytes : CL::bytes;
  static constexpr size_t CREG = CB_ > sizeof(double2) * XG * 6 * N ? CB_ : sizeof(double2) * XG * 6 * N;
  static constexpr int C0 = 0, F0 = (int)((CREG + 15) / 16);  // double2 offsets of the coarse / fine regions
  static constexpr int F_TW = F0, F_CP = F_TW + fft_tw_size<N, RF>(), F_D = F_CP + 6 * KP, F_ND = 9 * KP,
                       F_G = F_D + (F_ND + 1) / 2;  // first fine group's X
  static constexpr size_t bytes = sizeof(double2) * (F_G + NPG * 6 * N);
  // fine groups read their radix-R twiddles from TMEM whenever the transform keeps full tables (as k_fine
  // does: the two schedules must round alike)
  static constexpr int TWT = fft_tw_tcols<N, RF>() > 0 ? 2 : 0;
  static constexpr int CPG0 = FineTmem<N, TG>::COLS > FineTmem<N, TGX>::COLS ? FineTmem<N, TG>::COLS : FineTmem<N, TGX>::COLS;
  static constexpr int CPG = (CPG0 + (TWT == 2 ? fft_tw_tcols<N, RF>() : 0) + 31) / 32 * 32;  // TMEM columns per fine group
  static constexpr int T = TC + NPG * TG;
};

// fine worker group: claim the lowest-iteration ready pair task (k, p) — slices 2p, 2p+1 of U^k, ready
// when prog[k] covers them — run the fine pair integrator, write F^k, set doneF[k][p] (release)
// young: claim the most recently ready task instead of the oldest (the second fine group of a CTA
// without a coarse role: its tasks run slower beside the first, so it takes those with the most slack)
template <int N, int RF, int TG, int FSCHEME, int TWT>
__device__ __forceinline__ void fine_worker_loop(const PipeArgs& a, const NamedGroup grp, double2* W,
                                                 const FineSmemTab& ft, uint32_t tcol, int* task, bool young = false) {
  constexpr size_t L = (size_t)3 * (N / 2 + 1) * 2;
  const int S = a.S, Kit = a.K, npairs = a.npairs;
  double2* Yb = W + 3 * N;
  const uint32_t twcol = tcol + FineTmem<N, TG>::COLS;  // this group's twiddle copies (TWT = 2)
  if constexpr (TWT == 2) {
    tw_tmem_fill<N, RF, 2>(ft.TW, twcol + ((uint32_t)(32 * ((threadIdx.x >> 5) & 3)) << 16), grp.tid());
    tmem_wait_st();
    tmem_fence_before();
    grp.sync();
    tmem_fence_after();
  }
  for (;;) {
    if (grp.tid() == 0) {
      int tk = -1, tp = -1;
      Watch w = watch_start(a.hb);
      for (unsigned it = 0;; ++it) {
        const int lim = min(Kit, *(volatile int*)a.stopk) - 1;  // F^k is needed by sweep k+1 <= stop
        bool all_claimed = true;
#if RSW_PIPE_CLAIM == 1
        // the oldest ready task first: sweeps advance at one pace, so the iteration whose next unclaimed
        // pair became ready the most slices ago holds the earliest deadline (sweep k+1 needs it)
        int bk = -1, bt = 0, bpp = 0, bage = -1;
        for (int k = 0; k <= lim; ++k) {
          const unsigned t = *(volatile unsigned*)(a.next + k);
          if ((int)t >= a.pair_hi - a.pair_lo) continue;
          all_claimed = false;
          const int pp = a.pair_lo + (int)t;
          const int need = (2 * pp + 1 < S) ? 2 * pp + 1 : 2 * pp;
          const int age = (int)(ld_acquire_gpu(a.prog + k) / (unsigned)a.GC) - need;  // slices finalized past it
          if (age >= 0 && (bage < 0 || (young ? age < bage : age > bage))) {
            bage = age;
            bk = k;
            bt = (int)t;
            bpp = pp;
          }
        }
        if (bk >= 0 && atomicCAS(a.next + bk, (unsigned)bt, (unsigned)bt + 1) == (unsigned)bt) {
          tk = bk;
          tp = bpp;
        }
#else
        for (int k = 0; k <= lim && tk < 0; ++k) {
          const unsigned t = *(volatile unsigned*)(a.next + k);  // local task index: pair pair_lo + t
          if ((int)t >= a.pair_hi - a.pair_lo) continue;
          all_claimed = false;
          const int pp = a.pair_lo + (int)t;
          const int need = (2 * pp + 1 < S) ? 2 * pp + 1 : 2 * pp;  // U^k_{2p}, U^k_{2p+1}
          if (ld_acquire_gpu(a.prog + k) >= (unsigned)(a.GC * need) && atomicCAS(a.next + k, t, t + 1) == t) {
            tk = k;
            tp = pp;
          }
        }
#endif
        if (tk >= 0 || all_claimed) break;
        if ((it & 63) == 63 && watchdog_expired(w, a.wd, a.hb)) break;
        __nanosleep(128);
      }
      task[0] = tk;
      task[1] = tp;
    }
    grp.sync();
    const int tk = task[0], tp = task[1];
    if (tk < 0) break;
    const int nA = 2 * tp, nB = nA + 1;
    unsigned long long* tf =
        a.trace ? a.trace + 2 * (Kit + 1) + (size_t)(Kit + 1) * S + ((size_t)tk * npairs + tp) * 2 : nullptr;
    const unsigned long long t_start = (grp.tid() == 0) ? gtimer() : 0ull;
    if (tf && grp.tid() == 0) tf[0] = t_start;
    const double* Uk = a.Uall + (size_t)tk * (S + 1) * L;
    double* Fk = a.Fall + (size_t)tk * S * L;
    fine_pair_run<N, RF, TG, FSCHEME, false, NamedGroup, false, TWT>(grp, W, Yb, ft, tcol, a.ft.g, Uk + nA * L,
                                                                   nB < S ? Uk + nB * L : nullptr, Fk + nA * L,
                                                                   nB < S ? Fk + nB * L : nullptr, a.m_fine, a.h, a.hb,
                                                                   twcol);
    grp.sync();  // the whole pair's F is written
    if (a.npeers > 0) {
      // multi-GPU: push the pair's endpoints into every peer's F^k at the same offset (NVLink stores to
      // IPC-mapped memory), make them visible at system scope, then release the peers' done flags
      const size_t cnt = (size_t)(nB < S ? 2 : 1) * L / 2;  // double2 entries
      const double2* src = reinterpret_cast<const double2*>(Fk + nA * L);
      for (int r = 0; r < a.npeers; ++r) {  // (peer pointer tables in device memory: dynamic indexing)
        double2* dst = reinterpret_cast<double2*>(a.peerF[r] + (size_t)tk * S * L + nA * L);
        for (size_t i = grp.tid(); i < cnt; i += TG) dst[i] = __ldcg(src + i);
      }
      __threadfence_system();
      grp.sync();
      if (grp.tid() == 0)
        for (int r = 0; r < a.npeers; ++r) st_release_sys_u32(a.peerDoneF[r] + (size_t)tk * npairs + tp, 1u);
    }
    if (grp.tid() == 0) {
      st_release_u32(a.doneF + (size_t)tk * npairs + tp, 1u);
      const unsigned long long t_end = gtimer();
      if (tf) tf[1] = t_end;
      atomicAdd(a.stamps + 2 * (Kit + 1), t_end - t_start);  // fine-task latency sum / count (stats)
      atomicAdd(a.stamps + 2 * (Kit + 1) + 1, 1ull);
    }
  }
}

// r_k = max_n sqrt(Σ num / Σ den) over the slices of the sweep (fixed order, as the bulk sweep); the
// first r_k < tol or a divergence lowers stopk.  Called by the group's rank-0 coarse sub-CTA.
template <int N, int TC>
__device__ __forceinline__ void sweep_residual(const PipeArgs& a, const double* rparts, int k, double* red,
                                               const NamedGroup& cg, int ct) {
  constexpr int KP = N / 3 + 1;
  double mx = 0.0;
  bool bad = false;
  for (int s = ct; s < a.S; s += TC) {
    double num = 0.0, den = 0.0;
    for (int q = 0; q < KP; ++q) {
      num += __ldcg(rparts + ((size_t)s * KP + q) * 2);
      den += __ldcg(rparts + ((size_t)s * KP + q) * 2 + 1);
    }
    const double r = sqrt(num / den);
    if (!(r == r) || isinf(r)) bad = true;
    mx = fmax(mx, r);
  }
  red[ct] = bad ? __longlong_as_double(0x7ff8000000000000LL) : mx;
  cg.sync();
  if (ct == 0) {
    double m = 0.0;
    bool nan = false;
    for (int t = 0; t < TC; ++t) {
      if (red[t] != red[t]) nan = true;
      m = fmax(m, red[t]);
    }
    const double r = nan ? __longlong_as_double(0x7ff8000000000000LL) : m;
    a.resid[k] = r;
    if (!(r == r) || r > 1e6 || (a.tol > 0 && r < a.tol)) atomicMin(a.stopk, k);
  }
}

// Coarse sub-CTA of a triad group: sweeps k = g, g + NG, ... with N̄ in triad form — a stage
// is poll -> owned N̄ (coefficient blocks in shared memory) -> RK update and publication, with no group
// barrier (stage-input ring of TRIAD_NB buffers); a discarded sweep aborts in its stage-input poll.
template <int N, int TC, int NOWN, class LY>
__device__ __forceinline__ void coarse_role_triad(const PipeArgs& a, const NamedGroup& cg, int ct, int g, int c, int gd,
                                                  int gslot, double2* smem, unsigned* s_flag) {
  using TL = typename LY::TL;
  constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1, NH = N / 2 + 1, Kc3 = 3 * Kc, NB = TRIAD_NB;
  constexpr size_t L = (size_t)3 * NH * 2;
  const int S = a.S, Kit = a.K, P = a.GC, M = a.M;
  double2* cs = smem + LY::C0;
  double2* C = cs + TL::C;
  double2* HP = cs + TL::HP;
  double2* Vs = cs + TL::VS;
  double2* KSs = cs + TL::KS;
  double2* kk = cs + TL::KK;
  double2* un_s = cs + TL::UN;
  double2* yv = cs + TL::YV;
  double* sd = reinterpret_cast<double*>(cs + TL::D);
  double* red = sd + TL::RED;
  int* yidx = reinterpret_cast<int*>(sd + TL::YI);
  double* gsm = sd + TL::GS;
  double2* rph = cs + TL::RPH;
  double2* pre = cs + TL::PRE;
  int* pre_ok = reinterpret_cast<int*>(sd + TL::POK);
  double* Wl = a.wsm ? reinterpret_cast<double*>(smem + (LY::bytes + 15) / 16) : nullptr;  // (null: read the global table)
  if (Wl) triad_stage_table<N, NOWN>(a.at.triad, Wl, c, P, ct, TC);
  owned_consts<N, NOWN>(a.base, a.at.triad_ph, gsm, rph, c, P, ct, TC);
  cg.sync();
  constexpr unsigned YP = yin_pages(N);
  const unsigned PPG = ((unsigned)(M / 2 > 0 ? M / 2 : 1) * Kc3 + 255) / 256, GPG = 1 + YP + PPG;
  unsigned* bar = reinterpret_cast<unsigned*>(homed_page(a.arena[gd], gslot * GPG));
  const HomedX ax{a.arena[gd], gslot * GPG + 1, gslot * GPG + 1 + YP};
  const int nst = a.base.scheme == 0 ? 4 : 2;
  unsigned epoch = 0;
  for (int k = g; k <= Kit; k += a.NG) {
    for (int i = c * TC + ct; i < NB * Kc3; i += P * TC) st_relaxed_v2(ax.y(i), yin_sentinel());
    const bool stop_now = (c == 0) && (*(volatile int*)a.stopk < k || *(volatile unsigned*)a.wd != 0);
    if (group_barrier(bar, P, epoch, stop_now, a.wd, a.hb, s_flag, cg)) break;
    if (c == 0 && ct == 0) {
      const unsigned long long t = gtimer();
      a.stamps[2 * k] = t;
      if (a.trace) a.trace[2 * k] = t;
    }
    CoarseArgs ca = a.base;
    ca.U = a.Uall + (size_t)k * (S + 1) * L;
    ca.G = a.Gall + (size_t)k * S * L;
    ca.Uprev = k ? a.Uall + (size_t)(k - 1) * (S + 1) * L : ca.U;
    ca.Gprev = k ? a.Gall + (size_t)(k - 1) * S * L : ca.G;
    ca.F = k ? a.Fall + (size_t)(k - 1) * S * L : nullptr;
    ca.rparts = k ? a.rparts + (size_t)k * S * KP * 2 : nullptr;
    ca.part = nullptr;
    ca.nparts = 1;
    ca.yin = nullptr;
    ca.n_end = S;
    ca.wprog = k ? a.prog + (k - 1) : nullptr;
    ca.wunit = (unsigned)P;
    ca.wF = k ? a.doneF + (size_t)(k - 1) * a.npairs : nullptr;
    ca.wd = a.wd;
    ca.hb = a.hb;
    ca.wsys = a.npeers > 0 || a.pair_hi - a.pair_lo < a.npairs;
    ca.stopk = a.stopk;
    ca.kself = k;
    ca.prof = nullptr;
    unsigned ucount = 0;
    coarse_update_phase<N, TC, NOWN, NamedGroup, HomedX, true>(ca, ax, 0, 0, Vs, KSs, kk, un_s, red, nullptr, yv, yidx,
                                                               ucount, c, P, cg, nullptr, gsm);
    bool aborted = false;
    for (int n = 0; n < S && !aborted; ++n) {
      for (int st = 1; st <= nst; ++st) {
        unsigned long long* stp = (a.trace && g == 0 && c == 0 && ct == 0 && n >= 8 && n < 24 && k == g)
                                      ? a.trace + 2 * (Kit + 1) + (size_t)(Kit + 1) * S + 2 * (size_t)(Kit > 0 ? Kit : 1) * a.npairs +
                                            ((n - 8) * nst + st - 1) * 4
                                      : nullptr;
        if (stp) stp[0] = gtimer();
        if (st == nst && k > 0) finalize_early<N, NOWN>(ca, n, c, P, ct, pre, pre_ok);
        if (triad_stage_phase<N, TC, NOWN, NamedGroup, HomedX>(ax, (size_t)(ucount % NB) * Kc3, Wl, a.at.triad, rph, C, HP, kk, c, P, cg,
                                                               a.stopk, k, a.wd, a.hb, stp ? stp + 1 : nullptr)) {
          aborted = true;
          break;
        }
        ++ucount;
        coarse_update_phase<N, TC, NOWN, NamedGroup, HomedX, true>(ca, ax, st, n, Vs, KSs, kk, un_s, red, nullptr, yv,
                                                                   yidx, ucount, c, P, cg, nullptr, gsm,
                                                                   k > 0 ? pre : nullptr, pre_ok);
        if (stp) stp[3] = gtimer();
      }
      if (!aborted) {
        cg.sync();  // this CTA's part of U^k_{n+1}, G^k_n is written
        if (ct == 0) {
          red_release_add(a.prog + k, 1u);
          if (c == 0) atomicAdd(a.hb, 1u);
        }
        if (a.trace && c == 0 && ct == 0) a.trace[2 * (Kit + 1) + (size_t)k * S + n] = gtimer();
      }
    }
    // end of the sweep: every slice's residual partials are written.  A CTA that aborted in a poll raises
    // the abort bit here: the group's other CTAs either abort in their own polls (no more stage inputs
    // come from this CTA) or, having finished the sweep, meet the raised bit at this barrier — so the
    // whole group leaves together (without it a CTA that aborted at the last stage's poll would leave
    // the others waiting here)
    if (group_barrier(bar, P, epoch, aborted, a.wd, a.hb, s_flag, cg) || aborted) break;
    if (c == 0 && ct == 0) {
      const unsigned long long t = gtimer();
      a.stamps[2 * k + 1] = t;
      if (a.trace) a.trace[2 * k + 1] = t;
    }
    if (c == 0 && k > 0) sweep_residual<N, TC>(a, ca.rparts, k, red, cg, ct);
  }
  cg.sync();
}

template <int N, int RC, int TC, int NOWN, int NPC, int RF, int TG, int NPG, int FSCHEME, bool TRIAD = false>
__global__ void __launch_bounds__(TC + NPG * TG, 1) k_parareal_pipe(const PipeArgs a) {
  using LY = PipeLayout<N, RC, TC, NOWN, NPC, RF, TG, NPG, TRIAD>;
  using CL = typename LY::CL;
  static_assert(NPG * LY::CPG <= 512, "fine groups must fit in TMEM");
  static_assert(NPG <= 7, "named barrier ids (fine 1..7, split parts 8..11, staging 14, coarse 15)");
  constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1, NH = N / 2 + 1, Kc3 = 3 * Kc;
  constexpr size_t L = (size_t)3 * NH * 2;  // doubles per state
  extern __shared__ double2 smem[];
  __shared__ uint32_t tslot;
  __shared__ unsigned s_flag;
  __shared__ int s_role[3];  // coarse group (-1: none), rank in the group, die of the group's arrays
  __shared__ int s_task[NPG + LY::XG][2];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 0) {  // role: coarse group g, rank c (or none); die-aware: from this SM's die ticket
    int g = -1, c = 0, d = 0, slot = 0;
    if (a.die_aware) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      d = smid < 192 ? (int)((a.diemask[smid >> 6] >> (smid & 63)) & 1ull) : 0;
      const int t = (int)atomicAdd(a.dticket + d, 1u);
      slot = t / a.GC;
      if (slot < a.ndg[d]) {
        g = a.dg[d][slot];
        c = t % a.GC;
      }
    } else {
      const int t = (int)atomicAdd(a.ticket, 1u);
      if (t < a.NG * a.GC) {
        g = t / a.GC;
        c = t % a.GC;
        d = g & 1;
        slot = g >> 1;
      }
    }
    s_role[0] = g;
    s_role[1] = c;
    s_role[2] = d | (slot << 1);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const int S = a.S, Kit = a.K;
  // fine tables (shared by every fine group of the CTA), staged by all threads
  const FineSmemTab ft = stage_fine_tables<N, RF, TC + NPG * TG>(
      smem + LY::F_TW, smem + LY::F_CP, reinterpret_cast<double*>(smem + LY::F_D), a.ft, threadIdx.x, TC + NPG * TG);
  __syncthreads();

  // fine groups take the low warps and the coarse sub-CTA the high ones (RSW_PIPE_COARSE_LOW = 0), or
  // the other way round: CB = the coarse sub-CTA's first thread, FB = the first fine group's
  constexpr int FT = NPG * TG;
  constexpr int CB = RSW_PIPE_COARSE_LOW ? 0 : FT, FB = RSW_PIPE_COARSE_LOW ? TC : 0;
  if ((int)threadIdx.x >= CB && (int)threadIdx.x < CB + TC) {
    // ===================================== coarse sub-CTA =====================================
    const NamedGroup cg{CB, 15, TC};
    const int ct = (int)threadIdx.x - CB;
    // XG more fine groups on the coarse threads (in the coarse region of smem): in a CTA without a coarse
    // role, and in a coarse CTA once its group's sweeps are done (the later iterations' fine tasks are
    // then the bottleneck: each finished group adds GC fine groups)
    auto extra_fine = [&]() {
      constexpr int XG = LY::XG, TGX = LY::TGX;
      const int xi = ct / TGX;
      if (xi < XG && (NPG + XG) * LY::CPG <= 512)
        fine_worker_loop<N, RF, TGX, FSCHEME, LY::TWT>(a, NamedGroup{CB + xi * TGX, 1 + NPG + xi, TGX},
                                            smem + LY::C0 + (size_t)xi * 6 * N, ft,
                                            tslot + (uint32_t)((NPG + xi) * LY::CPG), s_task[NPG + xi],
                                            a.extra_young != 0);
    };
    if (s_role[0] >= 0) {
      if constexpr (TRIAD) {
      coarse_role_triad<N, TC, NOWN, LY>(a, cg, ct, s_role[0], s_role[1], s_role[2] & 1, s_role[2] >> 1, smem,
                                         &s_flag);
      } else {
      const int g = s_role[0], c = s_role[1], P = a.GC, gd = s_role[2] & 1, gslot = s_role[2] >> 1;
      double2* cs = smem + LY::C0;
      double2* X = cs + CL::X;
      double2* Y = cs + CL::Y;
      double2* TW = cs + CL::TW;
      double2* C = cs + CL::C;
      double2* A = cs + CL::A;
      double2* Vs = cs + CL::VS;
      double2* KSs = cs + CL::KS;
      double2* kk = cs + CL::KK;
      double2* un_s = cs + CL::UN;
      double2* rdb = cs + CL::RDB;
      double2* PH = cs + CL::PH;
      double2* yv = cs + CL::YV;
      double* sd = reinterpret_cast<double*>(cs + CL::D);
      double* red = sd + CL::RED;
      double* GA = sd + CL::GA;
      double* GP = sd + CL::GP;
      double* GQ = sd + CL::GQ;
      double* SW = sd + CL::SW;
      int* yidx = reinterpret_cast<int*>(sd + CL::YI);
      const AvgTab& tab = a.at;
      const int M = a.M;
      fill_packed_twiddles<N, LY::RC, TC>(TW, tab.tw, ct);
      for (int k = ct; k <= K; k += TC) {
        GA[k] = __ldg(tab.g.a + k);
        GP[k] = __ldg(tab.g.p + k);
        GQ[k] = __ldg(tab.g.q + k);
      }
      for (int q = 0; q < NPC; ++q) {  // phases / weights of this CTA's pairs c, c + P, ...
        const int pr = c + q * P;
        if (pr >= M / 2) break;
        const int mA = 2 * pr + 1, mB = 2 * pr + 2;
        for (int k = ct; k <= K; k += TC) {
          PH[(size_t)q * 2 * KP + k] = __ldg(tab.phase + (size_t)mA * KP + k);
          PH[(size_t)q * 2 * KP + KP + k] = __ldg(tab.phase + (size_t)mB * KP + k);
        }
        if (ct == 0) {
          SW[2 * q] = __ldg(tab.w + mA);
          SW[2 * q + 1] = mB <= M - 1 ? __ldg(tab.w + mB) : 0.0;
        }
      }
      cg.sync();
      // the group's exchange arrays in pages homed on die gd: barrier counter, stage inputs, partials
      constexpr unsigned YP = yin_pages(N);
      const unsigned PPG = ((unsigned)(M / 2 > 0 ? M / 2 : 1) * Kc3 + 255) / 256, GPG = 1 + YP + PPG;
      unsigned* bar = reinterpret_cast<unsigned*>(homed_page(a.arena[gd], gslot * GPG));
      const HomedX ax{a.arena[gd], gslot * GPG + 1, gslot * GPG + 1 + YP};
      const int nst = a.base.scheme == 0 ? 4 : 2;
      unsigned epoch = 0;
      for (int k = g; k <= Kit; k += a.NG) {
        // sweep start: the three stage-input buffers of the group start empty
        for (int i = c * TC + ct; i < 3 * Kc3; i += P * TC) st_relaxed_v2(ax.y(i), yin_sentinel());
        const bool stop_now = (c == 0) && (*(volatile int*)a.stopk < k || *(volatile unsigned*)a.wd != 0);
        if (group_barrier(bar, P, epoch, stop_now, a.wd, a.hb, &s_flag, cg)) break;
        if (c == 0 && ct == 0) {
          const unsigned long long t = gtimer();
          a.stamps[2 * k] = t;  // sweep k start (stats)
          if (a.trace) a.trace[2 * k] = t;
        }
        CoarseArgs ca = a.base;
        ca.U = a.Uall + (size_t)k * (S + 1) * L;
        ca.G = a.Gall + (size_t)k * S * L;
        ca.Uprev = k ? a.Uall + (size_t)(k - 1) * (S + 1) * L : ca.U;
        ca.Gprev = k ? a.Gall + (size_t)(k - 1) * S * L : ca.G;
        ca.F = k ? a.Fall + (size_t)(k - 1) * S * L : nullptr;
        ca.rparts = k ? a.rparts + (size_t)k * S * KP * 2 : nullptr;
        ca.part = nullptr;  // (addressed through ax)
        ca.nparts = M / 2 > 0 ? M / 2 : 1;
        ca.yin = nullptr;
        ca.n_end = S;
        ca.wprog = k ? a.prog + (k - 1) : nullptr;
        ca.wunit = (unsigned)P;
        ca.wF = k ? a.doneF + (size_t)(k - 1) * a.npairs : nullptr;
        ca.wd = a.wd;
        ca.hb = a.hb;
        ca.wsys = a.npeers > 0 || a.pair_hi - a.pair_lo < a.npairs;  // flags of other ranks' tasks
        ca.stopk = a.stopk;
        ca.kself = k;
        ca.prof = nullptr;
        unsigned ucount = 0;
        coarse_update_phase<N, TC, NOWN>(ca, ax, 0, 0, Vs, KSs, kk, un_s, red, rdb, yv, yidx, ucount, c, P, cg);
        bool aborted = false;
        for (int n = 0; n < S && !aborted; ++n) {
          for (int st = 1; st <= nst; ++st) {
            // optional stage-phase stamps (trace, group 0 rank 0, slices 8..23 of sweep g): samples / barrier / update
            unsigned long long* stp = (a.trace && g == 0 && c == 0 && ct == 0 && n >= 8 && n < 24 && k == g)
                                          ? a.trace + 2 * (Kit + 1) + (size_t)(Kit + 1) * S + 2 * (size_t)(Kit > 0 ? Kit : 1) * a.npairs +
                                                ((n - 8) * nst + st - 1) * 4
                                          : nullptr;
            // trace of the stage-input hand-off (same slices): every CTA's update-phase end, CTA 0's
            // arrival of the complete stage input
            const int sidx = (n - 8) * nst + st - 1;
            unsigned long long* hand = (a.trace && g == 0 && ct == 0 && n >= 8 && n < 24 && k == g && c < 64)
                                           ? a.trace + 2 * (Kit + 1) + (size_t)(Kit + 1) * S +
                                                 2 * (size_t)(Kit > 0 ? Kit : 1) * a.npairs + 256
                                           : nullptr;
            if (stp) stp[0] = gtimer();
            coarse_samples_phase<N, LY::RC, TC, NamedGroup, NPC, LY::SPLIT>(ax, (size_t)(ucount % 3) * Kc3, M, tab, X, Y, TW,
                                                             C, A, PH, SW, GA, GP, GQ, nullptr, c, P, cg,
                                                             (hand && c == 0) ? hand + 4096 + sidx : nullptr);
            if (stp) stp[1] = gtimer();
            const bool raise = (c == 0) && (*(volatile int*)a.stopk < k || *(volatile unsigned*)a.wd != 0);
            if (group_barrier(bar, P, epoch, raise, a.wd, a.hb, &s_flag, cg)) {
              aborted = true;
              break;
            }
            if (stp) stp[2] = gtimer();
            ++ucount;
            coarse_update_phase<N, TC, NOWN>(ca, ax, st, n, Vs, KSs, kk, un_s, red, rdb, yv, yidx, ucount, c, P, cg);
            if (stp) stp[3] = gtimer();
            if (hand) hand[sidx * 64 + c] = gtimer();
          }
          if (!aborted) {
            cg.sync();  // this CTA's part of U^k_{n+1}, G^k_n is written
            if (ct == 0) {
              red_release_add(a.prog + k, 1u);
              if (c == 0) atomicAdd(a.hb, 1u);  // watchdog heartbeat: a slice of sweep k is done
            }
            if (a.trace && c == 0 && ct == 0) a.trace[2 * (Kit + 1) + (size_t)k * S + n] = gtimer();
          }
        }
        if (aborted) break;
        if (group_barrier(bar, P, epoch, false, a.wd, a.hb, &s_flag, cg)) break;  // every slice's residual partials written
        if (c == 0 && ct == 0) {
          const unsigned long long t = gtimer();
          a.stamps[2 * k + 1] = t;  // sweep k end (stats)
          if (a.trace) a.trace[2 * k + 1] = t;
        }
        if (c == 0 && k > 0) {  // r_k = max_n sqrt(Σ num / Σ den) (fixed order, as the bulk sweep)
          double mx = 0.0;
          bool bad = false;
          for (int s = ct; s < S; s += TC) {
            double num = 0.0, den = 0.0;
            for (int q = 0; q <= K; ++q) {
              num += __ldcg(ca.rparts + ((size_t)s * KP + q) * 2);
              den += __ldcg(ca.rparts + ((size_t)s * KP + q) * 2 + 1);
            }
            const double r = sqrt(num / den);
            if (!(r == r) || isinf(r)) bad = true;
            mx = fmax(mx, r);
          }
          red[ct] = bad ? __longlong_as_double(0x7ff8000000000000LL) : mx;
          cg.sync();
          if (ct == 0) {
            double m = 0.0;
            bool nan = false;
            for (int t = 0; t < TC; ++t) {
              if (red[t] != red[t]) nan = true;
              m = fmax(m, red[t]);
            }
            const double r = nan ? __longlong_as_double(0x7ff8000000000000LL) : m;
            a.resid[k] = r;
            if (!(r == r) || r > 1e6 || (a.tol > 0 && r < a.tol)) atomicMin(a.stopk, k);
          }
        }
      }
      cg.sync();  // every coarse thread is past the sweeps: the coarse region of smem is free
      }  // !TRIAD
    }
    if ((s_role[0] < 0 && a.extra_fine) || RSW_PIPE_REUSE_COARSE) extra_fine();
  } else {
    // ======================================= fine worker group 0 =======================================
    // (coarse_solo: the CTAs of a coarse group leave their SM to the sweep, no fine work beside it)
    if (a.coarse_solo && s_role[0] >= 0) goto fine_done;
    {
    const int gi = ((int)threadIdx.x - FB) / TG;
    fine_worker_loop<N, RF, TG, FSCHEME, LY::TWT>(a, NamedGroup{FB + gi * TG, 1 + gi, TG, 0, (RSW_PIPE_FINE_WSWAP && !RSW_PIPE_COARSE_LOW && TG >= 128) ? 1 : 0}, smem + LY::F_G + (size_t)gi * 6 * N,
                                        ft, tslot + (uint32_t)(gi * LY::CPG), s_task[gi]);
    }
  fine_done:;
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc<512>(tslot);
  }
}

// ---------------------------------------------------------------------------------------------
// launcher: picks the configuration for n, checks co-residency (2 CTAs per SM), launches
// ---------------------------------------------------------------------------------------------
template <int N, int NOWN, int NPC, int FSCHEME, bool TRIAD = false>
static inline cudaError_t launch_pipe_nf(const PipeArgs& a, int grid, size_t* out, cudaStream_t st) {
  constexpr int RC = coarse_radix<N>();
  constexpr int TC = TRIAD ? RSW_PIPE_TRIAD_TC
                           : (RSW_PIPE_COARSE_THREADS > coarse_threads<N>() ? RSW_PIPE_COARSE_THREADS : coarse_threads<N>());
  constexpr int RF = fine_radix<N>(), TG = (TRIAD ? RSW_PIPE_TRIAD_TMUL : RSW_PIPE_FINE_TMUL) * core_threads<N, RF>();
  constexpr int CPG = (FineTmem<N, TG>::COLS + 31) / 32 * 32;
  constexpr int NPG0 = TRIAD ? RSW_PIPE_TRIAD_NPG : RSW_PIPE_FINE_GROUPS;
  constexpr int NPG = NPG0 * CPG <= 512 ? NPG0 : 512 / CPG;
  using LY = PipeLayout<N, RC, TC, NOWN, NPC, RF, TG, NPG, TRIAD>;
  auto kfn = k_parareal_pipe<N, RC, TC, NOWN, NPC, RF, TG, NPG, FSCHEME, TRIAD>;
  PipeArgs a2 = a;
  cudaError_t e;
  if (TRIAD) {  // the owned-block copy of the triad coefficients when it fits, else the global table
    int dev = 0, optin = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
    if ((LY::bytes + 15) / 16 * 16 + a.wsm > (size_t)optin) a2.wsm = 0;
  }
  const size_t sm = TRIAD ? (LY::bytes + 15) / 16 * 16 + a2.wsm : LY::bytes;
  e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  if (grid <= 0) {  // query: co-resident CTAs (tensor-memory kernels: one per SM)
    int per_sm = 0, dev = 0, sms = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, LY::T, sm)) != cudaSuccess) return e;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if (out) *out = (size_t)(per_sm > 1 ? 1 : per_sm) * sms;
    if (getenv("RSW_PIPE_TRACE"))
      fprintf(stderr, "[rsw pipe] n=%d: %d threads (coarse %d + %d fine groups of %d), %zu B smem, %d CTA/SM\n", N,
              LY::T, TC, NPG, TG, sm, per_sm);
    return cudaSuccess;
  }
  if (TRIAD && getenv("RSW_PIPE_TRACE"))
    fprintf(stderr, "[rsw pipe] triad coefficients: %s (%zu B per CTA)\n", a2.wsm ? "shared memory" : "global table", a.wsm);
  void* args[] = {(void*)&a2};
  return cudaLaunchCooperativeKernel((const void*)kfn, dim3(grid), dim3(LY::T), args, sm, st);
}

template <int N>
static inline cudaError_t launch_pipe_n(const PipeArgs& a, int fine_scheme, int grid, size_t* out, cudaStream_t st) {
  constexpr int K = N / 3;
  const int nown = (K + 1 + a.GC - 1) / a.GC;
  const int npc = (a.M / 2 + a.GC - 1) / a.GC;  // sample pairs per coarse CTA
  if (a.at.triad) {  // triad sweeps: owned modes only (no sample pairs)
#define PIPE_TCFG(NW)                                                                                    \
  if (nown <= NW) return fine_scheme == 0 ? launch_pipe_nf<N, NW, 1, 0, true>(a, grid, out, st)          \
                         : fine_scheme == 1 ? launch_pipe_nf<N, NW, 1, 1, true>(a, grid, out, st)        \
                                            : launch_pipe_nf<N, NW, 1, 2, true>(a, grid, out, st);
    PIPE_TCFG(2)
    PIPE_TCFG(4)
    PIPE_TCFG(8)
#undef PIPE_TCFG
    return cudaErrorInvalidConfiguration;
  }
#define PIPE_CFG(NW, NP)                                                                            \
  if (nown <= NW && npc <= NP) return fine_scheme == 0 ? launch_pipe_nf<N, NW, NP, 0>(a, grid, out, st) \
                                    : fine_scheme == 1 ? launch_pipe_nf<N, NW, NP, 1>(a, grid, out, st) \
                                                       : launch_pipe_nf<N, NW, NP, 2>(a, grid, out, st);
  PIPE_CFG(2, 1)
  PIPE_CFG(2, 2)
  PIPE_CFG(4, 2)
  PIPE_CFG(8, 4)
  PIPE_CFG(8, 8)
#undef PIPE_CFG
  return cudaErrorInvalidConfiguration;
}

}  // namespace rsw
