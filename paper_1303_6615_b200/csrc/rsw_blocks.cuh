// rsw_blocks.cuh — device building blocks shared by the standalone kernels (rsw_k_*.cu) and the
// pipelined parareal megakernel (rsw_pipeline.cu): radix / thread choices, pair load / store,
// the fine pair integrator (a2 / a2'), and the coarse-sweep phases (a3 / a4 / a5).
#pragma once
#include "rsw_internal.h"
#include "rsw_device.cuh"

#include <cstdlib>

namespace rsw {

// Radix / thread choices of the in-place register FFT core (nl_core), R values per thread, T = 3N/R
// threads rounded up to whole warps.  Plans (passes): 1024 = 4.16.16 at R = 16 (8: 2.8.8.8),
// 512 = 8.8.8, 256 = 4.8.8, 128 = 2.8.8.  Fine kernel at n = 1024: two 192-thread pair-groups per
// CTA sharing the tables (fine_groups).  Coarse sweep (latency bound, one sample pair per CTA):
// radix 8 — at n <= 256 with 192 threads (the extra threads speed up the mode loops), at n = 1024 with
// 384 (four radix-8 passes on twice the warps beat three radix-16 passes: C5 stage 17.1 -> 16.6 us).
template <int N>
__host__ __device__ constexpr int fine_radix() { return N <= 32 ? 4 : (N <= 512 ? 8 : 16); }
template <int N>
__host__ __device__ constexpr int fine_groups() { return N >= 1024 ? 2 : 1; }
template <int N, int R>
__host__ __device__ constexpr int core_threads() { return (3 * (N / R) + 31) / 32 * 32; }
#ifndef RSW_COARSE_R1024
#define RSW_COARSE_R1024 8  // radix of the coarse sweep's N-evals at n >= 512: 8 (384 threads at n = 1024) beats 16 (192): C5 stage 17.1 -> 16.6 us
#endif
template <int N>
__host__ __device__ constexpr int coarse_radix() { return N <= 32 ? 4 : N <= 256 ? 8 : RSW_COARSE_R1024; }
template <int N>
__host__ __device__ constexpr int coarse_threads() { return core_threads<N, coarse_radix<N>()>() > 192 ? core_threads<N, coarse_radix<N>()>() : 192; }

// ---------------------------------------------------------------------------------------------
// shared helpers: load a pair of half-spectrum states into packed eigen coordinates, and store
// ---------------------------------------------------------------------------------------------
template <int N, int T>
__device__ __forceinline__ void load_pair_eigen(const double* __restrict__ uA, const double* __restrict__ uB,
                                                const ModeGeom g, double2* C /*[3][Kc]*/, int t0 = -1) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  const double2* A = reinterpret_cast<const double2*>(uA);
  const double2* B = reinterpret_cast<const double2*>(uB);
  for (int j = (t0 < 0 ? (int)threadIdx.x : t0); j < Kc; j += T) {
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
                                                double* __restrict__ oB, int t0 = -1) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  double2* A = reinterpret_cast<double2*>(oA);
  double2* B = reinterpret_cast<double2*>(oB);
  for (int k = (t0 < 0 ? (int)threadIdx.x : t0); k < NH; k += T) {
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

// per-configuration fine tables staged in shared memory (one copy per CTA)
struct FineSmemTab {
  const double2* TW;  // packed twiddles of nl_core
  const double2* CP;  // [6][K+1]
  const double* C0;   // [6][K+1]
  const double *GA, *GP, *GQ;
};

template <int N, int R, int T>
__device__ __forceinline__ FineSmemTab stage_fine_tables(double2* smem_tw, double2* smem_cp, double* smem_d,
                                                         const FineTab& tab, int t, int nthr) {
  constexpr int K = N / 3, KP = K + 1;
  double* sC0 = smem_d;
  double* sGA = sC0 + 6 * KP;
  double* sGP = sGA + KP;
  double* sGQ = sGP + KP;
  fill_packed_twiddles<N, R, T>(smem_tw, tab.tw, t, nthr);
  for (int i = t; i < 6 * KP; i += nthr) {
    smem_cp[i] = __ldg(tab.cp + i);
    sC0[i] = __ldg(tab.c0 + i);
  }
  for (int i = t; i < KP; i += nthr) {
    sGA[i] = __ldg(tab.g.a + i);
    sGP[i] = __ldg(tab.g.p + i);
    sGQ[i] = __ldg(tab.g.q + i);
  }
  return FineSmemTab{smem_tw, smem_cp, sC0, sGA, sGP, sGQ};
}

template <int N, int TG>
struct FineTmem {  // TMEM columns of one fine pair-group: per mode slot o, S1 / S0 / S2 at o*36 + {0, 12, 24}
  static constexpr int Kc = 2 * (N / 3) + 1, OMAX = (Kc + TG - 1) / TG, WG = (TG / 32 + 3) / 4;
  static constexpr int COLS = WG * OMAX * 36;
};

// One pair of slices advanced by m fine steps (a2 / a2') by a warp-aligned thread group: the state
// lives in the group's TMEM columns, the N-evals in its X / Y buffers.  Used by k_fine (the whole
// CTA) and by the fine workers of the pipelined parareal kernel (one of several groups of a CTA).
// TMEM layout of the group's thread-private slots: lane quarter = (CTA warp) mod 4; column block =
// (group warp) / 4 (TBLK = false: groups own disjoint column ranges starting at tcol) or (CTA warp) / 4
// (TBLK = true: tcol is the CTA's base and the groups of a CTA interleave, 3 blocks for 12 warps).
// TWT / twcol: twiddle policy of the FFT core (fft_tw_src) and, for TWT = 2, the TMEM column address of
// the CTA's twiddle region (filled by the caller with tw_tmem_fill).
// po / poff: optional peer outputs (multi-GPU bulk schedule): the pair's endpoints are also stored at
// po->out[r] + poff (A) and + poff + L (B, when present), then made visible at system scope.
template <int N, int R, int TG, int SCHEME, bool LIN, class GRP, bool TBLK = false, int TWT = 0>
__device__ __forceinline__ void fine_pair_run(const GRP& grp, double2* W, double2* Y, const FineSmemTab& st_,
                                              uint32_t tcol, const ModeGeom& gg, const double* uA,
                                              const double* uB, double* oA, double* oB, int m_steps, double h,
                                              unsigned* hb = nullptr, uint32_t twcol = 0,
                                              const PeerOut* po = nullptr, size_t poff = 0) {
  constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1, OMAX = FineTmem<N, TG>::OMAX;
  const double2* sCP = st_.CP;
  const double* sC0 = st_.C0;
  const double* sGA = st_.GA;
  const double* sGP = st_.GP;
  const double* sGQ = st_.GQ;
  const int t = grp.tid();
  const int warp = threadIdx.x >> 5, gwarp = t >> 5;
  load_pair_eigen<N, TG>(uA, uB, gg, W, t);  // C[α][j] staged in W
  grp.sync();
  // thread-private TMEM slot of mode slot o: columns o*36 + {S1: 0, S0: 12, S2: 24} + 4α
  const uint32_t tb = tcol + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(((TBLK ? warp : gwarp) >> 2) * OMAX * 36);
  const uint32_t twt = twcol + ((uint32_t)(32 * (warp & 3)) << 16);
  double2 c0v[OMAX][3];
#pragma unroll
  for (int o = 0; o < OMAX; ++o) {
    const int j = t + o * TG;
#pragma unroll
    for (int al = 0; al < 3; ++al) c0v[o][al] = (j < Kc) ? W[al * Kc + j] : make_double2(0.0, 0.0);
  }
  grp.sync();  // C fully read before W receives the first N-eval input
#pragma unroll
  for (int o = 0; o < OMAX; ++o) {
    const int j = t + o * TG;
    const int jj = j < Kc ? j : 0;
    const int kap = kappa_of(jj, K), ak = kap < 0 ? -kap : kap;
    if (SCHEME == 1) {  // Strang prologue: S1 = v = E2 c
#pragma unroll
      for (int al = 0; al < 3; ++al) c0v[o][al] = dmul(al - 1, sCP[1 * KP + ak], sC0[1 * KP + ak], c0v[o][al]);
    }
    tmem_st3(tb + o * 36, c0v[o]);
    if (!LIN && j < Kc) {
      const double as = kap < 0 ? -sGA[ak] : sGA[ak];
      put_input_eigen<N, R>(W, full_index(kap, N), (double)kap, as, sGP[ak], sGQ[ak], c0v[o]);
    }
  }
  tmem_wait_st();
  grp.sync();

  constexpr bool RK = (SCHEME == 0 || SCHEME == 2);  // four-stage schemes with S0 / S2 in TMEM
  const int nst = RK ? 4 : 2;
  for (int step = 0; step < m_steps; ++step) {
    const bool last_step = (step == m_steps - 1);
    if (hb && t == 0 && (step & 7) == 7) atomicAdd(hb, 1u);  // pipelined: heartbeat of the watchdog
    for (int st = 0; st < nst; ++st) {
      if (!LIN) nl_core<N, R, TG, GRP, TWT>(W, Y, st_.TW, grp, twt);
      // epilogue (this stage's update) fused with the prologue of the next N-eval (rolled when a
      // thread owns many modes: an unrolled body of 4 modes spills at 168 registers)
#pragma unroll (OMAX > 2 ? 1 : OMAX)
      for (int o = 0; o < OMAX; ++o) {
        const int j = t + o * TG;
        const bool valid = j < Kc;
        const int jj = valid ? j : 0;
        const int kap = kappa_of(jj, K), ak = kap < 0 ? -kap : kap;
        const int kf = full_index(kap, N);
        const uint32_t ts = tb + o * 36;
        double2 s1[3], s0[3], s2[3];
        // S1 (every stage), with S0 = E2 c (stage 1) or S2 = E2 a - Q Nu (IF: E c; stage 2) under one wait
        if (RK && st == 1) tmem_ld3x2(ts, s1, ts + 12, s0);
        else if (RK && st == 2) tmem_ld3x2(ts, s1, ts + 24, s2);
        else tmem_ld3(ts, s1);
        const double as = kap < 0 ? -sGA[ak] : sGA[ak];
        const double p = sGP[ak], q = sGQ[ak];
        double2 nn[3];
        if (!LIN && valid) {
          get_output_eigen<N, R>(W, kf, (double)kap, as, p, q, nn);
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
          } else if (SCHEME == 2) {
            // integrating-factor RK4 (Lawson form of RK4 on v = e^{-tA}u, forward factors only):
            //   k1 = N(u); a = E2 (u + h/2 k1); k2 = N(a); b = E2 u + h/2 k2; k3 = N(b);
            //   c = E u + h E2 k3; k4 = N(c); u+ = E u + h/6 (E k1 + 2 E2 k2 + 2 E2 k3 + k4)
            // S0 = E2 u, S2 = E u, S1 accumulates u+
            if (st == 0) {
              const double2 c = s1[al];
              const double2 e2c = dmul(alpha, CP(1), C0(1), c);
              const double2 ec = dmul(alpha, CP(0), C0(0), c);
              s0[al] = e2c;
              s2[al] = ec;
              s1[al] = caxpy(h / 6.0, dmul(alpha, CP(0), C0(0), nn[al]), ec);
              x[al] = caxpy(0.5 * h, dmul(alpha, CP(1), C0(1), nn[al]), e2c);
            } else if (st == 1) {
              x[al] = caxpy(0.5 * h, nn[al], s0[al]);
              s1[al] = caxpy(h / 3.0, dmul(alpha, CP(1), C0(1), nn[al]), s1[al]);
            } else if (st == 2) {
              const double2 e2k = dmul(alpha, CP(1), C0(1), nn[al]);
              x[al] = caxpy(h, e2k, s2[al]);
              s1[al] = caxpy(h / 3.0, e2k, s1[al]);
            } else {
              s1[al] = caxpy(h / 6.0, nn[al], s1[al]);
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
        if (RK || st == 1) tmem_st3(ts, s1);
        if (RK && st == 0) {
          tmem_st3(ts + 12, s0);
          tmem_st3(ts + 24, s2);
        }
        if (!LIN && valid) put_input_eigen<N, R>(W, kf, (double)kap, as, p, q, x);
      }
      tmem_wait_st();
      grp.sync();
    }
  }
  // final state S1 -> C[α][j] in W (the last stage's N-eval inputs are dead; every thread is past
  // its last W read at the barrier above), then store
#pragma unroll
  for (int o = 0; o < OMAX; ++o) {
    const int j = t + o * TG;
    double2 s1[3];
    tmem_ld3(tb + o * 36, s1);
    if (j < Kc) {
#pragma unroll
      for (int al = 0; al < 3; ++al) W[al * Kc + j] = s1[al];
    }
  }
  grp.sync();
  store_pair_prim<N, TG>(W, gg, oA, oB, t);
  if (po && po->n > 0) {
    constexpr size_t L = (size_t)3 * (N / 2 + 1) * 2;
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)  // constant indices: the parameter array stays in parameter space
      if (r < po->n) store_pair_prim<N, TG>(W, gg, po->out[r] + poff, oB ? po->out[r] + poff + L : nullptr, t);
    __threadfence_system();
  }
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
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
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

// bounded spins (pipelined parareal): acquire loads, back off, give up once NOTHING in the kernel has
// progressed for ~4 s — the heartbeat `hb` (bumped by the fine workers every 8 steps and by every
// finished coarse slice) did not move — or when another CTA raised the watchdog flag wd.  A
// dependency that never completes is a bug: the kernel then reports an error instead of hanging the
// GPU, while a legitimately long wait (one fine solve of many steps) keeps the heartbeat moving.
struct Watch {
  unsigned long long t0;
  unsigned hb;
};
__device__ __forceinline__ Watch watch_start(const unsigned* hb) {
  return Watch{gtimer(), hb ? *(volatile const unsigned*)hb : 0u};
}
__device__ __forceinline__ bool watchdog_expired(Watch& w, unsigned* wd, const unsigned* hb) {
  const unsigned long long now = gtimer();
  if (hb) {
    const unsigned h = *(volatile const unsigned*)hb;
    if (h != w.hb) {
      w.hb = h;
      w.t0 = now;
    }
  }
  // limit: hb[1] ms without progress (the host writes it next to the heartbeat; RSW_WATCHDOG_MS, 4 s)
  const unsigned long long lim = hb ? 1000000ull * *(volatile const unsigned*)(hb + 1) : 4000000000ull;
  if (now - w.t0 > lim) {
    if (wd) atomicExch(wd, 1u);
    return true;
  }
  return wd && *(volatile unsigned*)wd != 0;
}
// stopk / kself: give up as well once the run stopped before iteration kself (the waiting sweep is
// discarded: its remaining work only has to reach the next group barrier, where it aborts)
// sys: the flag is released by another GPU (multi-GPU pipelined schedule): system-scope acquire
__device__ __forceinline__ void spin_until_geq(const unsigned* p, unsigned target, unsigned* wd, const unsigned* hb,
                                               const int* stopk = nullptr, int kself = 0, bool sys = false) {
  auto ld = [&] { return sys ? ld_acquire_sys(p) : ld_acquire_gpu(p); };
  if (ld() >= target) return;
  Watch w = watch_start(hb);
  for (unsigned it = 0;; ++it) {
    if (ld() >= target) return;
    if (stopk && *(volatile const int*)stopk < kself) return;
    if ((it & 63) == 63 && watchdog_expired(w, wd, hb)) return;
    __nanosleep(64);
  }
}

// Stage input through a triple-buffered shared array (replaces "owners write y -> grid barrier ->
// everyone loads y"): update phase u writes its owned entries of the next stage input into
// ybuf[u%3] (each entry once) and resets the same entries of ybuf[(u+2)%3] to the sentinel; the
// samples phase polls ybuf[u%3] until no entry holds the sentinel.  Safe without fences: each
// 8-byte half is single-copy atomic; the reset of ybuf[(u+2)%3] happens after every reader of it
// (samples phase u-1) passed the release/acquire grid barrier before update u, and it is ordered
// before any reader of ybuf[(u+2)%3] (samples phase u+2) by the grid barrier after samples u+1.
#ifndef RSW_POLL_SLEEP_NS
#define RSW_POLL_SLEEP_NS 0  // back-off of the stage-input poll and the group-barrier spin (0: none)
#endif
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

// Addressing of a coarse group's exchange arrays: element i of the stage-input triple buffer (y) and
// of the per-pair partials (part).  FlatX: plain arrays (bulk sweep).  HomedX: 4 KB pages of a
// HomedArena (rsw_internal.h) homed on the group's die, 256 double2 per page.
struct FlatX {
  double2* yb;
  double2* pt;
  __device__ __forceinline__ double2* y(size_t i) const { return yb + i; }
  __device__ __forceinline__ double2* part(size_t i) const { return pt + i; }
};
struct HomedX {
  HomedArena h;
  unsigned yp, pp;  // first logical pages of the stage inputs and of the partials
  __device__ __forceinline__ double2* at(unsigned p0, size_t i) const {
    return reinterpret_cast<double2*>(homed_page(h, p0 + (unsigned)(i >> 8))) + (i & 255);
  }
  __device__ __forceinline__ double2* y(size_t i) const { return at(yp, i); }
  __device__ __forceinline__ double2* part(size_t i) const { return at(pp, i); }
};

// Samples phase of one RK stage (Alg.1): poll the stage input y into C, then evaluate this
// CTA's sample pairs (m_A, m_B) = (2p+1, 2p+2), p = rank, rank + P, ..., SPLIT pairs at a time on
// SPLIT thread parts (each with its own X/Y at X + h*6N and named barrier 8 + h), writing one
// partial Σ_{m in pair} w_m P+_m N(P-_m y) per pair to part[p] (per-pair partials: the owners'
// reduction order is then independent of the CTA count, so every schedule agrees bitwise).
template <int N, int R, int T, class GRP = CtaGroup, int NPC = 1, int SPLIT = 1, class AX = FlatX>
__device__ __forceinline__ void coarse_samples_phase(const AX& ax, size_t yoff, int M, const AvgTab& tab,
                                                     double2* X, double2* /*Y (= X + 3N)*/, const double2* TW,
                                                     double2* C, double2* /*A (unused)*/, const double2* PH,
                                                     const double* SW, const double* GA, const double* GP,
                                                     const double* GQ, unsigned long long* cyc = nullptr,
                                                     int rank = -1, int P = -1, const GRP& grp = GRP(),
                                                     unsigned long long* ystamp = nullptr) {
  static_assert(T % SPLIT == 0 && (T / SPLIT) % 32 == 0, "parts must be whole warps (bar.sync counts)");
  static_assert(3 * (N / R) <= T / SPLIT, "each part must cover 3N/R FFT threads");
  constexpr int TH = T / SPLIT;
  const int tid_ = grp.tid();
  if (rank < 0) {
    rank = blockIdx.x;
    P = gridDim.x;
  }
#define STAMP(i) \
  if (cyc && tid_ == 0) cyc[i] = clock64();
  STAMP(0)
  // PH: phases e^{iωτ_m} of this CTA's first NPC pairs, [NPC][2][K+1] (null: load from the table);
  // SW: their weights; GA/GP/GQ: geometry a, p, q per |κ| staged in shared memory
  constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1;
  constexpr double invN = 1.0 / N;
  // stage input (triple-buffered, sentinel = not yet written): poll, keep
  for (int i = tid_; i < 3 * Kc; i += T) {
    const double2* yi = ax.y(yoff + i);
    double2 v = ld_relaxed_v2(yi);
    while (is_sentinel(v.x) || is_sentinel(v.y)) {
      if (RSW_POLL_SLEEP_NS > 0) __nanosleep(RSW_POLL_SLEEP_NS);  // (spinning warps take issue slots from co-resident ones)
      v = ld_relaxed_v2(yi);
    }
    C[i] = v;
  }
  grp.sync();
  STAMP(5)
  if (ystamp && tid_ == 0) *ystamp = gtimer();  // trace: the whole stage input has arrived
  const int h = SPLIT > 1 ? tid_ / TH : 0, th = tid_ - h * TH;
  const NamedGroup hg{grp.base() + h * TH, 8 + h, TH};  // named barriers 8..11
  double2* Xh = X + (size_t)h * 6 * N;
  double2* Yh = Xh + 3 * N;
  const int npairs = M / 2;  // samples 1..M-1 -> pairs (1,2), (3,4), ...; last B may be M (w=0)
  for (int pr = rank + h * P; pr < npairs; pr += SPLIT * P) {
    const int mA = 2 * pr + 1, mB = 2 * pr + 2;
    const bool hasB = mB <= M - 1;
    const int q = (pr - rank) / P;  // this CTA's q-th pair: phases / weights cached when q < NPC
    const bool cached = PH && q < NPC;
    const double2* PHq = PH + (size_t)q * 2 * KP;
    const double* SWq = SW + 2 * q;
    for (int j = th; j < Kc; j += TH) {
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
      const double as = kap < 0 ? -GA[ak] : GA[ak];
      const double2 pA = cached ? PHq[ak] : __ldg(tab.phase + (size_t)mA * KP + ak);
      const double2 pB = !hasB ? make_double2(1.0, 0.0) : (cached ? PHq[KP + ak] : __ldg(tab.phase + (size_t)mB * KP + ak));
      double2 c[3];
      // packed eigen input: P-_{mA} y + i P-_{mB} y   (P-: α=-1 -> e^{+iωτ}, α=+1 -> e^{-iωτ})
      const double2 ym = C[j], y0 = C[Kc + j], yp = C[2 * Kc + j];
      const double2 bm = hasB ? cmul(ym, pB) : make_double2(0.0, 0.0);
      const double2 b0 = hasB ? y0 : make_double2(0.0, 0.0);
      const double2 bp = hasB ? cmulc(yp, pB) : make_double2(0.0, 0.0);
      c[0] = cadd(cmul(ym, pA), cmuli(bm));
      c[1] = cadd(y0, cmuli(b0));
      c[2] = cadd(cmulc(yp, pA), cmuli(bp));
      put_input_eigen<N, R>(Xh, full_index(kap, N), (double)kap, as, GP[ak], GQ[ak], c);
    }
    if (SPLIT > 1) hg.sync(); else grp.sync();
    STAMP(1)
    if (SPLIT > 1) nl_core<N, R, TH>(Xh, Yh, TW, hg); else nl_core<N, R, T>(Xh, Yh, TW, grp);
    STAMP(2)
    const double wA = cached ? SWq[0] : __ldg(tab.w + mA), wB = hasB ? (cached ? SWq[1] : __ldg(tab.w + mB)) : 0.0;
    const size_t pb = (size_t)pr * 3 * Kc;
    for (int j = th; j < Kc; j += TH) {
      const int kap = kappa_of(j, K), ak = kap < 0 ? -kap : kap;
      const double as = kap < 0 ? -GA[ak] : GA[ak];
      const double p = GP[ak], q = GQ[ak];
      // unpack the two samples from the raw outputs Z(±κ): with D = diag(-iκ, -1, -iκ)/N the map of the
      // packed pair, conj(D(-κ) Z(-κ)) = D(κ) conj Z(-κ), so N_A(κ) = D(κ) (Z(κ) + conj Z(-κ))/2 and
      // N_B(κ) = D(κ) (-i)(Z(κ) - conj Z(-κ))/2: the half-sums go through the fused eigen map (scale 1/2N)
      constexpr int FS = fft_fs<N, R>();
      const int ip = fpad<R>(full_index(kap, N)), im = fpad<R>(full_index(-kap, N));
      double2 ra[3], rb[3], ea[3], eb[3];
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        const double2 zp = Xh[f * FS + ip], zc = cconj(Xh[f * FS + im]);
        ra[f] = cadd(zp, zc);
        rb[f] = cmulmi(csub(zp, zc));
      }
      eigen_from_raw(ra[0], ra[1], ra[2], (double)kap, as, p, q, 0.5 * invN, ea);
      eigen_from_raw(rb[0], rb[1], rb[2], (double)kap, as, p, q, 0.5 * invN, eb);
      const double2 pA = cached ? PHq[ak] : __ldg(tab.phase + (size_t)mA * KP + ak);
      const double2 z0 = make_double2(0.0, 0.0);
      double2 am = caxpy(wA, cmulc(ea[0], pA), z0);  // P+: α=-1 -> e^{-iωτ}, α=+1 -> e^{+iωτ}
      double2 a0 = caxpy(wA, ea[1], z0);
      double2 ap = caxpy(wA, cmul(ea[2], pA), z0);
      if (hasB) {
        const double2 pB = cached ? PHq[KP + ak] : __ldg(tab.phase + (size_t)mB * KP + ak);
        am = caxpy(wB, cmulc(eb[0], pB), am);
        a0 = caxpy(wB, eb[1], a0);
        ap = caxpy(wB, cmul(eb[2], pB), ap);
      }
      *ax.part(pb + j) = am;
      *ax.part(pb + Kc + j) = a0;
      *ax.part(pb + 2 * Kc + j) = ap;
    }
    if (SPLIT > 1) hg.sync(); else grp.sync();  // all mirror reads of X done before the next prologue
    STAMP(3)
  }
  if (SPLIT > 1) grp.sync();
  STAMP(4)
#undef STAMP
}

// ---------------------------------------------------------------------------------------------
// Triad form of the averaged nonlinearity (round 2).  The paper writes the averaged nonlinear term as
// a sum over wavenumber triads (Eq. "nonlinear term for average, RSW"):
//   [e^{sL} N(e^{-sL} u)]_κ^γ = Σ_{κ1+κ2=κ} Σ_{α,β} e^{i(ω^γ_κ - ω^α_κ1 - ω^β_κ2)s} C^{γαβ}_{κκ1κ2} u^α_κ1 u^β_κ2,
// so the M-sample average of Alg.1 is the same bilinear form with the coefficient
//   W^{γαβ}_{κκ1} = Φ(γω_κ - αω_κ1 - βω_κ2) C^{γαβ}_{κκ1κ2},   Φ(λ) = Σ_{m=1}^{M-1} w_m e^{iλτ_m}
// — exactly the quadrature sum (no resonance truncation: every triad is kept with its quadrature
// weight).  The dealiased pseudo-spectral product is an exact convolution (|κ1|, |κ2| <= K = n/3), and
// the first factor of every product of N (u u_x = (u²/2)_x, u v_x, (h u)_x) is u, whose eigen expansion
// has no α = 0 part, so α ranges over {-1, +1}: 18 coefficients per (κ, κ1).  Two exact reductions make
// every coefficient ONE real number: the window is symmetric (w_m = w_{M-m}), so with the centre
// τ_c = T0/(2ε) Φ(λ) = e^{iλτ_c} R(λ), R(λ) = Σ_m w_m cos(λ(τ_m - τ_c)) real, and e^{iλτ_c} factors into
// per-mode phases — the contraction runs in the frame rotated by e^{-τ_c L} (stage input y'_α = y_α
// e^{-iαωτ_c}, output × e^{iγωτ_c}); and each C^{γαβ} is purely real ((γ = 0) == (β = 0)) or purely
// imaginary (the eigenvectors' components are real or imaginary).  The host builds W' = R C (real or
// imaginary part) once per configuration (rsw_capi.cu build_triad); table layout, double units: block
// κ = 0..K at TRIAD_E * triad_rows_before(κ), inside it entry e = (γ+1)*6 + (α>0)*3 + (β+1) of row i at
// e*nk + i, row i <-> κ1 = κ - K + i, κ2 = K - i, nk = 2K + 1 - κ rows.  One N̄ evaluation costs 60 DP
// instructions per (κ, κ1) (6 complex products, 18 two-FMA accumulations) — for C3 ~0.66 M per stage
// instead of 64 pair N-evals — and needs no cross-CTA reduction: the CTA that owns κ computes N̄_κ whole.
// ---------------------------------------------------------------------------------------------
// TRIAD_E, triad_nk, triad_rows_before, triad_local_entries: rsw_internal.h
template <int N, int NOWN>
__device__ __forceinline__ void triad_stage_table(const double* __restrict__ Wg, double* Wl, int rank, int P, int tid,
                                                  int nthr) {
  constexpr int K = N / 3;
  size_t lo = 0;
  for (int o = 0; o < NOWN; ++o) {
    const int kap = rank + o * P;
    if (kap > K) break;
    const size_t cnt = (size_t)TRIAD_E * triad_nk(kap, K);
    const double* src = Wg + (size_t)TRIAD_E * triad_rows_before(kap, K);
    for (size_t i = tid; i < cnt; i += nthr) Wl[lo + i] = __ldg(src + i);
    lo += cnt;
  }
}

// Stage-input ring of the triad sweeps: no barrier separates a stage's reads of its input from the
// owners' next writes, so the ring is deeper (TRIAD_NB buffers) and publication u resets the buffer of
// stage u - NB/2: every reader of it is done (publishing u needs all of input u-1, i.e. every owner
// published u-1, which it did after reading input u-2), and the next writer of it (stage u + NB/2)
// acted on input u + NB/2 - 1, published after a fence that follows this reset (the resetting
// threads fence after every (NB/4)-th publication, NB/4 <= NB/2 - 1).  TRIAD_NB: rsw_internal.h.

// One RK stage's N̄ in triad form: poll the stage input y (ring buffer at yoff) into C, then for each
// owned |κ| = rank + o P the 3 eigen entries γ of N̄_κ (coefficients from the shared-memory copy Wl, or
// — Wl null, the copy does not fit next to the kernel's other buffers — from the global table Wg); the -κ entries by the real-field symmetry
// N̄^γ_{-κ} = conj N̄^{-γ}_κ (the eigenbasis of -κ is the conjugate of +κ's with α reversed).  Fixed
// summation order, independent of T, P and the warp that runs an item: for part h < NPART (triad_parts)
// lane l sums rows i ≡ 32h + l (mod 32 NPART) in ascending i, a fixed xor tree sums the 32 lanes, then
// N̄ = ((part 0 + part 1) + part 2) + ... — so the bulk and pipelined sweeps agree bitwise.  stopk (pipelined schedule):
// the poll gives up once the run stopped before iteration kself, or the watchdog fired; returns true
// then (the whole group takes the same decision on its own, every wait of a discarded sweep aborts).
// per-sweep constants of the triad coarse CTAs in shared memory (the L1 left beside ~200 KB of shared
// memory does not keep them): gsm[o*8 + {0..5}] = a, p, q, e^{-μκ⁴ΔT/2}, e^{-iωΔT/ε} of owned mode o, and
// the frame rotation e^{iω_k τ_c}, k = 0..K
template <int N, int NOWN>
__device__ __forceinline__ void owned_consts(const CoarseArgs& ca, const double2* __restrict__ rph_g, double* gsm,
                                             double2* rph, int rank, int P, int tid, int nthr) {
  constexpr int K = N / 3;
  for (int i = tid; i < NOWN * 8; i += nthr) {
    const int o = i / 8, c = i % 8, ak = rank + o * P;
    double v = 0.0;
    if (ak <= K) {
      if (c == 0) v = __ldg(ca.g.a + ak);
      else if (c == 1) v = __ldg(ca.g.p + ak);
      else if (c == 2) v = __ldg(ca.g.q + ak);
      else if (c == 3) v = __ldg(ca.dhalf + ak);
      else if (c == 4) v = __ldg(ca.back + ak).x;
      else if (c == 5) v = __ldg(ca.back + ak).y;
    }
    gsm[i] = v;
  }
  for (int k = tid; k <= K; k += nthr) rph[k] = __ldg(rph_g + k);
}

// warps per owned mode of the triad sweeps: 2 at n <= 256 (<= 171 rows), 4 above (683 rows at n = 1024)
template <int N>
__host__ __device__ constexpr int triad_parts() { return N <= 256 ? 2 : 4; }

// one lane's share of N̄_κ: rows i = i0, i0 + 32 NPART, ... (ascending), all 18 coefficients of a row loaded
// before its products are used (so the loads overlap), accumulated into acc[γ] in a fixed order
// PREF: the next row's coefficients are loaded while this row is computed (coefficients from L2)
#ifndef RSW_TRIAD_SPLIT
#define RSW_TRIAD_SPLIT 0  // 1: separate accumulators for the α = -1 and α = +1 terms (12 FMA chains per lane, not 6): measured neutral-to-worse (C3 22.9 vs 22.6 ms)
#endif
template <int N, int NPART, bool PREF = false, class LDW>
__device__ __forceinline__ void triad_rows(double2* acc_out, const double2* C, int kap, int nk, int i0, LDW ldw) {
  constexpr int K = N / 3, Kc = 2 * K + 1, NA = RSW_TRIAD_SPLIT ? 2 : 1;
  double2 acc[NA][3];
#pragma unroll
  for (int a = 0; a < NA; ++a)
#pragma unroll
    for (int g = 0; g < 3; ++g) acc[a][g] = make_double2(0.0, 0.0);
  double wn[18];
  if (PREF && i0 < nk)
#pragma unroll
    for (int e = 0; e < 18; ++e) wn[e] = ldw(e, i0);
  for (int i = i0; i < nk; i += 32 * NPART) {
    double wv[18];
    if (PREF) {
#pragma unroll
      for (int e = 0; e < 18; ++e) wv[e] = wn[e];
      if (i + 32 * NPART < nk)
#pragma unroll
        for (int e = 0; e < 18; ++e) wn[e] = ldw(e, i + 32 * NPART);
    } else {
#pragma unroll
      for (int e = 0; e < 18; ++e) wv[e] = ldw(e, i);
    }
    const int k1 = kap - K + i, k2 = K - i;
    const int j1 = k1 >= 0 ? k1 : k1 + Kc, j2 = k2 >= 0 ? k2 : k2 + Kc;
    const double2 am = C[j1], ap = C[2 * Kc + j1];
    double2 pr[6];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double2 yb = C[b * Kc + j2];
      pr[b] = make_double2(fma(am.x, yb.x, -am.y * yb.y), fma(am.x, yb.y, am.y * yb.x));
      pr[3 + b] = make_double2(fma(ap.x, yb.x, -ap.y * yb.y), fma(ap.x, yb.y, ap.y * yb.x));
    }
#pragma unroll
    for (int g = 0; g < 3; ++g) {
#pragma unroll
      for (int ab2 = 0; ab2 < 6; ++ab2) {
        const double w = wv[g * 6 + ab2];
        double2& A = acc[NA == 2 ? ab2 / 3 : 0][g];
        if ((g == 1) == (ab2 % 3 == 1)) {  // real coefficient
          A.x = fma(w, pr[ab2].x, A.x);
          A.y = fma(w, pr[ab2].y, A.y);
        } else {  // imaginary coefficient i w
          A.x = fma(-w, pr[ab2].y, A.x);
          A.y = fma(w, pr[ab2].x, A.y);
        }
      }
    }
  }
#pragma unroll
  for (int g = 0; g < 3; ++g) acc_out[g] = NA == 2 ? cadd(acc[0][g], acc[1][g]) : acc[0][g];
}

template <int N, int T, int NOWN, class GRP = CtaGroup, class AX = FlatX>
__device__ __forceinline__ bool triad_stage_phase(const AX& ax, size_t yoff, const double* Wl, const double* Wg,
                                                  const double2* RPH, double2* C, double2* hp,
                                                  double2* kk, int rank, int P, const GRP& grp,
                                                  const int* stopk = nullptr, int kself = 0, unsigned* wd = nullptr,
                                                  const unsigned* hb = nullptr, unsigned long long* stamp = nullptr,
                                                  unsigned long long* cyc = nullptr) {
  constexpr int K = N / 3, Kc = 2 * K + 1;
  const int tid_ = grp.tid();
  bool ab = false;
#define TSTAMP(i) \
  if (cyc && tid_ == 0) cyc[i] = clock64();
  TSTAMP(0)
  for (int i = tid_; i < 3 * Kc; i += T) {
    const double2* yi = ax.y(yoff + i);
    double2 v = ld_relaxed_v2(yi);
    if (stopk && (is_sentinel(v.x) || is_sentinel(v.y))) {
      Watch w = watch_start(hb);
      for (unsigned it = 0; is_sentinel(v.x) || is_sentinel(v.y); ++it) {
        if ((it & 255) == 255 && (*(volatile const int*)stopk < kself || watchdog_expired(w, wd, hb))) {
          ab = true;
          break;
        }
        v = ld_relaxed_v2(yi);
      }
      if (ab) break;
    } else {
      while (is_sentinel(v.x) || is_sentinel(v.y)) v = ld_relaxed_v2(yi);
    }
    // into the rotated frame: y'_α = y_α e^{-iαωτ_c} (α = -1: × e^{iωτ_c}, α = +1: × its conjugate)
    const int al = i / Kc, j = i - al * Kc, kap = kappa_of(j, K);
    if (al != 1) {
      const double2 r = RPH[kap < 0 ? -kap : kap];  // (shared memory, owned_consts)
      v = al == 0 ? cmul(v, r) : cmulc(v, r);
    }
    C[i] = v;
  }
  TSTAMP(1)
  if (stopk) {
    if (grp.sync_or(ab)) return true;
  } else {
    grp.sync();
  }
  TSTAMP(2)
  if (stamp && tid_ == 0) stamp[0] = gtimer();  // trace: the whole stage input has arrived
  const int lane = tid_ & 31;
  constexpr int NPART = triad_parts<N>();  // warps per owned mode (rows i ≡ 32h + l mod 32 NPART)
  for (int it = tid_ >> 5; it < NPART * NOWN; it += T / 32) {
    const int o = it / NPART, hh = it % NPART, kap = rank + o * P;
    if (kap > K) continue;  // (warp-uniform)
    const int nk = triad_nk(kap, K);
    double2 acc[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    // coefficient block: the CTA's shared-memory copy (Wl; explicit ld.shared — a pointer that may be
    // either space compiles to generic loads), or the global table when it did not fit
    if (Wl) {
      size_t lo = 0;
      for (int q = 0; q < o; ++q) lo += (size_t)TRIAD_E * triad_nk(rank + q * P, K);
      const unsigned wsh = (unsigned)__cvta_generic_to_shared(Wl + lo);
      triad_rows<N, NPART>(acc, C, kap, nk, 32 * hh + lane, [&](int e, int i) {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(wsh + 8u * (unsigned)(e * nk + i)));
        return v;
      });
    } else {
      const double* Wb = Wg + (size_t)TRIAD_E * triad_rows_before(kap, K);
      // (next-row prefetch where the global table is the rule, n >= 512; at n <= 256 it is a rare fallback
      // whose extra registers cost the pipelined kernel's shared-memory path: C3 22.4 -> 25.5 ms)
      triad_rows<N, NPART, (N >= 512)>(acc, C, kap, nk, 32 * hh + lane,
                                       [&](int e, int i) { return __ldg(Wb + (size_t)e * nk + i); });
    }
#pragma unroll
    for (int g = 0; g < 3; ++g)
      for (int w = 16; w > 0; w >>= 1) {
        acc[g].x += __shfl_xor_sync(0xffffffffu, acc[g].x, w);
        acc[g].y += __shfl_xor_sync(0xffffffffu, acc[g].y, w);
      }
    if (lane == 0)
#pragma unroll
      for (int g = 0; g < 3; ++g) hp[(o * NPART + hh) * 3 + g] = acc[g];
  }
  TSTAMP(3)
  grp.sync();
  TSTAMP(4)
  if (tid_ < NOWN * 3) {
    const int o = tid_ / 3, g = tid_ % 3, kap = rank + o * P;
    if (kap <= K) {
      double2 v = hp[(o * NPART) * 3 + g];
#pragma unroll
      for (int h = 1; h < NPART; ++h) v = cadd(v, hp[(o * NPART + h) * 3 + g]);
      if (g != 1) {  // back from the rotated frame: × e^{iγωτ_c}
        const double2 r = RPH[kap];
        v = g == 0 ? cmulc(v, r) : cmul(v, r);
      }
      kk[o * 6 + g] = v;
      kk[o * 6 + 3 + (2 - g)] = cconj(v);
    }
  }
  TSTAMP(5)
#undef TSTAMP
  if (stamp && tid_ == 0) stamp[1] = gtimer();  // trace: this CTA's N̄ entries are done
  return false;
}

// phase 2 of one RK stage, thread-parallel over the CTA's owned modes |κ| = b + o P (o < NOWN):
// items i = o*6 + e, entries e = (α, +κ) for e < 3, (α, -κ) for e >= 3.  The stage base v and the RK
// accumulator ks of owned modes live in this CTA's shared memory for the whole sweep; the stage
// input y is published to global memory for the samples phase of every CTA.
// NB = 3: the quadrature sweeps' triple buffer (reset of the previous stage's buffer, ordered by the
// stage's barrier); NB = TRIAD_NB: the triad sweeps' ring (reset NB/2 stages back, fenced; see above)
template <int N, int NOWN, int T, class GRP = CtaGroup, class AX = FlatX, int NB = 3>
__device__ __forceinline__ void push_stage_input(const AX& ax, const double2* yv, const int* yidx, unsigned u,
                                                 const GRP& grp = GRP()) {
  const int tid_ = grp.tid();
  constexpr int Kc3 = 3 * (2 * (N / 3) + 1);
  constexpr unsigned RB = NB == 3 ? 2u : (unsigned)(NB / 2);  // buffer reset: (u + RB) % NB
  // (each entry is published by the thread that computed it — yv[t], yidx[t] — so the triad sweeps need
  // no barrier here; the quadrature sweeps keep theirs)
  if (NB == 3) grp.sync();
  if (tid_ < NOWN * 6 && yidx[tid_] >= 0) {
    st_relaxed_v2(ax.y((size_t)(u % NB) * Kc3 + yidx[tid_]), yv[tid_]);
    st_relaxed_v2(ax.y((size_t)((u + RB) % NB) * Kc3 + yidx[tid_]), yin_sentinel());
    if (NB != 3 && (u % (unsigned)(NB / 4)) == (unsigned)(NB / 4 - 1)) __threadfence();
  }
}

// Early prefetch of the finalize operands (F_n, G_n of the previous sweep, U_{n+1} of the previous
// iterate) at the start of a slice's last stage, when the fine task and the previous sweep's slice are
// ALREADY complete (non-blocking acquire checks): their L2 round trip then overlaps the stage's N̄
// instead of following it.  pre_ok[t] = 0 leaves the wait and the loads to coarse_update_phase.
template <int N, int NOWN>
__device__ __forceinline__ void finalize_early(const CoarseArgs& ca, int n, int rank, int P, int tid_, double2* pre,
                                               int* pre_ok) {
  constexpr int K = N / 3, NH = N / 2 + 1;
  if (tid_ >= NOWN * 3) return;
  const size_t Ls = (size_t)3 * NH;
  const int o = tid_ / 3, f = tid_ % 3, ak = rank + o * P;
  int ok = 0;
  if (ak <= K) {
    const bool fr = !ca.wF || (ca.wsys ? ld_acquire_sys(ca.wF + n / 2) : ld_acquire_gpu(ca.wF + n / 2)) >= 1u;
    const bool pr = !ca.wprog || ld_acquire_gpu(ca.wprog) >= ca.wunit * (unsigned)(n + 1);
    if (fr && pr) {
      double2 F = make_double2(0.0, 0.0), G = make_double2(0.0, 0.0), U = make_double2(0.0, 0.0);
      if (ca.F) F = __ldcg(reinterpret_cast<const double2*>(ca.F) + (size_t)n * Ls + f * NH + ak);
      if (ca.F) G = __ldcg(reinterpret_cast<const double2*>(ca.Gprev) + (size_t)n * Ls + f * NH + ak);
      if (ca.rparts) U = __ldcg(reinterpret_cast<const double2*>(ca.Uprev) + (size_t)(n + 1) * Ls + f * NH + ak);
      pre[tid_ * 3] = F;
      pre[tid_ * 3 + 1] = G;
      pre[tid_ * 3 + 2] = U;
      ok = 1;
    }
  }
  pre_ok[tid_] = ok;
}

template <int N, int T, int NOWN, class GRP = CtaGroup, class AX = FlatX, bool TRIAD = false>
__device__ __forceinline__ void coarse_update_phase(const CoarseArgs& ca, const AX& ax, int stage, int n, double2* Vs,
                                                    double2* KSs, double2* kk, double2* un_s, double* nd_s,
                                                    double2* red_buf, double2* yv, int* yidx, unsigned ucount,
                                                    int rank = -1, int P = -1, const GRP& grp = GRP(),
                                                    unsigned long long* cyc = nullptr, const double* gsm = nullptr,
                                                    const double2* pre = nullptr, const int* pre_ok = nullptr) {
  const int tid_ = grp.tid();
#define USTAMP(i) \
  if (cyc && tid_ == 0) cyc[i] = clock64();
  USTAMP(0)
  constexpr int K = N / 3, Kc = 2 * K + 1, NH = N / 2 + 1;
  if (rank < 0) {
    rank = blockIdx.x;
    P = gridDim.x;
  }
  const size_t Ls = (size_t)3 * NH;
  const double dT = ca.dT;
  auto entry = [&](int o, int e, int& ak, int& al, int& j) {
    ak = rank + o * P;
    al = e % 3;
    j = (e < 3) ? ak : ((ak == 0) ? 0 : Kc - ak);
  };
  const bool last = (ca.scheme == 0) ? (stage == 4) : (stage == 2);
  double2 *zU = nullptr, *zG = nullptr;  // finalize: the tail modes of U_{n+1} and G_n, zeroed off the critical path
  auto zero_tail = [&]() {
    if (zU)
      for (int k = K + 1; k < NH; ++k) {
        zU[k - K] = make_double2(0.0, 0.0);
        zG[k - K] = make_double2(0.0, 0.0);
      }
  };
  // prefetch the finalize operands (F_n, old G_n, old U_{n+1}) before the reduction's L2 round trip
  double2 pf_F = make_double2(0.0, 0.0), pf_G = make_double2(0.0, 0.0), pf_U = make_double2(0.0, 0.0);
  if (stage > 0 && last && tid_ < NOWN * 3 && pre && pre_ok[tid_]) {  // early prefetch (finalize_early) succeeded
    pf_F = pre[tid_ * 3];
    pf_G = pre[tid_ * 3 + 1];
    pf_U = pre[tid_ * 3 + 2];
  } else if (stage > 0 && last && tid_ < NOWN * 3) {
    const int o = tid_ / 3, f = tid_ % 3, ak = rank + o * P;
    if (ak <= K) {
      // pipelined parareal: F(U^{k-1}_n) and the previous sweep's slice n must be complete
      if (ca.wF) spin_until_geq(ca.wF + n / 2, 1u, ca.wd, ca.hb, ca.stopk, ca.kself, ca.wsys != 0);
      if (ca.wprog) spin_until_geq(ca.wprog, ca.wunit * (unsigned)(n + 1), ca.wd, ca.hb, ca.stopk, ca.kself);
      // (G_n only enters the correction, U_{n+1} only the residual: the k = 0 sweep needs neither)
      if (ca.F) pf_F = __ldcg(reinterpret_cast<const double2*>(ca.F) + (size_t)n * Ls + f * NH + ak);
      if (ca.F) pf_G = __ldcg(reinterpret_cast<const double2*>(ca.Gprev) + (size_t)n * Ls + f * NH + ak);
      if (ca.rparts) pf_U = __ldcg(reinterpret_cast<const double2*>(ca.Uprev) + (size_t)(n + 1) * Ls + f * NH + ak);
    }
  }
  USTAMP(1)
  if (stage > 0) {
    if constexpr (!TRIAD) {
    // deterministic reduction of the per-pair partials in a fixed order that depends only on the number
    // of partials (not on the CTA size or the owned-mode count, so every schedule agrees bitwise): RQ
    // lanes per item, lane q sums partials q, q+RQ, ... ascending, then a fixed xor tree over the RQ
    // lanes (shuffles inside one warp).  Above 128 partials (the paper's ε = 1e-2 case has 225) RQ = 32 keeps a lane's
    // loads in one round of 8 (one L2 round trip instead of four); up to 128, RQ = 8 (16 lanes would
    // halve the items per round and cost the round trip back: measured on C5's 128)
    constexpr int ITEMS = NOWN * 6;
    const int RQ = ca.nparts <= 128 ? 8 : 32, IPR = T / RQ;  // items per round
    static_assert(T % 32 == 0, "reduction layout");
    for (int it0 = 0; it0 < ITEMS; it0 += IPR) {
      const int it = it0 + tid_ / RQ, qd = tid_ % RQ;
      double2 sacc = make_double2(0.0, 0.0);
      int ak = 0, al = 0, j = 0;
      if (it < ITEMS) entry(it / 6, it % 6, ak, al, j);
      if (it < ITEMS && ak <= K) {
        const size_t e0 = (size_t)al * Kc + j;
        for (int b0 = qd; b0 < ca.nparts; b0 += 8 * RQ) {  // 8 independent L2 loads in flight, summed in order
          double2 buf[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int b = b0 + u * RQ;
            buf[u] = b < ca.nparts ? __ldcg(ax.part(e0 + (size_t)b * 3 * Kc)) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) sacc = cadd(sacc, buf[u]);
        }
      }
      for (int w = RQ / 2; w > 0; w >>= 1) {
        sacc.x += __shfl_xor_sync(0xffffffffu, sacc.x, w);
        sacc.y += __shfl_xor_sync(0xffffffffu, sacc.y, w);
      }
      if (it < ITEMS && qd == 0) kk[it] = sacc;
    }
    USTAMP(2)
#ifdef RSW_REDUCE_PROBE
    {  // debug: the same loads again (hot in L2, code hot in the i-cache): is the first round slow?
      double sink = 0.0;
      for (int it0 = 0; it0 < ITEMS; it0 += IPR) {
        const int it = it0 + tid_ / RQ, qd = tid_ % RQ;
        int ak = 0, al = 0, j = 0;
        if (it < ITEMS) entry(it / 6, it % 6, ak, al, j);
        if (it < ITEMS && ak <= K) {
          const size_t e0 = (size_t)al * Kc + j;
          for (int b0 = qd; b0 < ca.nparts; b0 += 8 * RQ) {
            double2 buf[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int b = b0 + u * RQ;
              buf[u] = b < ca.nparts ? __ldcg(ax.part(e0 + (size_t)b * 3 * Kc)) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) sink += buf[u].x;
          }
        }
      }
      if (sink == 1.2345e300) kk[0].x = sink;
    }
    USTAMP(9)
#endif
    }  // !TRIAD (the triad stage phase wrote kk whole)
    grp.sync();
    USTAMP(3)
    if (tid_ < NOWN * 6) {
      int ak, al, j;
      const int it = tid_;
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
    USTAMP(4)
    if (!last) {
      push_stage_input<N, NOWN, T, GRP, AX, TRIAD ? TRIAD_NB : 3>(ax, yv, yidx, ucount, grp);
      USTAMP(5)
      return;
    }
    grp.sync();
    USTAMP(5)
    // finalize: D half step, back-transform, primitive G, parareal update (thread per (o, f))
    if (tid_ < NOWN * 3) {
      const int o = tid_ / 3, f = tid_ % 3, ak = rank + o * P;
      if (ak <= K) {
        // (gsm: the owned modes' constants staged in shared memory by the caller, owned_consts)
        const double a = gsm ? gsm[o * 8] : __ldg(ca.g.a + ak), p = gsm ? gsm[o * 8 + 1] : __ldg(ca.g.p + ak),
                     q = gsm ? gsm[o * 8 + 2] : __ldg(ca.g.q + ak);
        const double dh = gsm ? gsm[o * 8 + 3] : __ldg(ca.dhalf + ak);
        // e^{-iωΔT/ε}: α=+1 entry of e^{-(ΔT/ε)L̂} (R3)
        const double2 bt = gsm ? make_double2(gsm[o * 8 + 4], gsm[o * 8 + 5]) : __ldg(ca.back + ak);
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
        nd_s[tid_ * 2] = wk * (d.x * d.x + d.y * d.y);
        nd_s[tid_ * 2 + 1] = wk * (un.x * un.x + un.y * un.y);
        *Gst = g;
        *Uo = un;
        un_s[tid_] = un;
        if (ak == K) {  // modes K < k <= N/2 stay zero: written after the next stage input is out (zero_tail)
          zU = Uo;
          zG = Gst;
        }
      }
    }
    grp.sync();
    if (ca.rparts && tid_ < NOWN) {
      const int ak = rank + tid_ * P;
      if (ak <= K) {
        const double* t = nd_s + tid_ * 6;
        ca.rparts[((size_t)n * (K + 1) + ak) * 2 + 0] = t[0] + t[2] + t[4];
        ca.rparts[((size_t)n * (K + 1) + ak) * 2 + 1] = t[1] + t[3] + t[5];
      }
    }
    USTAMP(6)
    if (n + 1 >= ca.n_end) {  // no next slice
      zero_tail();
      return;
    }
  } else {
    // stage 0: load U_0 of owned modes
    if (tid_ < NOWN * 3) {
      const int o = tid_ / 3, f = tid_ % 3, ak = rank + o * P;
      if (ak <= K) un_s[tid_] = reinterpret_cast<const double2*>(ca.U)[(size_t)n * Ls + f * NH + ak];
    }
    grp.sync();
  }
  // first stage input of the next slice: v = e^{ΔT D̂/2} u (Alg.2), eigen, both signs of κ
  if (tid_ < NOWN * 6) {
    int ak, al, j;
    const int it = tid_, o = it / 6, e = it % 6;
    entry(o, e, ak, al, j);
    if (ak <= K && !(ak == 0 && e >= 3)) {
      const double a = gsm ? gsm[o * 8] : __ldg(ca.g.a + ak), p = gsm ? gsm[o * 8 + 1] : __ldg(ca.g.p + ak),
                   q = gsm ? gsm[o * 8 + 2] : __ldg(ca.g.q + ak);
      double2 u[3], c[3];
#pragma unroll
      for (int f = 0; f < 3; ++f) u[f] = (e < 3) ? un_s[o * 3 + f] : cconj(un_s[o * 3 + f]);
      to_eigen(e < 3 ? a : -a, p, q, u, c);
      const double2 v = cscale(c[al], gsm ? gsm[o * 8 + 3] : __ldg(ca.dhalf + ak));
      Vs[it] = v;
      yv[it] = v;
      yidx[it] = al * Kc + j;
    } else {
      yidx[it] = -1;
    }
  }
  USTAMP(7)
  push_stage_input<N, NOWN, T, GRP, AX, TRIAD ? TRIAD_NB : 3>(ax, yv, yidx, ucount, grp);
  zero_tail();
  grp.sync();
  USTAMP(8)
#undef USTAMP
}

// LEAN (triad sweeps): no FFT buffers or twiddles (X, Y, TW empty); A holds the triad half-sums, PH the
// frame rotation
template <int N, int R, int T, int NOWN, int NPC = 1, int SPLIT = 1, bool LEAN = false>
struct CoarseLayout {  // dynamic shared memory of a coarse-sweep CTA (double2 units, then doubles); NPC cached pairs
  static constexpr int K = N / 3, Kc = 2 * K + 1, KP = K + 1, NR = (T > NOWN * 6 ? T : NOWN * 6);
  static constexpr int X = 0, Y = LEAN ? 0 : X + 3 * N, TW = LEAN ? 0 : X + SPLIT * 6 * N,
                       C = TW + (LEAN ? 0 : fft_tw_size<N, R>()), A = C + 3 * Kc,
                       VS = A + 3 * Kc, KS = VS + NOWN * 6, KK = KS + NOWN * 6, UN = KK + NOWN * 6,
                       RDB = UN + NOWN * 3, PH = RDB + T, YV = PH + NPC * 2 * KP, D = YV + NOWN * 6;
  static constexpr int RED = 0, GA = RED + NR, GP = GA + KP, GQ = GP + KP, SW = GQ + KP, YI = SW + 2 * NPC,
                       ND = YI + NOWN * 6;  // YI: int entry indices stored in double slots
  static constexpr size_t bytes = sizeof(double2) * D + sizeof(double) * ND;
};

}  // namespace rsw
