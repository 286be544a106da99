// rsw_internal.h — internal structs shared by the kernels (rsw_k_*.cu, rsw_pipeline.cu) and the host library
// (rsw_capi.cu).  Not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rsw_device.cuh"

namespace rsw {

// ETDRK4 / Strang per-mode diagonal coefficients in the eigenbasis (K6 host tables):
//   cp[i][|κ|] : α=+1 value (complex), α=-1 is its conjugate;  c0[i][|κ|] : α=0 value (real)
//   i = 0 E=e^{z}, 1 E2=e^{z/2}, 2 Q=(h/2)φ1(z/2), 3 f1=h(φ1-3φ2+4φ3)(z), 4 f2=h(2φ2-4φ3)(z),
//   5 f3=h(4φ3-φ2)(z);  z = h λ_α,  λ_α = -iαω/ε - μκ^4.
struct FineTab {
  ModeGeom g;
  const double2* cp;
  const double* c0;
  const double2* tw;  // e^{-2πi m/N}, m = 0..N-1
};

// Averaging tables: w[m] (m = 0..M-1, w[0] = 0), phase[m][|κ|] = e^{iω_κ τ_m} (m = 0..M)
struct AvgTab {
  ModeGeom g;
  const double* w;
  const double2* phase;
  const double2* tw;
  const double* triad = nullptr;      // triad coefficients W (rsw_blocks.cuh), or null: the M-sample quadrature
  const double2* triad_ph = nullptr;  // e^{iω_k τ_c}, k = 0..K: the triad form's frame rotation
};

// Arguments of the coarse combine kernel (one state chain)
struct CoarseArgs {
  ModeGeom g;
  const double2* part;  // [nparts][3][Kc]  one partial per sample pair
  int nparts;           // sample pairs M/2
  int scheme;           // 0 RK4, 1 midpoint
  double dT;
  const double* dhalf;  // e^{-μκ^4 ΔT/2}
  const double2* back;  // e^{-iω ΔT/ε}
  double2* v;           // [3][Kc]
  double2* ks;          // [3][Kc]
  double2* y;           // [3][Kc]
  double2* yin;         // [3][3][Kc] triple-buffered stage input (sentinel = not yet written)
  double* U;            // [S+1][3][N/2+1][2] (chain states, written)
  double* G;            // [S][3][N/2+1][2] (G(U_n) of this sweep, written)
  const double* Uprev;  // previous iterate U^{k-1} (residual); == U for the in-place classic sweep
  const double* Gprev;  // G(U^{k-1}_n) of the previous sweep; == G for the in-place classic sweep
  const double* F;      // [S][...] or null (k = 0 sweep / plain coarse step)
  const unsigned* wprog;  // pipelined: progress counter of the previous sweep (>= wunit*(n+1): slice n done), or null
  unsigned wunit;
  const unsigned* wF;     // pipelined: done flags of the previous iteration's fine pairs, or null
  unsigned* wd;           // pipelined: watchdog flag (set when a wait times out), or null
  const unsigned* hb;     // pipelined: progress heartbeat read by the watchdog, or null
  int wsys;               // pipelined multi-GPU: wF flags are released by other GPUs (system-scope acquire)
  const int* stopk;       // pipelined: first stopped iteration (waits of sweep kself > *stopk give up), or null
  int kself;
  double* rparts;       // [S][K+1][2] residual partials or null
  int n_end;            // number of chain steps (S)
  unsigned long long* prof;  // optional phase timestamps (CTA 0; RSW_PROFILE_COARSE=1), else null
};

constexpr int kMaxPeers = 8;  // ranks of one NVSwitch node
// stage-input ring depth of the triad coarse sweeps (rsw_blocks.cuh); the exchange arrays always hold
// this many stage-input buffers (the quadrature sweeps use the first three)
#ifndef RSW_TRIAD_NB
#define RSW_TRIAD_NB 16
#endif
constexpr int TRIAD_NB = RSW_TRIAD_NB;  // power of two >= 8 (ring reset distance NB/2, fence every NB/4 publications)
__host__ __device__ constexpr unsigned yin_pages(int n) { return (TRIAD_NB * 3u * (2u * (unsigned)(n / 3) + 1u) + 255u) / 256u; }

// triad coefficient table of N̄ (rsw_blocks.cuh triad_stage_phase, rsw_capi.cu build_triad)
constexpr int TRIAD_E = 18;
__host__ __device__ constexpr int triad_nk(int kap, int K) { return 2 * K + 1 - kap; }
__host__ __device__ constexpr long long triad_rows_before(int kap, int K) {
  return (long long)kap * (2 * K + 1) - (long long)kap * (kap - 1) / 2;
}
// double2 entries of the owned blocks of rank (κ = rank + o P, o < nown) — the CTA's shared-memory copy
__host__ __device__ inline size_t triad_local_entries(int K, int rank, int P, int nown) {
  size_t s = 0;
  for (int o = 0; o < nown; ++o) {
    const int kap = rank + o * P;
    if (kap > K) break;
    s += (size_t)TRIAD_E * triad_nk(kap, K);
  }
  return s;
}

// L2 die homing.  A B200 is two dies, each with its own L2; every 4 KB page of device
// memory is homed on one of them, and a flag / data hand-off between two SMs is about twice as fast
// (round trip ~2300 vs ~4400 cycles, tools/micro/pingpong.cu) when both SMs sit on the die that homes
// the page.  Inside a 2 MB chunk (one physical page of the allocation) the home die of 4 KB page i
// (0..511) is the parity of i & 0x1EF — every page-index bit but bit 4 (address bit 16) — XOR a
// per-chunk constant (a GF(2) fit with no error over all 512 pages of four chunks,
// tools/micro/pingpong.cu scan).  A HomedArena is a 2 MB-aligned run of chunks addressed through the
// pages homed on one die: logical page q -> chunk q / 256, page pair r = q % 256, page 2r or 2r+1 —
// whichever has hash parity (kmask >> chunk) & 1 (bit c = the parity this die homes in chunk c,
// measured by k_die_probe).
struct HomedArena {
  char* base;
  unsigned long long kmask;
  int flat = 0;  // 1: logical page q is physical page q (both dies' pages interleaved, no homing)
};
// logical page q of arena h (host and device)
__host__ __device__ __forceinline__ char* homed_page(const HomedArena& h, unsigned q) {
  if (h.flat) return h.base + ((size_t)q << 12);
  const unsigned c = q >> 8, r = q & 255u;
#ifdef __CUDA_ARCH__
  const unsigned pc = __popc(r & 0xF7u);  // hash parity of page 2r (= parity of 2r & 0x1EF)
#else
  const unsigned pc = (unsigned)__builtin_popcount(r & 0xF7u);
#endif
  const unsigned pidx = 2u * r + ((pc ^ (unsigned)(h.kmask >> c)) & 1u);
  return h.base + ((size_t)c << 21) + ((size_t)pidx << 12);
}
constexpr int kMaxDieGroups = 32;  // coarse groups per die with die-aware placement

// Pipelined parareal (rsw_pipeline.cu): every iteration's buffers stay resident
struct PipeArgs {
  CoarseArgs base;      // geometry, scheme, dT, D half step, back-transform (per-sweep pointers set in-kernel)
  AvgTab at;
  FineTab ft;
  int S, K, M, m_fine, NG, GC, npairs;
  double h, tol;
  double* Uall;         // [K+1][S+1][state]   U^k (row 0 = u0)
  double* Gall;         // [K+1][S][state]     G(U^k_n)
  double* Fall;         // [K][S][state]       F(U^k_n)
  double* rparts;       // [K+1][S][K_modes+1][2]
  double* resid;        // [K+1]               r_k
  unsigned* prog;       // [K+1]   sweep progress (CTA-slices finalized)
  unsigned* doneF;      // [K][npairs] fine pair done flags
  unsigned* next;       // [K]     next unclaimed fine pair per iteration
  int* stopk;           // first iteration that stopped the run (K+1: none)
  unsigned* wd;         // watchdog flag
  unsigned* hb;         // progress heartbeat (fine steps, coarse slices): waits time out only without progress
  unsigned* ticket;     // role tickets
  unsigned* gbar;       // [NG][32] group barrier counters
  double2* ybuf;        // [NG][3][3Kc] stage inputs
  double2* part;        // [NG][GC][3Kc] partial sums
  unsigned long long* trace;  // optional timeline (RSW_PIPE_TRACE): sweep [K+1][2], slice [K+1][S], fine [K][npairs][2]
  unsigned long long* stamps; // always: sweep start / end [K+1][2] (globaltimer ns), fine-task latency sum, count
  // multi-GPU pipelined schedule: this rank runs every sweep (replicated) but only the fine tasks of its
  // slice shard, pairs [pair_lo, pair_hi), and pushes each finished pair to the peers' Fall over NVLink
  // (IPC-mapped), releasing the peer's doneF flag at system scope; one GPU: [0, npairs), no peers
  int pair_lo, pair_hi, npeers;
  double* const* peerF;         // device array [npeers]: the peers' Fall
  unsigned* const* peerDoneF;   // device array [npeers]: the peers' doneF
  // coarse groups' exchange arrays (barrier counter, stage inputs, partials) in die-homed pages: group
  // on die d, slot i (i-th group of that die) owns logical pages [i GP, (i+1) GP) of arena[d].  With
  // die_aware, a CTA takes its coarse role from a per-die ticket (dticket[d]) so every CTA of a group
  // sits on the die that homes its arrays (diemask: bit s = SM s on die 1); otherwise group g uses
  // die g & 1, slot g >> 1 and CTAs take roles from the global ticket.
  HomedArena arena[2];
  int die_aware;
  unsigned long long diemask[3];
  int ndg[2];
  signed char dg[2][kMaxDieGroups];  // group id of slot i on die d
  unsigned* dticket;                 // [2]
  size_t wsm;                        // triad sweeps (at.triad != null): shared-memory bytes of the largest owned-block copy
  int extra_fine;                    // CTAs without a coarse role run a second fine group on their coarse threads
  int extra_young;                   // ... which claims the most recently ready task (not the oldest)
  int coarse_solo;                   // CTAs with a coarse role run no fine group (RSW_PIPE_COARSE_SOLO=1)
};
bool pipeline_supported(int n);
cudaError_t launch_parareal_pipe(int n, const PipeArgs& a, int fine_scheme, int grid, size_t* out, cudaStream_t st);

// Fine-sweep outputs also stored straight into other GPUs' buffers (multi-GPU bulk schedule: the
// exchange of the fine endpoints fused into the fine kernel's epilogue; NVLink stores to IPC-mapped
// memory).  out[r] receives the same slices at the same offsets as the local output.
struct PeerOut {
  int n;
  double* out[kMaxPeers];
};
cudaError_t launch_fine(int n, int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                        const FineTab& tab, cudaStream_t st, const PeerOut* po = nullptr);
cudaError_t launch_nonlinear(int n, const double* in, double* out, int S, const FineTab& tab, cudaStream_t st);
cudaError_t launch_avg_states(int n, const double* in, double* out, int S, int M, const AvgTab& tab,
                              cudaStream_t st);
// Bulk coarse sweep placement: its exchange arrays (barrier counter page, stage-input pages, partial
// pages) in arena[d] pages; with die_ok and at most die_n[d] CTAs the sweep runs on die d only (every
// SM gets one CTA, the CTAs on die d take ranks from *ticket, the others exit at once), so every
// hand-off of the serial chain stays inside one die's L2.  A sweep on both dies uses
// the arena flat (pages of both dies interleaved: homing all of it on one die measured slower).
struct SweepPlace {
  HomedArena arena[2];
  unsigned bpage, ypage, ppage;
  int die_ok, die_n[2];
  unsigned long long diemask[3];
  unsigned* ticket;  // zeroed by the launcher
};
// pages of the bulk sweep's exchange arrays (barrier, stage inputs, partials) for n, M
unsigned sweep_pages(int n, int M);
cudaError_t launch_coarse_sweep(int n, const CoarseArgs& ca, const AvgTab& tab, int M, const SweepPlace& pl,
                                double* r_out, int* grid_used, int* die_used, cudaStream_t st);
cudaError_t launch_strang_sweep(int n, const FineTab& tab, double h, double* U, double* G, const double* F,
                                double* Gnew, int S, double* r_out, cudaStream_t st);
cudaError_t launch_dfma_peak(double* out, int blocks, int iters, cudaStream_t st);
// L2 die-homing probe (one CTA per SM, cooperative): res[0, nb) = smid of block b; res[nb + 2x + p] =
// master-side cycles per round trip between block 0 and block x through page p of chunk 0;
// res[3 nb + 6c + 2v + p] = the same with the first same-die partner through page 2r + p of chunk c
// (r = 0, 8, 200 for v = 0, 1, 2).  arena: nch 2 MB-aligned chunks; ctl: nb + 2 zeroed words.
cudaError_t launch_die_probe(char* arena, int nch, unsigned* ctl, long long* res, int nb, int rounds, cudaStream_t st);
// bad[0] |= any non-zero mode k > n/3, bad[1] |= any Im û_0 != 0, over n_states states
cudaError_t launch_check_states(int n, const double* u, int n_states, unsigned* bad, cudaStream_t st);

}  // namespace rsw
