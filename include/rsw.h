/*
 * rsw.h — C-ABI of librsw.so: the B200-native (sm_100a) hot path of the asymptotic parareal
 * method for the 1-D rotating shallow water (RSW) equations, arxiv 1303.6615.
 *
 *   u_t + ε^{-1} L u = N(u) + D u,   u = (v1, v2, h) on the periodic domain [0, 2π)
 *                                                    (Eq. full eqn; RSW P:1045-1095)
 *
 * Citations "P:n" are lines of /root/reference/PAPER.md; "R#" are the readings listed in
 * DESIGN.md §3 (where the paper is silent, ambiguous or garbled).
 *
 * ----------------------------------------------------------------------------------------------
 * STATE LAYOUT (every state argument):
 *   double[batch][3][n/2+1][2]  — field-major (v1, v2, h), wavenumber k = 0..n/2, (re, im).
 *   û_k = (1/n) Σ_j u_j e^{-ikx_j}, x_j = 2πj/n (so k = 0 is the mean).  Real fields (R16):
 *   Im(û_0) must be 0.  Dealiasing (R10): modes k > n/3 must be 0 on input and are 0 on output.
 *   parareal_iterate checks u0 on the device (it synchronises anyway) and returns RSW_ERR_CONFIG on a
 *   violation; rsw_check_states performs the same check for any batch (synchronous).  The purely
 *   asynchronous entry points (fine / averaged / coarse / nonlinear) do not check: the Python
 *   binding calls rsw_check_states before them unless told not to.
 *
 * MEMORY: all state pointers are DEVICE pointers (caller-owned, e.g. torch CUDA tensors),
 *   8-byte aligned, on the current device, unless a parameter says "host".
 *   The library never retains a caller pointer after a call returns.  It caches per-configuration
 *   coefficient tables and workspace (keyed by every parameter that affects them) until
 *   rsw_shutdown().
 * STREAMS: `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All work
 *   is enqueued on it; only parareal_iterate synchronises (once per iteration, to read r_k).
 * ERRORS: every argument is validated before any launch; no exceptions cross the ABI;
 *   rsw_last_error() returns a thread-local message describing the last non-OK status.
 * There is NO CPU fallback: a call that cannot run on the GPU returns RSW_ERR_CUDA.
 * ----------------------------------------------------------------------------------------------
 */
#ifndef RSW_H_
#define RSW_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Physical parameters: ε Rossby number, F (Froude = F^{1/2} ε), μ hyperviscosity
   (D̂(k) = -μk^4, sign R2), n = grid points = FFT length (power of two, 16..1024; the cap is
   reading R18 of DESIGN.md: the largest BASELINE configuration is n = 1024 and the on-chip layout of
   a state pair — three packed fields plus the product buffer, 4(n + n/16) complex — fits one CTA's
   shared memory only up to n = 1024 next to the coefficient tables). */
typedef struct {
  double eps, F, mu;
  int32_t n;
} rsw_params;

typedef enum {
  RSW_OK = 0,
  RSW_ERR_CONFIG = 1,     /* invalid argument (nothing was launched) */
  RSW_NOT_CONVERGED = 2,  /* parareal: tol > 0 and no r_k < tol within max_iters (U valid) */
  RSW_ERR_DIVERGED = 3,   /* parareal: r_k non-finite or > 1e6 (SPEC S:399 guard) */
  RSW_ERR_CUDA = 4,
  RSW_ERR_NCCL = 5
} rsw_status;

enum { RSW_FINE_ETDRK4 = 0, RSW_FINE_STRANG = 1, RSW_FINE_IFRK4 = 2 };
/* RSW_FINE_IFRK4: integrating-factor baseline ("operator integrating factor method",
   P:1215-1219): classical RK4 on v = e^{-tA} u (Lawson form, forward factors only),
   u+ = E u + h/6 (E k1 + 2 E2 k2 + 2 E2 k3 + k4). */
enum { RSW_COARSE_RK4 = 0, RSW_COARSE_MIDPOINT = 1, RSW_COARSE_STRANG = 2 };
/* RSW_COARSE_STRANG: standard parareal — the coarse solver is one Strang step of
   size dT on the full equation (Alg.3 with m = 1); T0 and M are then ignored. */
enum { RSW_FLAG_LINEAR_ONLY = 1u }; /* N ≡ 0: exact-linear test mode only */

/* Layout check (STATE LAYOUT above; R10, R16) of n_states device states u: RSW_ERR_CONFIG if any
   mode k > n/3 is non-zero or any Im(û_0) != 0, RSW_OK otherwise.  Synchronises `stream`. */
rsw_status rsw_check_states(const rsw_params* p, int32_t n_states, const double* u, void* stream);

/* Device topology used by the coarse sweeps' placement: die_sms[d] = the SMs on die d
   of the current device (die 0 = the probe master's die), *probed = 1 when the die-homing probe found
   two dies and the page hash, 0 when placement is off (then die_sms = {SM count, 0}).  Runs the probe
   (one cooperative launch, ~5 ms) on first use; synchronous; die_sms: HOST int32[2]. */
rsw_status rsw_device_topology(int32_t* die_sms, int32_t* probed);

/* N(u) = -(v1 ∂x v1, v1 ∂x v2, ∂x(h v1)) for n_states independent states, evaluated
   pseudo-spectrally (inverse FFT -> pointwise products -> FFT, 2/3 rule).
   Operator table, sign R1.  u_in and out must not alias.
   (The inner kernel of every other entry point, exposed for parity tests.) */
rsw_status rsw_nonlinear(const rsw_params* p, int32_t n_states, const double* u_in, double* out,
                         void* stream);

/* Fine propagator φ_ΔT (the parfor of Alg.4): each of n_slices independent states is
   advanced by dT with m = ceil(dT/dt - 1e-9) steps of dt_eff = dT/m (R9) of
     scheme RSW_FINE_ETDRK4: ETDRK4 (Cox & Matthews 2002; cited P:1168-1169), or
     scheme RSW_FINE_STRANG: Strang splitting, Alg.3 P:518-548 with the explicit midpoint (R7),
   the linear part e^{hA}, A = -L̂/ε + D̂ (R3), applied exactly per wavenumber in the eigenbasis of
   L̂.  flags: RSW_FLAG_LINEAR_ONLY.  u_in == u_out is allowed (in-place). */
rsw_status rsw_fine_propagate(const rsw_params* p, int32_t scheme, uint32_t flags, double dT,
                              double dt, int32_t n_slices, const double* u_in, double* u_out,
                              void* stream);

/* HMM averaged nonlinearity (Eq. numerical average, discretized P:289-293; ε-scaled form P:313;
   Alg.1; kernel ρ P:383-390), for n_states independent states:
     N̄(v) = Σ_{m=1}^{M-1} w_m e^{τ_m L̂} N(e^{-τ_m L̂} v),  τ_m = s_m/ε, s_m = T0 m/M  (R4),
     w_m = ρ(m/M) / Σ_j ρ(j/M),  ρ(s) = exp(-1/(s(1-s)))  (R5).
   The sum over samples is evaluated in ascending m (deterministic).  For n <= 512 the sum is taken in
   triad form (rsw_triad_coefficients: the same quadrature sum, reordered exactly; RSW_COARSE_TRIAD=0
   selects the per-sample pseudo-spectral evaluation).  rhs_out must not alias. */
rsw_status rsw_averaged_rhs(const rsw_params* p, double T0, int32_t M, int32_t n_states,
                            const double* u_in, double* rhs_out, void* stream);

/* Triad coefficients of N̄ (HOST output).  The paper writes the averaged nonlinear term as
   a sum over wavenumber triads with interaction coefficients; with Alg.1's quadrature
   (the same w_m, τ_m as rsw_averaged_rhs) the eigen coordinates (c-, c0, c+) of N̄ are
     N̄^γ_κ = Σ_{κ1=κ-K}^{K} Σ_{α=±1} Σ_{β=-1,0,1} Φ(γω_κ - αω_{κ1} - βω_{κ2}) C^{γαβ}_{κκ1κ2} c^α_{κ1} c^β_{κ2},
     Φ(λ) = Σ_{m=1}^{M-1} w_m e^{iλτ_m},   κ2 = κ - κ1,   κ = 0..K = n/3,
   in the eigenbasis r^∓ = (∓iω, 1, ia)/(√2ω), r^0 = (0, ia, 1)/ω, a = κ/√F, ω = √(1+a²).
   The window is symmetric, so Φ(λ) = e^{iλτ_c} R(λ) with τ_c = T0/(2ε) and R real; each C^{γαβ} is
   purely real when (γ = 0) == (β = 0) and purely imaginary otherwise.  `out` receives ONE double per
   coefficient, W' = R(λ) C (its real part, or its imaginary part for the imaginary ones), for the
   contraction in the rotated frame: c'^α_k = c^α_k e^{-iαω_k τ_c},  N̄^γ_κ = e^{iγω_κ τ_c} Σ W' c' c'
   (× i for the imaginary ones).  Layout: block κ = 0..K starts at 18 (κ(2K+1) - κ(κ-1)/2); inside it
   entry e = (γ+1) 6 + (α > 0) 3 + (β+1) of row i (κ1 = κ - K + i, i = 0..2K-κ) is at e (2K+1-κ) + i.
   The coarse sweeps (rsw_coarse_propagate, parareal_iterate) evaluate N̄ in this form (pipelined
   schedule n <= 256, bulk any n), rsw_averaged_rhs for n <= 512 (environment RSW_COARSE_TRIAD=0: the
   M-sample quadrature everywhere).  *count receives the number of doubles; out may be NULL (size
   query).  Pure host computation (no GPU needed); RSW_ERR_CONFIG on bad parameters. */
rsw_status rsw_triad_coefficients(const rsw_params* p, double T0, int32_t M, double* out, int64_t* count);

/* Coarse propagator φ̄_ΔT (Alg.2, φ̄ P:415-417) for n_states independent states:
     v = e^{ΔT D̂/2} u;  one RK4 (R6; or midpoint, RSW_COARSE_MIDPOINT) step of size dT on v' = N̄(v);
     v = e^{ΔT D̂/2} v;  G(u) = e^{-(ΔT/ε) L̂} v   (back-transform sign R3).
   u_in == u_out is allowed. */
rsw_status rsw_coarse_propagate(const rsw_params* p, int32_t coarse_scheme, double dT, double T0,
                                int32_t M, int32_t n_states, const double* u_in, double* u_out,
                                void* stream);

/* Schedule of the parareal iteration (results are bitwise identical; only the order of the work
   differs):
     RSW_SCHEDULE_AUTO      pipelined when supported (n in {64, 128, 256}, coarse RK4 or midpoint, enough
                            co-resident CTAs for its coarse groups; multi-GPU: see below), bulk otherwise;
     RSW_SCHEDULE_BULK      per iteration: the fine sweep over all slices, then the serial coarse sweep;
     RSW_SCHEDULE_PIPELINED one persistent kernel in which sweep k trails sweep k-1 slice by slice and
                            each fine solve F(U^k_n) starts as soon as U^k_n exists (SURVEY
                            NEXT-3); RSW_ERR_CONFIG if the configuration is not supported. */
enum { RSW_SCHEDULE_AUTO = 0, RSW_SCHEDULE_BULK = 1, RSW_SCHEDULE_PIPELINED = 2 };

typedef struct {
  double dT, dt, T0, tol;
  int32_t M, n_slices, max_iters, fine_scheme, coarse_scheme;
  int32_t schedule; /* RSW_SCHEDULE_* */
} parareal_config;

typedef struct rsw_comm rsw_comm; /* opaque; NULL = single GPU */

/* Optional per-call statistics (may be NULL).  Times are device-measured (CUDA events) ms. */
typedef struct {
  double fine_ms, comm_ms, coarse_ms, total_ms;
  int64_t fine_slice_steps; /* slice-steps advanced by THIS rank's fine sweeps */
  int64_t kernel_launches;  /* kernels this library launched during the call (the u0 layout check included) */
  int32_t pipelined;        /* 1: the pipelined schedule ran (fine / coarse times overlap: only
                               total_ms is meaningful, fine_ms = coarse_ms = total_ms) */
  /* phase split of the time to solution (P:718-725 cost terms).  Pipelined: sweep0_ms = the k = 0
     coarse sweep, lag_ms = mean time each further iteration adds (sweep k end - sweep k-1 end),
     fine_task_ms = mean latency of one fine pair task (in-kernel globaltimer stamps).  Bulk:
     sweep0_ms = the k = 0 sweep, lag_ms = one iteration (fine sweep + exchange + coarse sweep),
     fine_task_ms = one fine sweep of this rank's shard. */
  double sweep0_ms, lag_ms, fine_task_ms;
  /* pipelined: coarse groups (concurrent sweeps) and CTAs per group; die_aware = 1 when every group's
     CTAs sit on one die of the GPU with the group's exchange arrays homed in that die's L2 (probed
     once per workspace) */
  int32_t coarse_groups, group_ctas, die_aware;
  /* 1: the coarse sweeps evaluated N̄ in triad form (rsw_triad_coefficients), 0: M-sample quadrature */
  int32_t coarse_triad;
} rsw_parareal_stats;

/* The asymptotic parareal iteration (Eq. HMM parareal iteration P:428-430; Alg.4):
     k = 0:  U_0 = u0, U_{n+1} = G(U_n), n = 0..S-1;
     k >= 1: F_n = F(U^{k-1}_n) in parallel (this rank's shard, then an all-gather over `comm`);
             serial sweep U^k_{n+1} = G(U^k_n) + (F_n - G_n), G_n <- G(U^k_n)   (R13, R14);
             r_k = max_{n=1..S} ||U^k_n - U^{k-1}_n|| / ||U^k_n||  (relative L2, R12).
   u0: device [3][n/2+1][2].  U: device [S+1][3][n/2+1][2] (replicated, bitwise identical on every
   rank).  resid_hist: HOST double[max_iters].  iters_done: HOST.  tol <= 0: run exactly
   max_iters iterations; tol > 0: stop at the first r_k < tol (RSW_NOT_CONVERGED if none).
   Requires 0 <= max_iters <= n_slices and n_slices divisible by the comm world size.
   u0 is layout-checked on the device first (RSW_ERR_CONFIG on a violation).  Bulk schedule with a
   communicator of world > 1: the fine kernel stores rank r's block [lo_r, hi_r) (rsw_shard_range)
   straight into every peer's F at offset lo_r (NVLink stores to IPC-mapped memory, between two
   stream barriers); RSW_ALLGATHER=1, or a world-1 communicator, uses an in-place ncclAllGather.
   RSW_BULK_MIRROR=1 (one GPU, tests): the fine kernel also stores into a same-GPU copy of F, which
   is returned as F_out.
   Testing: with comm == NULL and the environment variable RSW_VIRTUAL_WORLD=P (P <= 16), the fine
   sweep runs as P separate shard launches into P separate shard buffers, and F is assembled from them
   with one copy per shard at offset lo_r; results must be bitwise equal to P = 1.
   Schedule knobs (results bitwise identical under all of them): RSW_PIPELINE=0 (auto → bulk),
   RSW_PIPE_GC / RSW_PIPE_NG (coarse sub-CTAs per sweep / concurrent sweeps), RSW_PIPE_TRACE=1
   (timeline to stderr), RSW_PIPE_MIRROR=1 (one GPU: also push every fine pair into a same-GPU copy of
   F, the multi-GPU store path, checked against F).  The pipelined schedule's dependency waits give up
   (RSW_ERR_CUDA) only after RSW_WATCHDOG_MS (default 4000) ms without ANY progress in the kernel (a
   heartbeat bumped by fine steps and coarse slices).
   Multi-GPU (comm with world > 1): AUTO / PIPELINED run the pipelined schedule when n <= 256 and
   n_slices is divisible by 2 x world (every rank runs the replicated sweeps and its shard's fine
   tasks, pushing each finished pair into the peers' F over NVLink: IPC-mapped buffers, system-scope
   release / acquire); otherwise the bulk schedule with the in-place all-gather.
   Workspace: calls on different streams are ordered by an event the library records at the end of
   each call, so they never overlap on the shared per-device workspace. */
rsw_status parareal_iterate(const rsw_params* p, const parareal_config* cfg, const double* u0,
                            double* U, double* resid_hist, int32_t* iters_done, rsw_comm* comm,
                            void* stream);

/* As parareal_iterate, additionally returning the last iteration's fine endpoints F_n and coarse
   values G_n (device [S][3][n/2+1][2] each; either may be NULL) and statistics (host; may be
   NULL). */
rsw_status parareal_iterate_ex(const rsw_params* p, const parareal_config* cfg, const double* u0,
                               double* U, double* resid_hist, int32_t* iters_done, rsw_comm* comm,
                               void* stream, double* F_out, double* G_out,
                               rsw_parareal_stats* stats);

/* Checkpoint / resume: the state {U^k, G(U^k_n), k} determines the continuation of the
   iteration.  A checkpoint is the U and G_out of a parareal_iterate_ex call that ran k iterations;
   parareal_resume continues from it with iterations k_done+1 .. cfg->max_iters (bulk schedule): U
   (device [S+1][3][n/2+1][2]) is read as U^{k_done} and overwritten with the result, G_in (device
   [S][3][n/2+1][2]) holds G(U^{k_done}_n).  resid_hist (host) receives the residuals of the
   iterations run here (cfg->max_iters - k_done entries), *iters_done the total count.  The result is
   bitwise that of one uninterrupted bulk run of max_iters iterations.  RSW_ERR_CONFIG for
   k_done < 0, k_done > max_iters, a NULL G_in or schedule = RSW_SCHEDULE_PIPELINED. */
rsw_status parareal_resume(const rsw_params* p, const parareal_config* cfg, double* U, const double* G_in,
                           int32_t k_done, double* resid_hist, int32_t* iters_done, rsw_comm* comm,
                           void* stream, double* F_out, double* G_out, rsw_parareal_stats* stats);

/* Slices owned by `rank` of `world` in the fine sweep: [*lo, *hi) (contiguous blocks, §8(e)). */
rsw_status rsw_shard_range(int32_t n_slices, int32_t rank, int32_t world, int32_t* lo,
                           int32_t* hi);

/* NCCL communicator owned by the library (NCCL is loaded at run time).  out128/id128: 128 host
   bytes (ncclUniqueId), created on rank 0 and broadcast by the caller (e.g. torch.distributed). */
rsw_status rsw_nccl_unique_id(void* out128);
rsw_status rsw_comm_init(const void* id128, int32_t rank, int32_t world, rsw_comm** out);
rsw_status rsw_comm_destroy(rsw_comm* comm);

/* Measured FP64 peak of the current device (DFMA chains on every SM, M0 microbenchmark):
   *tflops (host) = 2 * DFMA lanes * iterations / kernel time.  Used as the roofline denominator. */
rsw_status rsw_fp64_peak(double* tflops, void* stream);

/* Analytic flop counts per unit of work, for throughput reporting:
   which = 0: F_N (one N(u)), 1: ETDRK4 step, 2: Strang step, 3: one N̄ sample,
   4: one whole N̄ in triad form (180 flops per (κ, κ1) row: 6 complex products, 18 complex FMAs). */
double rsw_flops_per_unit(int32_t n, int32_t which);

const char* rsw_last_error(void); /* thread-local; never NULL */
void rsw_shutdown(void);          /* frees cached tables and workspace */

#ifdef __cplusplus
}
#endif
#endif /* RSW_H_ */
