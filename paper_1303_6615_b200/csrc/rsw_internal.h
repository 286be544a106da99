// rsw_internal.h — internal structs shared by the kernels (rsw_kernels.cu) and the host library
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
};

// Arguments of the coarse combine kernel (one state chain)
struct CoarseArgs {
  ModeGeom g;
  const double2* part;  // [nparts][3][Kc]
  int nparts;
  int scheme;           // 0 RK4, 1 midpoint
  double dT;
  const double* dhalf;  // e^{-μκ^4 ΔT/2}
  const double2* back;  // e^{-iω ΔT/ε}
  double2* v;           // [3][Kc]
  double2* ks;          // [3][Kc]
  double2* y;           // [3][Kc]
  double2* yin;         // [3][3][Kc] triple-buffered stage input (sentinel = not yet written)
  double* U;            // [S+1][3][N/2+1][2] (chain states)
  double* G;            // [S][3][N/2+1][2]
  const double* F;      // [S][...] or null (k = 0 sweep / plain coarse step)
  double* rparts;       // [S][K+1][2] residual partials or null
  int n_end;            // number of chain steps (S)
  unsigned long long* prof;  // optional phase timestamps (CTA 0; RSW_PROFILE_COARSE=1), else null
};

cudaError_t launch_fine(int n, int scheme, bool lin, const double* in, double* out, int S, int m, double h,
                        const FineTab& tab, cudaStream_t st);
cudaError_t launch_nonlinear(int n, const double* in, double* out, int S, const FineTab& tab, cudaStream_t st);
cudaError_t launch_avg_states(int n, const double* in, double* out, int S, int M, const AvgTab& tab,
                              cudaStream_t st);
cudaError_t launch_coarse_sweep(int n, const CoarseArgs& ca, const AvgTab& tab, int M, unsigned* bar, double* r_out,
                                int* grid_used, cudaStream_t st);
cudaError_t launch_strang_sweep(int n, const FineTab& tab, double h, double* U, double* G, const double* F,
                                double* Gnew, int S, double* r_out, cudaStream_t st);
cudaError_t launch_dfma_peak(double* out, int blocks, int iters, cudaStream_t st);

}  // namespace rsw
