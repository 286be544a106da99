/*
 * rsw_oracle.c — THE ORACLE: a plain, slow, obviously-correct CPU implementation of the
 * asymptotic-parareal hot path for 1-D rotating shallow water (arxiv 1303.6615).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library.  The product (paper_1303_6615_b200/) never
 * links, imports or calls it, and this file shares no code, header, table or constant generator
 * with the CUDA path.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "R#" = a reading listed in DESIGN.md §3
 * (taken from SURVEY.md §8(c)).
 *
 * What is computed, by definition and step by step in the paper's order:
 *   - transforms: naive O(n^2) DFT, twiddles e^{-2πi (jk mod n)/n} from an integer-reduced index;
 *   - per-wavenumber exponentials and φ-functions: numeric eigendecomposition (hand-written
 *     Jacobi on the real 6x6 embedding of the Hermitian matrix H_k = i L̂(k)), then
 *     f(hA_k) = V diag(f(h ν_j)) V^H;
 *   - φ-functions near 0: Kassam–Trefethen contour mean (128 points, radius 2); direct formula
 *     elsewhere;
 *   - N(u) (sign R1), ETDRK4 (Cox–Matthews, cited P:1168-1169), Strang (Alg.3
 *     P:518-548, R7), N̄ (Alg.1, R4/R5), coarse averaged RK4 inside
 *     Alg.2's D half-steps (R6), parareal (Eq. HMM parareal iteration P:428-430,
 *     Alg.4, R12-R14).
 *
 * State layout (same bytes as the product's C-ABI, declared independently here):
 *   double[batch][3][n/2+1][2] — fields (v1, v2, h), wavenumbers k = 0..n/2, (re, im);
 *   û_k = (1/n) Σ_j u_j e^{-ikx_j}, x_j = 2πj/n.
 *
 * Pins: every function here is checked by tests/test_oracle_pins.py against brute force, closed
 * forms, library routines (numpy.fft, scipy expm / quad, mpmath), invariants, textbook reductions
 * and convergence orders (DESIGN.md §4 maps each function to its pins); tools/oracle_mutations.py
 * applies 21 plausible one-line mistakes and every one fails a pin.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double _Complex cplx;

/* Mirrors the product's rsw_params byte layout; declared separately on purpose. */
typedef struct {
  double eps, F, mu;
  int32_t n;
} orc_params;

typedef struct {
  double dT, dt, T0, tol;
  int32_t M, n_slices, max_iters, fine_scheme, coarse_scheme;
} orc_parareal_config;

enum { ORC_OK = 0, ORC_ERR_CONFIG = 1, ORC_NOT_CONVERGED = 2, ORC_ERR_DIVERGED = 3 };
enum { ORC_FINE_ETDRK4 = 0, ORC_FINE_STRANG = 1, ORC_FINE_IFRK4 = 2 };
enum { ORC_COARSE_RK4 = 0, ORC_COARSE_MIDPOINT = 1, ORC_COARSE_STRANG = 2 };
enum { ORC_FLAG_LINEAR_ONLY = 1u };

static const double ORC_PI = 3.14159265358979323846264338327950288;

/* ------------------------------------------------------------------------------------------ */
/* Sizes                                                                                       */
/* ------------------------------------------------------------------------------------------ */

/* R10: n grid points = FFT length; retained wavenumbers |k| <= K = floor(n/3). */
static int n_half(int n) { return n / 2 + 1; }
static int k_max(int n) { return n / 3; }
static size_t state_len(int n) { return (size_t)3 * (size_t)n_half(n); } /* complex entries */

/* ------------------------------------------------------------------------------------------ */
/* Naive DFT (§8(c) item 1).  x_j real, j = 0..n-1;  X_k, k = 0..n/2.                           */
/* ------------------------------------------------------------------------------------------ */

typedef struct {
  int n;
  cplx *tw; /* tw[m] = e^{-2πi m/n}, m = 0..n-1 */
} dft_table;

static void dft_table_init(dft_table *t, int n) {
  t->n = n;
  t->tw = (cplx *)malloc(sizeof(cplx) * (size_t)n);
  for (int m = 0; m < n; ++m) {
    double a = -2.0 * ORC_PI * (double)m / (double)n;
    t->tw[m] = cos(a) + I * sin(a);
  }
}
static void dft_table_free(dft_table *t) { free(t->tw); }

/* X_k = (1/n) Σ_{j=0}^{n-1} x_j e^{-2πi jk/n}   (normalised forward transform, k = 0..n/2) */
static void dft_forward(const dft_table *t, const double *x, cplx *X) {
  const int n = t->n;
  for (int k = 0; k <= n / 2; ++k) {
    cplx s = 0.0;
    for (int j = 0; j < n; ++j) s += x[j] * t->tw[((long)j * k) % n];
    X[k] = s / (double)n;
  }
}

/* x_j = Σ_{k=-n/2+1}^{n/2} X_k e^{+2πi jk/n}, with X_{-k} = conj(X_k) (real field, R16). */
static void dft_inverse(const dft_table *t, const cplx *X, double *x) {
  const int n = t->n;
  for (int j = 0; j < n; ++j) {
    cplx s = 0.0;
    for (int k = -n / 2 + 1; k <= n / 2; ++k) {
      cplx Xk = (k >= 0) ? X[k] : conj(X[-k]);
      long m = ((long)j * (long)k) % n;
      if (m < 0) m += n;
      s += Xk * conj(t->tw[m]); /* e^{+2πi jk/n} */
    }
    x[j] = creal(s);
  }
}

/* ------------------------------------------------------------------------------------------ */
/* Pseudo-spectral nonlinearity N(u) (operator table; sign R1; dealiasing R10).      */
/*   N(u) = -( v1 ∂x v1,  v1 ∂x v2,  ∂x(h v1) )                                                 */
/* ------------------------------------------------------------------------------------------ */

typedef struct {
  dft_table dft;
  double *v1, *v1x, *v2x, *h, *p1, *p2, *p3;
  cplx *tmp;
} nl_work;

static void nl_work_init(nl_work *w, int n) {
  dft_table_init(&w->dft, n);
  w->v1 = (double *)malloc(sizeof(double) * 7 * (size_t)n);
  w->v1x = w->v1 + n;
  w->v2x = w->v1 + 2 * n;
  w->h = w->v1 + 3 * n;
  w->p1 = w->v1 + 4 * n;
  w->p2 = w->v1 + 5 * n;
  w->p3 = w->v1 + 6 * n;
  w->tmp = (cplx *)malloc(sizeof(cplx) * (size_t)n_half(n));
}
static void nl_work_free(nl_work *w) {
  dft_table_free(&w->dft);
  free(w->v1);
  free(w->tmp);
}

/* u, out: [3][n/2+1] complex; out may not alias u. */
static void nonlinear(int n, const cplx *u, cplx *out, nl_work *w) {
  const int nh = n_half(n), K = k_max(n);
  const cplx *V1 = u, *V2 = u + nh, *H = u + 2 * nh;
  /* spectral derivatives ∂x -> ik ("F^{-1/2}∂x" symbol convention) */
  dft_inverse(&w->dft, V1, w->v1);
  for (int k = 0; k < nh; ++k) w->tmp[k] = I * (double)k * V1[k];
  dft_inverse(&w->dft, w->tmp, w->v1x);
  for (int k = 0; k < nh; ++k) w->tmp[k] = I * (double)k * V2[k];
  dft_inverse(&w->dft, w->tmp, w->v2x);
  dft_inverse(&w->dft, H, w->h);
  /* pointwise products on the grid */
  for (int j = 0; j < n; ++j) {
    w->p1[j] = w->v1[j] * w->v1x[j]; /* v1 (v1)_x */
    w->p2[j] = w->v1[j] * w->v2x[j]; /* v1 (v2)_x */
    w->p3[j] = w->h[j] * w->v1[j];   /* h v1, then ∂x */
  }
  cplx *O1 = out, *O2 = out + nh, *O3 = out + 2 * nh;
  dft_forward(&w->dft, w->p1, O1);
  dft_forward(&w->dft, w->p2, O2);
  dft_forward(&w->dft, w->p3, O3);
  for (int k = 0; k < nh; ++k) {
    O1[k] = -O1[k];
    O2[k] = -O2[k];
    O3[k] = -(I * (double)k * O3[k]);
    if (k > K) O1[k] = O2[k] = O3[k] = 0.0; /* 2/3 rule */
  }
  /* Reality of the k=0 mode (R16): each output is the transform of a real field, so Im = 0
     up to round-off; keep it exactly 0 as the state layout requires. */
  O1[0] = creal(O1[0]);
  O2[0] = creal(O2[0]);
  O3[0] = creal(O3[0]);
}

/* ------------------------------------------------------------------------------------------ */
/* Per-wavenumber linear algebra: L̂(k) from P:1082-1085 with ∂x -> ik; D̂(k) = -μk^4 (R2).      */
/* Numeric eigendecomposition of the Hermitian H_k = i L̂(k) via a cyclic Jacobi sweep on the    */
/* real symmetric 6x6 embedding [[Re H, -Im H], [Im H, Re H]] (§8(c) item 2).                   */
/* ------------------------------------------------------------------------------------------ */

typedef struct {
  double lam[3]; /* eigenvalues of H_k, ascending */
  cplx V[3][3];  /* V[i][j] = component i of eigenvector j (orthonormal columns) */
} mode_eig;

static void symbol_L(double k, double F, cplx L[3][3]) {
  const double a = k / sqrt(F); /* F^{-1/2} ∂x -> i k F^{-1/2} */
  L[0][0] = 0.0;
  L[0][1] = -1.0;
  L[0][2] = I * a;
  L[1][0] = 1.0;
  L[1][1] = 0.0;
  L[1][2] = 0.0;
  L[2][0] = I * a;
  L[2][1] = 0.0;
  L[2][2] = 0.0;
}

static void jacobi_sym(int n, double *S, double *Vm) {
  /* Cyclic Jacobi for a real symmetric n x n matrix S (row-major); on exit S is diagonal and
     the columns of Vm are the eigenvectors.  Textbook rotation (Golub & Van Loan §8.5). */
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Vm[i * n + j] = (i == j) ? 1.0 : 0.0;
  double fro = 0.0;
  for (int i = 0; i < n * n; ++i) fro += S[i] * S[i];
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += S[p * n + q] * S[p * n + q];
    if (off <= 1e-34 * fro) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        double apq = S[p * n + q];
        if (fabs(apq) < 1e-300) continue;
        double theta = (S[q * n + q] - S[p * n + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        /* S <- J^T S J, J = identity except J_pp = J_qq = c, J_pq = s, J_qp = -s */
        for (int r = 0; r < n; ++r) { /* columns p,q */
          double srp = S[r * n + p], srq = S[r * n + q];
          S[r * n + p] = c * srp - s * srq;
          S[r * n + q] = s * srp + c * srq;
        }
        for (int r = 0; r < n; ++r) { /* rows p,q */
          double spr = S[p * n + r], sqr = S[q * n + r];
          S[p * n + r] = c * spr - s * sqr;
          S[q * n + r] = s * spr + c * sqr;
        }
        for (int r = 0; r < n; ++r) {
          double vrp = Vm[r * n + p], vrq = Vm[r * n + q];
          Vm[r * n + p] = c * vrp - s * vrq;
          Vm[r * n + q] = s * vrp + c * vrq;
        }
      }
  }
}

static void mode_eigen(double k, double F, mode_eig *e) {
  cplx L[3][3], H[3][3];
  symbol_L(k, F, L);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) H[i][j] = I * L[i][j];
  double S[36], Vm[36];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double re = creal(H[i][j]), im = cimag(H[i][j]);
      S[i * 6 + j] = re;
      S[i * 6 + (j + 3)] = -im;
      S[(i + 3) * 6 + j] = im;
      S[(i + 3) * 6 + (j + 3)] = re;
    }
  jacobi_sym(6, S, Vm);
  /* eigenvalues of the embedding come in equal pairs; sort and take one of each pair */
  int idx[6] = {0, 1, 2, 3, 4, 5};
  for (int a = 0; a < 6; ++a)
    for (int b = a + 1; b < 6; ++b)
      if (S[idx[b] * 6 + idx[b]] < S[idx[a] * 6 + idx[a]]) {
        int tmp = idx[a];
        idx[a] = idx[b];
        idx[b] = tmp;
      }
  for (int j = 0; j < 3; ++j) {
    int c = idx[2 * j];
    e->lam[j] = 0.5 * (S[idx[2 * j] * 6 + idx[2 * j]] + S[idx[2 * j + 1] * 6 + idx[2 * j + 1]]);
    /* a real eigenvector (x, y) of the embedding gives the complex eigenvector x + i y */
    double nrm = 0.0;
    cplx v[3];
    for (int i = 0; i < 3; ++i) {
      v[i] = Vm[i * 6 + c] + I * Vm[(i + 3) * 6 + c];
      nrm += creal(v[i] * conj(v[i]));
    }
    nrm = sqrt(nrm);
    for (int i = 0; i < 3; ++i) e->V[i][j] = v[i] / nrm;
  }
}

/* ------------------------------------------------------------------------------------------ */
/* φ-functions (Cox–Matthews / Kassam–Trefethen, cited P:252-253)                   */
/*   φ0(z) = e^z, φ1 = (e^z-1)/z, φ2 = (e^z-1-z)/z^2, φ3 = (e^z-1-z-z^2/2)/z^3                   */
/* ------------------------------------------------------------------------------------------ */

static cplx phi_direct(int j, cplx z) {
  cplx ez = cexp(z);
  switch (j) {
  case 0: return ez;
  case 1: return (ez - 1.0) / z;
  case 2: return (ez - 1.0 - z) / (z * z);
  default: return (ez - 1.0 - z - 0.5 * z * z) / (z * z * z);
  }
}

/* For |z| < 1 the direct formula cancels catastrophically: use the mean value of the analytic
   function over the circle |w - z| = 2 (128-point trapezoid, Kassam & Trefethen 2005); every
   node then has |w| >= 1 where the direct formula is accurate to round-off. */
static cplx phi(int j, cplx z) {
  if (j == 0 || cabs(z) >= 1.0) return phi_direct(j, z);
  const int P = 128;
  cplx s = 0.0;
  for (int p = 0; p < P; ++p) {
    double th = 2.0 * ORC_PI * ((double)p + 0.5) / (double)P;
    s += phi_direct(j, z + 2.0 * (cos(th) + I * sin(th)));
  }
  return s / (double)P;
}

/* ------------------------------------------------------------------------------------------ */
/* Matrix functions f(hA_k), A_k = -L̂(k)/ε + D̂(k) I  (Eq. full eqn; R2, R3).               */
/* With H = V diag(λ) V^H and L̂ = -iH:  A = V diag(iλ/ε - μk^4) V^H.                            */
/* ------------------------------------------------------------------------------------------ */

typedef cplx (*scalar_fn)(cplx z, const void *ctx);

static void matfun(const mode_eig *e, const cplx nu[3], scalar_fn f, const void *ctx,
                   cplx M[3][3]) {
  cplx d[3];
  for (int j = 0; j < 3; ++j) d[j] = f(nu[j], ctx);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      cplx s = 0.0;
      for (int j = 0; j < 3; ++j) s += e->V[r][j] * d[j] * conj(e->V[c][j]);
      M[r][c] = s;
    }
}

static void matvec(const cplx M[3][3], const cplx x[3], cplx y[3]) {
  for (int r = 0; r < 3; ++r) y[r] = M[r][0] * x[0] + M[r][1] * x[1] + M[r][2] * x[2];
}

/* eigenvalues ν_j of hA_k */
static void hA_eigs(const orc_params *p, const mode_eig *e, double k, double h, cplx nu[3]) {
  for (int j = 0; j < 3; ++j) nu[j] = h * (I * e->lam[j] / p->eps - p->mu * k * k * k * k);
}

typedef struct { double h; } hctx;
static cplx f_exp(cplx z, const void *c) { (void)c; return cexp(z); }
static cplx f_Q(cplx z, const void *c) { /* (h/2) φ1(z) with z = hA/2 */
  return 0.5 * ((const hctx *)c)->h * phi(1, z);
}
static cplx f_f1(cplx z, const void *c) {
  return ((const hctx *)c)->h * (phi(1, z) - 3.0 * phi(2, z) + 4.0 * phi(3, z));
}
static cplx f_f2(cplx z, const void *c) {
  return ((const hctx *)c)->h * (2.0 * phi(2, z) - 4.0 * phi(3, z));
}
static cplx f_f3(cplx z, const void *c) {
  return ((const hctx *)c)->h * (4.0 * phi(3, z) - phi(2, z));
}

/* ETDRK4 coefficient matrices for one wavenumber (Cox & Matthews 2002, cited P:1168-1169):
     E = e^{hA}, E2 = e^{hA/2}, Q = (h/2)φ1(hA/2),
     f1 = h(φ1 - 3φ2 + 4φ3)(hA), f2 = h(2φ2 - 4φ3)(hA), f3 = h(4φ3 - φ2)(hA). */
typedef struct {
  cplx E[3][3], E2[3][3], Q[3][3], f1[3][3], f2[3][3], f3[3][3];
} etd_coef;

static void etd_coefficients(const orc_params *p, double k, double h, etd_coef *c) {
  mode_eig e;
  mode_eigen(k, p->F, &e);
  cplx nu[3], nu2[3];
  hA_eigs(p, &e, k, h, nu);
  hA_eigs(p, &e, k, 0.5 * h, nu2);
  hctx hc = {h};
  matfun(&e, nu, f_exp, NULL, c->E);
  matfun(&e, nu2, f_exp, NULL, c->E2);
  matfun(&e, nu2, f_Q, &hc, c->Q);
  matfun(&e, nu, f_f1, &hc, c->f1);
  matfun(&e, nu, f_f2, &hc, c->f2);
  matfun(&e, nu, f_f3, &hc, c->f3);
}

/* e^{τ L̂(k)} = V diag(e^{-iτλ_j}) V^H  (L̂ = -iH) */
typedef struct { double tau; } tctx;
static cplx f_expL(cplx lam, const void *c) {
  return cexp(-I * ((const tctx *)c)->tau * creal(lam));
}
static void expL(const mode_eig *e, double tau, cplx M[3][3]) {
  cplx lam[3] = {e->lam[0], e->lam[1], e->lam[2]};
  tctx tc = {tau};
  matfun(e, lam, f_expL, &tc, M);
}

/* ------------------------------------------------------------------------------------------ */
/* Helpers on half-spectrum states                                                             */
/* ------------------------------------------------------------------------------------------ */

/* apply a per-wavenumber 3x3 matrix (given for k = 0..K) to a state; modes k > K -> 0 */
static void apply_modes(int n, const cplx (*M)[3][3], const cplx *x, cplx *y) {
  const int nh = n_half(n), K = k_max(n);
  for (int k = 0; k < nh; ++k) {
    cplx xi[3] = {x[k], x[nh + k], x[2 * nh + k]}, yo[3];
    if (k <= K) {
      matvec(M[k], xi, yo);
    } else {
      yo[0] = yo[1] = yo[2] = 0.0;
    }
    y[k] = yo[0];
    y[nh + k] = yo[1];
    y[2 * nh + k] = yo[2];
  }
}

/* keep the k=0 coefficients real (R16) */
static void realify_k0(int n, cplx *x) {
  const int nh = n_half(n);
  for (int f = 0; f < 3; ++f) x[f * nh] = creal(x[f * nh]);
}

/* ------------------------------------------------------------------------------------------ */
/* Fine propagators                                                                            */
/* ------------------------------------------------------------------------------------------ */

/* R9: m = ceil(dT/dt - 1e-9) steps of dt_eff = dT/m */
static int n_fine_steps(double dT, double dt) { return (int)ceil(dT / dt - 1e-9); }

typedef struct {
  int n, K;
  cplx (*E)[3][3], (*E2)[3][3], (*Q)[3][3], (*f1)[3][3], (*f2)[3][3], (*f3)[3][3];
} etd_table;

static void etd_table_init(etd_table *t, const orc_params *p, double h) {
  t->n = p->n;
  t->K = k_max(p->n);
  size_t m = (size_t)(t->K + 1);
  t->E = malloc(sizeof(*t->E) * m);
  t->E2 = malloc(sizeof(*t->E2) * m);
  t->Q = malloc(sizeof(*t->Q) * m);
  t->f1 = malloc(sizeof(*t->f1) * m);
  t->f2 = malloc(sizeof(*t->f2) * m);
  t->f3 = malloc(sizeof(*t->f3) * m);
  for (int k = 0; k <= t->K; ++k) {
    etd_coef c;
    etd_coefficients(p, (double)k, h, &c);
    memcpy(t->E[k], c.E, sizeof(c.E));
    memcpy(t->E2[k], c.E2, sizeof(c.E2));
    memcpy(t->Q[k], c.Q, sizeof(c.Q));
    memcpy(t->f1[k], c.f1, sizeof(c.f1));
    memcpy(t->f2[k], c.f2, sizeof(c.f2));
    memcpy(t->f3[k], c.f3, sizeof(c.f3));
  }
}
static void etd_table_free(etd_table *t) {
  free(t->E);
  free(t->E2);
  free(t->Q);
  free(t->f1);
  free(t->f2);
  free(t->f3);
}

/* One ETDRK4 step (Cox & Matthews 2002; §8(a) a2):
     Nu = N(u); a = E2 u + Q Nu; Na = N(a); b = E2 u + Q Na; Nb = N(b);
     c = E2 a + Q (2Nb - Nu); Nc = N(c); u+ = E u + f1 Nu + f2 (Na + Nb) + f3 Nc. */
static void etdrk4_step(const etd_table *t, int linear_only, cplx *u, nl_work *w, cplx *buf) {
  const int n = t->n;
  const size_t L = state_len(n);
  cplx *Nu = buf, *a = buf + L, *Na = buf + 2 * L, *b = buf + 3 * L, *Nb = buf + 4 * L,
       *c = buf + 5 * L, *Nc = buf + 6 * L, *t1 = buf + 7 * L, *t2 = buf + 8 * L;
#define NL(x, y)                                                                                  \
  do {                                                                                          \
    if (linear_only) memset((y), 0, sizeof(cplx) * L);                                          \
    else nonlinear(n, (x), (y), w);                                                             \
  } while (0)
  NL(u, Nu);
  apply_modes(n, t->E2, u, t1);
  apply_modes(n, t->Q, Nu, t2);
  for (size_t i = 0; i < L; ++i) a[i] = t1[i] + t2[i];
  NL(a, Na);
  apply_modes(n, t->Q, Na, t2);
  for (size_t i = 0; i < L; ++i) b[i] = t1[i] + t2[i];
  NL(b, Nb);
  apply_modes(n, t->E2, a, t1);
  for (size_t i = 0; i < L; ++i) t2[i] = 2.0 * Nb[i] - Nu[i];
  apply_modes(n, t->Q, t2, c);
  for (size_t i = 0; i < L; ++i) c[i] = t1[i] + c[i];
  NL(c, Nc);
  /* u+ = E u + f1 Nu + f2 (Na + Nb) + f3 Nc */
  apply_modes(n, t->E, u, t1);
  cplx *acc = a; /* a no longer needed */
  memcpy(acc, t1, sizeof(cplx) * L);
  apply_modes(n, t->f1, Nu, t1);
  for (size_t i = 0; i < L; ++i) acc[i] += t1[i];
  for (size_t i = 0; i < L; ++i) t2[i] = Na[i] + Nb[i];
  apply_modes(n, t->f2, t2, t1);
  for (size_t i = 0; i < L; ++i) acc[i] += t1[i];
  apply_modes(n, t->f3, Nc, t1);
  for (size_t i = 0; i < L; ++i) acc[i] += t1[i];
  memcpy(u, acc, sizeof(cplx) * L);
  realify_k0(n, u);
#undef NL
}

/* One Strang step, Alg.3 with the explicit-midpoint reading R7 and the sign R3:
     v = E2 u; k1 = N(v); w = v + h N(v + (h/2) k1); u+ = E2 w,   E2 = e^{(h/2)A}. */
static void strang_step(const etd_table *t, double h, int linear_only, cplx *u, nl_work *w,
                        cplx *buf) {
  const int n = t->n;
  const size_t L = state_len(n);
  cplx *v = buf, *k1 = buf + L, *mid = buf + 2 * L, *k2 = buf + 3 * L;
  apply_modes(n, t->E2, u, v);
  if (linear_only) {
    memset(k1, 0, sizeof(cplx) * L);
  } else {
    nonlinear(n, v, k1, w);
  }
  for (size_t i = 0; i < L; ++i) mid[i] = v[i] + 0.5 * h * k1[i];
  if (linear_only) {
    memset(k2, 0, sizeof(cplx) * L);
  } else {
    nonlinear(n, mid, k2, w);
  }
  for (size_t i = 0; i < L; ++i) v[i] = v[i] + h * k2[i];
  apply_modes(n, t->E2, v, u);
  realify_k0(n, u);
}

/* Integrating-factor baseline ("the operator integrating factor method (cf.
   Kassam-Trefethen)"; SPEC S:350 reading: factor e^{-tA}, classical RK4 on the
   transformed system).  With v(t) = e^{-tA} u(t), v' = g(t, v) = e^{-tA} N(e^{tA} v); one step of
   classical RK4 for v from v0 = u_n, then u_{n+1} = e^{hA} v1:
     K1 = g(0, v0), K2 = g(h/2, v0 + h/2 K1), K3 = g(h/2, v0 + h/2 K2), K4 = g(h, v0 + h K3),
     v1 = v0 + h/6 (K1 + 2K2 + 2K3 + K4).
   Written literally (the transforms e^{±(h/2)A}, e^{±hA} are separate per-mode matrices from the
   numeric eigendecomposition), not in the factored forward-only form the GPU uses. */
typedef struct {
  int n, K;
  cplx (*Ep)[3][3], (*Em)[3][3], (*E2p)[3][3], (*E2m)[3][3]; /* e^{hA}, e^{-hA}, e^{hA/2}, e^{-hA/2} */
} if_table;

static void if_table_init(if_table *t, const orc_params *p, double h) {
  t->n = p->n;
  t->K = k_max(p->n);
  size_t m = (size_t)(t->K + 1);
  t->Ep = malloc(sizeof(*t->Ep) * m);
  t->Em = malloc(sizeof(*t->Em) * m);
  t->E2p = malloc(sizeof(*t->E2p) * m);
  t->E2m = malloc(sizeof(*t->E2m) * m);
  for (int k = 0; k <= t->K; ++k) {
    mode_eig e;
    mode_eigen((double)k, p->F, &e);
    cplx nu[3], nu2[3], mnu[3], mnu2[3];
    hA_eigs(p, &e, (double)k, h, nu);
    hA_eigs(p, &e, (double)k, 0.5 * h, nu2);
    for (int j = 0; j < 3; ++j) {
      mnu[j] = -nu[j];
      mnu2[j] = -nu2[j];
    }
    matfun(&e, nu, f_exp, NULL, t->Ep[k]);
    matfun(&e, mnu, f_exp, NULL, t->Em[k]);
    matfun(&e, nu2, f_exp, NULL, t->E2p[k]);
    matfun(&e, mnu2, f_exp, NULL, t->E2m[k]);
  }
}
static void if_table_free(if_table *t) {
  free(t->Ep);
  free(t->Em);
  free(t->E2p);
  free(t->E2m);
}

/* g(τ, v) = e^{-τA} N(e^{τA} v) for τ = 0 (P = M = NULL), h/2 or h */
static void if_rhs(int n, int linear_only, const cplx (*P)[3][3], const cplx (*Mi)[3][3], const cplx *v,
                   cplx *out, nl_work *w, cplx *tmp) {
  const size_t L = state_len(n);
  if (linear_only) {
    memset(out, 0, sizeof(cplx) * L);
    return;
  }
  if (!P) {
    nonlinear(n, v, out, w);
    return;
  }
  apply_modes(n, P, v, tmp);
  nonlinear(n, tmp, out, w);
  memcpy(tmp, out, sizeof(cplx) * L);
  apply_modes(n, Mi, tmp, out);
}

static void ifrk4_step(const if_table *t, double h, int linear_only, cplx *u, nl_work *w, cplx *buf) {
  const int n = t->n;
  const size_t L = state_len(n);
  cplx *K1 = buf, *K2 = buf + L, *K3 = buf + 2 * L, *K4 = buf + 3 * L, *vs = buf + 4 * L,
       *tmp = buf + 5 * L;
  if_rhs(n, linear_only, NULL, NULL, u, K1, w, tmp);
  for (size_t i = 0; i < L; ++i) vs[i] = u[i] + 0.5 * h * K1[i];
  if_rhs(n, linear_only, (const cplx(*)[3][3])t->E2p, (const cplx(*)[3][3])t->E2m, vs, K2, w, tmp);
  for (size_t i = 0; i < L; ++i) vs[i] = u[i] + 0.5 * h * K2[i];
  if_rhs(n, linear_only, (const cplx(*)[3][3])t->E2p, (const cplx(*)[3][3])t->E2m, vs, K3, w, tmp);
  for (size_t i = 0; i < L; ++i) vs[i] = u[i] + h * K3[i];
  if_rhs(n, linear_only, (const cplx(*)[3][3])t->Ep, (const cplx(*)[3][3])t->Em, vs, K4, w, tmp);
  for (size_t i = 0; i < L; ++i) vs[i] = u[i] + (h / 6.0) * (K1[i] + 2.0 * K2[i] + 2.0 * K3[i] + K4[i]);
  apply_modes(n, (const cplx(*)[3][3])t->Ep, vs, u);
  realify_k0(n, u);
}

static void fine_one(const orc_params *p, int scheme, int linear_only, const etd_table *t,
                     double h, int m, const cplx *in, cplx *out) {
  const size_t L = state_len(p->n);
  nl_work w;
  nl_work_init(&w, p->n);
  cplx *buf = malloc(sizeof(cplx) * 9 * L);
  cplx *u = malloc(sizeof(cplx) * L);
  memcpy(u, in, sizeof(cplx) * L);
  if_table it = {0};
  if (scheme == ORC_FINE_IFRK4) if_table_init(&it, p, h);
  for (int s = 0; s < m; ++s) {
    if (scheme == ORC_FINE_STRANG) strang_step(t, h, linear_only, u, &w, buf);
    else if (scheme == ORC_FINE_IFRK4) ifrk4_step(&it, h, linear_only, u, &w, buf);
    else etdrk4_step(t, linear_only, u, &w, buf);
  }
  if (scheme == ORC_FINE_IFRK4) if_table_free(&it);
  memcpy(out, u, sizeof(cplx) * L);
  free(u);
  free(buf);
  nl_work_free(&w);
}

static int params_ok(const orc_params *p) {
  if (!p || !(p->eps > 0) || !isfinite(p->eps) || !(p->F > 0) || !isfinite(p->F) ||
      !(p->mu >= 0) || !isfinite(p->mu))
    return 0;
  if (p->n < 16 || p->n > 4096 || (p->n & (p->n - 1))) return 0;
  return 1;
}

/* φ_ΔT for n_slices independent states (the "parfor" of Alg.4). */
int oracle_fine_propagate(const orc_params *p, int32_t scheme, uint32_t flags, double dT,
                          double dt, int32_t n_slices, const double *u_in, double *u_out) {
  if (!params_ok(p) || !(dT > 0) || !(dt > 0) || dt > dT || n_slices < 0 || !u_in || !u_out)
    return ORC_ERR_CONFIG;
  if (scheme != ORC_FINE_ETDRK4 && scheme != ORC_FINE_STRANG && scheme != ORC_FINE_IFRK4) return ORC_ERR_CONFIG;
  const int m = n_fine_steps(dT, dt);
  const double h = dT / (double)m;
  etd_table t;
  /* Strang uses E2 = e^{(h/2)A}: same table entry as ETDRK4's E2 at step h */
  etd_table_init(&t, p, h);
  const size_t L = state_len(p->n);
  const int lin = (flags & ORC_FLAG_LINEAR_ONLY) != 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int s = 0; s < n_slices; ++s)
    fine_one(p, scheme, lin, &t, h, m, (const cplx *)u_in + (size_t)s * L,
             (cplx *)u_out + (size_t)s * L);
  etd_table_free(&t);
  return ORC_OK;
}

/* Single nonlinear evaluation for tests: out = N(u) for n_states states. */
int oracle_nonlinear(const orc_params *p, int32_t n_states, const double *u, double *out) {
  if (!params_ok(p) || n_states < 0 || !u || !out) return ORC_ERR_CONFIG;
  const size_t L = state_len(p->n);
#pragma omp parallel
  {
    nl_work w;
    nl_work_init(&w, p->n);
#pragma omp for
    for (int s = 0; s < n_states; ++s)
      nonlinear(p->n, (const cplx *)u + s * L, (cplx *)out + s * L, &w);
    nl_work_free(&w);
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* HMM averaged nonlinearity (Eq. numerical average, discretized P:289-293; ε-scaled form P:313, */
/* P:320-323; Alg.1; kernel P:383-390).                                              */
/*   N̄(v) = Σ_{m=1}^{M-1} w_m e^{τ_m L̂} N(e^{-τ_m L̂} v),  τ_m = s_m/ε,  s_m = T0 m/M (R4),      */
/*   w_m = ρ(m/M) / Σ_{j=1}^{M-1} ρ(j/M),  ρ(s) = exp(-1/(s(1-s))) on (0,1) (R5; C cancels).     */
/* ------------------------------------------------------------------------------------------ */

static double rho(double s) { return (s > 0.0 && s < 1.0) ? exp(-1.0 / (s * (1.0 - s))) : 0.0; }

void oracle_weights(int32_t M, double *w) {
  double tot = 0.0;
  for (int j = 1; j <= M - 1; ++j) tot += rho((double)j / (double)M);
  w[0] = 0.0;
  for (int m = 1; m <= M - 1; ++m) w[m] = rho((double)m / (double)M) / tot;
}

typedef struct {
  int n, K, M;
  double *w;
  mode_eig *eig; /* k = 0..K */
} avg_ctx;

static void avg_ctx_init(avg_ctx *a, const orc_params *p, int M) {
  a->n = p->n;
  a->K = k_max(p->n);
  a->M = M;
  a->w = malloc(sizeof(double) * (size_t)M);
  oracle_weights(M, a->w);
  a->eig = malloc(sizeof(mode_eig) * (size_t)(a->K + 1));
  for (int k = 0; k <= a->K; ++k) mode_eigen((double)k, p->F, &a->eig[k]);
}
static void avg_ctx_free(avg_ctx *a) {
  free(a->w);
  free(a->eig);
}

/* out = N̄(v) for one state; samples evaluated in parallel ("parfor", Alg.1), summed serially
   in ascending m ("Sum"). */
static void averaged_one(const orc_params *p, const avg_ctx *a, double T0, const cplx *v,
                         cplx *out) {
  const int n = p->n, K = a->K, M = a->M;
  const size_t L = state_len(n);
  cplx *X = malloc(sizeof(cplx) * L * (size_t)M); /* per-sample terms, m = 1..M-1 */
#pragma omp parallel
  {
    nl_work w;
    nl_work_init(&w, n);
    cplx *um = malloc(sizeof(cplx) * L), *nm = malloc(sizeof(cplx) * L);
    cplx (*Pm)[3][3] = malloc(sizeof(*Pm) * (size_t)(K + 1));
    cplx (*Pp)[3][3] = malloc(sizeof(*Pp) * (size_t)(K + 1));
#pragma omp for schedule(dynamic, 1)
    for (int m = 1; m <= M - 1; ++m) {
      const double s_m = T0 * (double)m / (double)M; /* Alg.1 */
      const double tau = s_m / p->eps;                /* P:313, R4 */
      for (int k = 0; k <= K; ++k) {
        expL(&a->eig[k], -tau, Pm[k]); /* e^{-τ L̂} */
        expL(&a->eig[k], tau, Pp[k]);  /* e^{+τ L̂} */
      }
      apply_modes(n, (const cplx(*)[3][3])Pm, v, um);
      nonlinear(n, um, nm, &w);
      apply_modes(n, (const cplx(*)[3][3])Pp, nm, X + (size_t)m * L);
      for (size_t i = 0; i < L; ++i) X[(size_t)m * L + i] *= a->w[m];
    }
    free(um);
    free(nm);
    free(Pm);
    free(Pp);
    nl_work_free(&w);
  }
  for (size_t i = 0; i < L; ++i) out[i] = 0.0;
  for (int m = 1; m <= M - 1; ++m)
    for (size_t i = 0; i < L; ++i) out[i] += X[(size_t)m * L + i];
  realify_k0(n, out);
  free(X);
}

int oracle_averaged_rhs(const orc_params *p, double T0, int32_t M, int32_t n_states,
                        const double *u_in, double *rhs_out) {
  if (!params_ok(p) || !(T0 > 0) || M < 2 || n_states < 0 || !u_in || !rhs_out)
    return ORC_ERR_CONFIG;
  avg_ctx a;
  avg_ctx_init(&a, p, M);
  const size_t L = state_len(p->n);
  for (int s = 0; s < n_states; ++s)
    averaged_one(p, &a, T0, (const cplx *)u_in + s * L, (cplx *)rhs_out + s * L);
  avg_ctx_free(&a);
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Coarse propagator φ̄_ΔT (Alg.2; φ̄ P:415-417; R3, R6, R7, R8):                      */
/*   v = e^{ΔT D/2} u;  RK4 (or midpoint) step of size ΔT on v' = N̄(v);  v = e^{ΔT D/2} v;       */
/*   G(u) = e^{-(ΔT/ε) L̂} v.                                                                    */
/* ------------------------------------------------------------------------------------------ */

typedef struct {
  avg_ctx a;
  cplx (*back)[3][3]; /* e^{-(ΔT/ε) L̂(k)} */
  double *dhalf;      /* e^{-μ k^4 ΔT/2} */
  etd_table strang;   /* standard parareal: one Strang step of size ΔT on the full eqn */
} coarse_ctx;

static void coarse_ctx_init(coarse_ctx *c, const orc_params *p, double dT, int M) {
  avg_ctx_init(&c->a, p, M);
  etd_table_init(&c->strang, p, dT);
  const int K = c->a.K;
  c->back = malloc(sizeof(*c->back) * (size_t)(K + 1));
  c->dhalf = malloc(sizeof(double) * (size_t)(K + 1));
  for (int k = 0; k <= K; ++k) {
    expL(&c->a.eig[k], -dT / p->eps, c->back[k]);
    double k4 = (double)k * k * k * k;
    c->dhalf[k] = exp(-p->mu * k4 * 0.5 * dT); /* e^{(ΔT/2) D̂}, D̂ = -μk^4 (R2) */
  }
}
static void coarse_ctx_free(coarse_ctx *c) {
  avg_ctx_free(&c->a);
  etd_table_free(&c->strang);
  free(c->back);
  free(c->dhalf);
}

static void d_half(int n, const double *dh, cplx *x) {
  const int nh = n_half(n), K = k_max(n);
  for (int f = 0; f < 3; ++f)
    for (int k = 0; k < nh; ++k) x[f * nh + k] = (k <= K) ? dh[k] * x[f * nh + k] : 0.0;
}

static void coarse_one(const orc_params *p, const coarse_ctx *c, int scheme, double dT,
                       double T0, const cplx *u, cplx *out) {
  const int n = p->n;
  const size_t L = state_len(n);
  if (scheme == ORC_COARSE_STRANG) {
    /* standard parareal: the coarse solver solves the full equation with one Strang step of size
       ΔT (Alg.3 with m = 1; "we use Strang splitting for the coarse solver") */
    fine_one(p, ORC_FINE_STRANG, 0, &c->strang, dT, 1, u, out);
    return;
  }
  cplx *v = malloc(sizeof(cplx) * L * 7);
  cplx *k1 = v + L, *k2 = v + 2 * L, *k3 = v + 3 * L, *k4 = v + 4 * L, *y = v + 5 * L,
       *t = v + 6 * L;
  memcpy(v, u, sizeof(cplx) * L);
  d_half(n, c->dhalf, v);
  if (scheme == ORC_COARSE_MIDPOINT) {
    /* P:495-498 with R7: v <- v + ΔT N̄(v + (ΔT/2) N̄(v)) */
    averaged_one(p, &c->a, T0, v, k1);
    for (size_t i = 0; i < L; ++i) y[i] = v[i] + 0.5 * dT * k1[i];
    averaged_one(p, &c->a, T0, y, k2);
    for (size_t i = 0; i < L; ++i) v[i] = v[i] + dT * k2[i];
  } else {
    /* classical RK4 on v' = N̄(v) (R6) */
    averaged_one(p, &c->a, T0, v, k1);
    for (size_t i = 0; i < L; ++i) y[i] = v[i] + 0.5 * dT * k1[i];
    averaged_one(p, &c->a, T0, y, k2);
    for (size_t i = 0; i < L; ++i) y[i] = v[i] + 0.5 * dT * k2[i];
    averaged_one(p, &c->a, T0, y, k3);
    for (size_t i = 0; i < L; ++i) y[i] = v[i] + dT * k3[i];
    averaged_one(p, &c->a, T0, y, k4);
    for (size_t i = 0; i < L; ++i)
      v[i] = v[i] + (dT / 6.0) * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
  }
  d_half(n, c->dhalf, v);
  apply_modes(n, (const cplx(*)[3][3])c->back, v, t); /* P:508-510 with sign R3 */
  realify_k0(n, t);
  memcpy(out, t, sizeof(cplx) * L);
  free(v);
}

int oracle_coarse_propagate(const orc_params *p, int32_t coarse_scheme, double dT, double T0,
                            int32_t M, int32_t n_states, const double *u_in, double *u_out) {
  if (!params_ok(p) || !(dT > 0) || !(T0 > 0) || M < 2 || n_states < 0 || !u_in || !u_out)
    return ORC_ERR_CONFIG;
  if (coarse_scheme != ORC_COARSE_RK4 && coarse_scheme != ORC_COARSE_MIDPOINT &&
      coarse_scheme != ORC_COARSE_STRANG)
    return ORC_ERR_CONFIG;
  coarse_ctx c;
  coarse_ctx_init(&c, p, dT, M);
  const size_t L = state_len(p->n);
  for (int s = 0; s < n_states; ++s)
    coarse_one(p, &c, coarse_scheme, dT, T0, (const cplx *)u_in + s * L,
               (cplx *)u_out + s * L);
  coarse_ctx_free(&c);
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Parareal (Eq. HMM parareal iteration P:428-430; Alg.4; R12, R13, R14).             */
/* ------------------------------------------------------------------------------------------ */

/* R12: relative L2 over all 3 fields from half-spectrum coefficients with Parseval weights
   w_0 = 1, w_k = 2 (0 < k < n/2), w_{n/2} = 1. */
static double wnorm2(int n, const cplx *x) {
  const int nh = n_half(n);
  double s = 0.0;
  for (int f = 0; f < 3; ++f)
    for (int k = 0; k < nh; ++k) {
      double wk = (k == 0 || k == n / 2) ? 1.0 : 2.0;
      cplx z = x[f * nh + k];
      s += wk * (creal(z) * creal(z) + cimag(z) * cimag(z));
    }
  return s;
}

double oracle_rel_l2(int32_t n, const double *a, const double *b) {
  const size_t L = state_len(n);
  cplx *d = malloc(sizeof(cplx) * L);
  for (size_t i = 0; i < L; ++i) d[i] = ((const cplx *)a)[i] - ((const cplx *)b)[i];
  double r = sqrt(wnorm2(n, d) / wnorm2(n, (const cplx *)b));
  free(d);
  return r;
}

/* U: [(S+1)][3][n/2+1][2].  F_out / G_out (optional, may be NULL): the last iteration's fine
   endpoints F_n = F(U^{k-1}_n) and coarse values G_n, n = 0..S-1.  tol <= 0: exactly max_iters
   iterations; tol > 0: stop at the first r_k < tol (ORC_NOT_CONVERGED if none). */
int oracle_parareal(const orc_params *p, const orc_parareal_config *cfg, const double *u0,
                    double *U_out, double *resid_hist, int32_t *iters_done, double *F_out,
                    double *G_out) {
  if (!params_ok(p) || !cfg || !u0 || !U_out || !iters_done) return ORC_ERR_CONFIG;
  const int S = cfg->n_slices;
  if (S < 1 || cfg->max_iters < 0 || cfg->max_iters > S || !(cfg->dT > 0) || !(cfg->dt > 0) ||
      cfg->dt > cfg->dT || !(cfg->T0 > 0) || cfg->M < 2)
    return ORC_ERR_CONFIG;
  if (cfg->max_iters > 0 && !resid_hist) return ORC_ERR_CONFIG;
  const int n = p->n;
  const size_t L = state_len(n);
  cplx *U = (cplx *)U_out;
  cplx *Uold = malloc(sizeof(cplx) * L * (size_t)(S + 1));
  cplx *F = malloc(sizeof(cplx) * L * (size_t)S);
  cplx *G = malloc(sizeof(cplx) * L * (size_t)S);
  cplx *g = malloc(sizeof(cplx) * L);
  coarse_ctx c;
  coarse_ctx_init(&c, p, cfg->dT, cfg->M);

  /* k = 0: U^0_0 = u0, U^0_{n+1} = φ̄(U^0_n)  (Alg.4, R13) */
  memcpy(U, u0, sizeof(cplx) * L);
  for (int s = 0; s < S; ++s) {
    coarse_one(p, &c, cfg->coarse_scheme, cfg->dT, cfg->T0, U + s * L, G + s * L);
    memcpy(U + (s + 1) * L, G + s * L, sizeof(cplx) * L);
  }
  int status = (cfg->tol > 0 && cfg->max_iters > 0) ? ORC_NOT_CONVERGED : ORC_OK;
  int done = 0;
  for (int k = 1; k <= cfg->max_iters; ++k) {
    memcpy(Uold, U, sizeof(cplx) * L * (size_t)(S + 1));
    /* parfor n: F_n = φ(U^{k-1}_n) */
    int rc = oracle_fine_propagate(p, cfg->fine_scheme, 0u, cfg->dT, cfg->dt, S,
                                   (const double *)Uold, (double *)F);
    if (rc != ORC_OK) {
      status = rc;
      break;
    }
    /* serial sweep: U^k_{n+1} = φ̄(U^k_n) + (F_n - G_n), G_n <- φ̄(U^k_n)   (R14) */
    for (int s = 0; s < S; ++s) {
      coarse_one(p, &c, cfg->coarse_scheme, cfg->dT, cfg->T0, U + s * L, g);
      for (size_t i = 0; i < L; ++i)
        U[(s + 1) * L + i] = g[i] + (F[s * L + i] - G[s * L + i]);
      memcpy(G + s * L, g, sizeof(cplx) * L);
    }
    /* residual r_k = max_{n=1..S} ||U^k_n - U^{k-1}_n|| / ||U^k_n||  (R12) */
    double r = 0.0;
    int finite = 1;
    for (int s = 1; s <= S; ++s) {
      double num = 0.0, den = wnorm2(n, U + s * L);
      cplx *d = g;
      for (size_t i = 0; i < L; ++i) d[i] = U[s * L + i] - Uold[s * L + i];
      num = wnorm2(n, d);
      double rs = sqrt(num / den);
      if (!isfinite(rs)) finite = 0;
      if (rs > r) r = rs;
    }
    resid_hist[k - 1] = r;
    done = k;
    if (!finite || r > 1e6) {
      status = ORC_ERR_DIVERGED; /* S:399 divergence guard */
      break;
    }
    if (cfg->tol > 0 && r < cfg->tol) {
      status = ORC_OK;
      break;
    }
  }
  *iters_done = done;
  if (F_out) memcpy(F_out, F, sizeof(cplx) * L * (size_t)S);
  if (G_out) memcpy(G_out, G, sizeof(cplx) * L * (size_t)S);
  coarse_ctx_free(&c);
  free(Uold);
  free(F);
  free(G);
  free(g);
  return status;
}

/* ------------------------------------------------------------------------------------------ */
/* Small entry points exposed for the pins in tests/                                          */
/* ------------------------------------------------------------------------------------------ */

void oracle_dft_forward(int32_t n, const double *x, double *X) {
  dft_table t;
  dft_table_init(&t, n);
  dft_forward(&t, x, (cplx *)X);
  dft_table_free(&t);
}

void oracle_dft_inverse(int32_t n, const double *X, double *x) {
  dft_table t;
  dft_table_init(&t, n);
  dft_inverse(&t, (const cplx *)X, x);
  dft_table_free(&t);
}

void oracle_phi(int32_t j, double zre, double zim, double *out) {
  cplx r = phi(j, zre + I * zim);
  out[0] = creal(r);
  out[1] = cimag(r);
}

/* eigen-decomposition of H_k = i L̂(k): lam[3], V[3][3] complex (row-major, columns = vectors) */
void oracle_mode_eigen(double k, double F, double *lam, double *V) {
  mode_eig e;
  mode_eigen(k, F, &e);
  for (int j = 0; j < 3; ++j) lam[j] = e.lam[j];
  memcpy(V, e.V, sizeof(e.V));
}

/* which: 0 E=e^{hA}, 1 E2, 2 Q, 3 f1, 4 f2, 5 f3, 6 e^{h L̂} (h read as τ) */
void oracle_mode_matrix(const orc_params *p, double k, double h, int32_t which, double *out) {
  if (which == 6) {
    mode_eig e;
    mode_eigen(k, p->F, &e);
    cplx M[3][3];
    expL(&e, h, M);
    memcpy(out, M, sizeof(M));
    return;
  }
  etd_coef c;
  etd_coefficients(p, k, h, &c);
  const cplx(*M)[3] = which == 0 ? c.E : which == 1 ? c.E2 : which == 2 ? c.Q
                    : which == 3 ? c.f1 : which == 4 ? c.f2 : c.f3;
  memcpy(out, M, sizeof(cplx) * 9);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
