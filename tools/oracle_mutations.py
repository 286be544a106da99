"""Mutation check of the oracle pins (test infrastructure): applies plausible one-line mistakes to
oracle/rsw_oracle.c one at a time, rebuilds, runs tests/test_oracle_pins.py and reports whether a pin
catches each one; the source is restored at the end.  Run from the repo root:
    python tools/oracle_mutations.py
"""
import subprocess, sys, shutil
src='oracle/rsw_oracle.c'
orig=open(src).read()
muts=[
 # the six mutations the round-1 review found surviving
 ("double wk = (k == 0 || k == n / 2) ? 1.0 : 2.0;","double wk = 1.0;"),
 ("double num = 0.0, den = wnorm2(n, U + s * L);","double num = 0.0, den = wnorm2(n, Uold + s * L);"),
 ("for (int s = 1; s <= S; ++s) {\n      double num","for (int s = 1; s < S; ++s) {\n      double num"),
 ("  d_half(n, c->dhalf, v); /* P:502-504 */","  /* dropped */"),
 ("  d_half(n, c->dhalf, v); /* P:491-493 */","  d_half(n, c->dhalf, v); d_half(n, c->dhalf, v);"),
 ("exp(-p->mu * k4 * 0.5 * dT)","exp(-p->mu * k4 * dT)"),
 # further plausible one-line mistakes across the oracle
 ("expL(&a->eig[k], -tau, Pm[k]); /* e^{-τ L̂} */","expL(&a->eig[k], tau, Pm[k]);"),
 ("expL(&a->eig[k], tau, Pp[k]);  /* e^{+τ L̂} */","expL(&a->eig[k], -tau, Pp[k]);"),
 ("const double s_m = T0 * (double)m / (double)M; /* Alg.1 P:473 */","const double s_m = T0 * (double)(m + 1) / (double)M;"),
 ("for (int m = 1; m <= M - 1; ++m) w[m] = rho((double)m / (double)M) / tot;","for (int m = 1; m <= M - 1; ++m) w[m] = rho((double)m / (double)M);"),
 ("U[(s + 1) * L + i] = g[i] + (F[s * L + i] - G[s * L + i]);","U[(s + 1) * L + i] = g[i] + (G[s * L + i] - F[s * L + i]);"),
 ("O3[k] = -(I * (double)k * O3[k]);","O3[k] = (I * (double)k * O3[k]);"),
 ("w->p3[j] = w->h[j] * w->v1[j];   /* h v1, then ∂x      P:1093 */","w->p3[j] = w->h[j] * w->v1x[j];"),
 ("for (size_t i = 0; i < L; ++i) t2[i] = 2.0 * Nb[i] - Nu[i];","for (size_t i = 0; i < L; ++i) t2[i] = 2.0 * Nb[i] + Nu[i];"),
 ("for (size_t i = 0; i < L; ++i) mid[i] = v[i] + 0.5 * h * k1[i];","for (size_t i = 0; i < L; ++i) mid[i] = v[i] + h * k1[i];"),
 ("expL(&c->a.eig[k], -dT / p->eps, c->back[k]);","expL(&c->a.eig[k], dT / p->eps, c->back[k]);"),
 ("if (k > K) O1[k] = O2[k] = O3[k] = 0.0; /* 2/3 rule */","if (k > n / 2) O1[k] = O2[k] = O3[k] = 0.0;"),
 ("v[i] = v[i] + (dT / 6.0) * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);","v[i] = v[i] + (dT / 6.0) * (k1[i] + 2.0 * k2[i] + k3[i] + 2.0 * k4[i]);"),
 ("return ((const hctx *)c)->h * (4.0 * phi(3, z) - phi(2, z));","return ((const hctx *)c)->h * (4.0 * phi(3, z) + phi(2, z));"),
 ("matfun(&e, nu2, f_exp, NULL, c->E2);","matfun(&e, nu, f_exp, NULL, c->E2);"),
 ("const double a = k / sqrt(F); /* F^{-1/2} ∂x -> i k F^{-1/2} */","const double a = k * sqrt(F);"),
]
try:
  for a,b in muts:
    assert orig.count(a)==1,a
    open(src,'w').write(orig.replace(a,b))
    subprocess.check_call(["make","-s","-B","-C","oracle"],stdout=subprocess.DEVNULL)
    r=subprocess.run([sys.executable,"-m","pytest","tests/test_oracle_pins.py","-q","-x","-p","no:cacheprovider"],capture_output=True,text=True)
    print(("CAUGHT " if r.returncode else "SURVIVED ")+b[:60].replace("\n"," "), r.stdout.strip().splitlines()[-1])
finally:
  open(src,'w').write(orig)
  subprocess.check_call(["make","-s","-B","-C","oracle"])
