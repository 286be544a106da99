"""Mutation check of the oracle pins (test infrastructure): applies plausible one-line mistakes to
oracle/rsw_oracle.c one at a time, rebuilds, runs tests/test_oracle_pins.py and reports whether a pin
catches each one; the source is restored at the end.  Run from the repo root:
    python tools/oracle_mutations.py
"""
import subprocess, sys, shutil
src='oracle/rsw_oracle.c'
orig=open(src).read()
muts=[
 ("double wk = (k == 0 || k == n / 2) ? 1.0 : 2.0;","double wk = 1.0;"),
 ("double num = 0.0, den = wnorm2(n, U + s * L);","double num = 0.0, den = wnorm2(n, Uold + s * L);"),
 ("for (int s = 1; s <= S; ++s) {\n      double num","for (int s = 1; s < S; ++s) {\n      double num"),
 ("  d_half(n, c->dhalf, v); /* P:502-504 */","  /* dropped */"),
 ("  d_half(n, c->dhalf, v); /* P:491-493 */","  d_half(n, c->dhalf, v); d_half(n, c->dhalf, v);"),
 ("exp(-p->mu * k4 * 0.5 * dT)","exp(-p->mu * k4 * dT)"),
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
