"""Model of the in-place DIF (synthesis) / DIT (analysis) FFT core planned for nl_core (dev tool).

Checks, in numpy, for a radix plan and a per-thread value count R:
  * the index / twiddle formulas: inverse of a natural-order spectrum lands in a digit-reversed grid
    order, pointwise products in that order, the conjugate-transposed passes bring the result back
    to natural order (compared with numpy.fft);
  * shared-memory bank conflicts of every pass in the padded layout of nl_core (element e of field f
    at f (N + N/R) + e + e/R; 16-byte accesses: a quarter warp is conflict-free iff its 8 slot
    indices are distinct mod 8), over the 3 N/R threads of the three fields.
Usage: python tools/fft_model.py 1024 16 4,16,16
"""
import sys

import numpy as np


def fpad(e, R):
    return e + e // R


def passes(N, plan):
    """per pass p: (r, L, d): block length L, stride d = L/r"""
    out, L = [], N
    for r in plan:
        out.append((r, L, L // r))
        L //= r
    assert L == 1
    return out


def butterfly_elems(b, r, L, d):
    blk, k1 = divmod(b, d)
    return [blk * L + k1 + d * s for s in range(r)], k1


def thread_butterflies(j, NJ, R, r):
    """butterflies of thread j in a pass of radix r: b = j + i*NJ, i < R/r"""
    return [j + i * NJ for i in range(R // r)]


def inverse_inplace(a, N, R, plan, sign=+1):
    x = a.astype(complex).copy()
    NJ = N // R
    for (r, L, d) in passes(N, plan):
        new = x.copy()
        for j in range(NJ):
            for b in thread_butterflies(j, NJ, R, r):
                idx, k1 = butterfly_elems(b, r, L, d)
                v = x[idx]
                # r-point DFT over k2, then twiddle w_L^{n2 k1}
                F = np.exp(sign * 2j * np.pi * np.outer(np.arange(r), np.arange(r)) / r)
                y = F @ v
                y *= np.exp(sign * 2j * np.pi * np.arange(r) * k1 / L)
                new[idx] = y
        x = new
    return x


def forward_inplace(x, N, R, plan, sign=-1):
    x = x.astype(complex).copy()
    NJ = N // R
    for (r, L, d) in reversed(passes(N, plan)):
        new = x.copy()
        for j in range(NJ):
            for b in thread_butterflies(j, NJ, R, r):
                idx, k1 = butterfly_elems(b, r, L, d)
                v = x[idx] * np.exp(sign * 2j * np.pi * np.arange(r) * k1 / L)
                F = np.exp(sign * 2j * np.pi * np.outer(np.arange(r), np.arange(r)) / r)
                new[idx] = F @ v
        x = new
    return x


def conflicts(N, R, plan):
    NJ, FS, T = N // R, N + N // R, 3 * (N // R)
    worst = 1
    for p, (r, L, d) in enumerate(passes(N, plan)):
        for i in range(R // r):
            for s in range(r):
                for q0 in range(0, T, 8):  # quarter warps over the field-major thread ids
                    ids = []
                    for t in range(q0, min(q0 + 8, T)):
                        f, j = divmod(t, NJ)
                        idx, _ = butterfly_elems(j + i * NJ, r, L, d)
                        ids.append((f * FS + fpad(idx[s], R)) % 8)
                    c = max(ids.count(v) for v in ids)
                    if c > worst:
                        print(f"  pass {p} (r={r}, L={L}, d={d}) i={i} s={s} quarter {q0}: {c}-way")
                    worst = max(worst, c)
    return worst


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    plan = [int(t) for t in sys.argv[3].split(",")] if len(sys.argv) > 3 else [4, 16, 16]
    rng = np.random.default_rng(0)
    a = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    b = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    ya, yb = inverse_inplace(a, N, R, plan), inverse_inplace(b, N, R, plan)
    ref_a = np.fft.ifft(a) * N
    print("inverse is a permutation of ifft:", np.allclose(np.sort_complex(ya), np.sort_complex(ref_a)))
    prod = ya * yb
    out = forward_inplace(prod, N, R, plan)
    ref = np.fft.fft(np.fft.ifft(a) * N * np.fft.ifft(b) * N)
    print("forward(products) == fft(products):", np.allclose(out, ref), np.abs(out - ref).max())
    print("worst bank conflict:", conflicts(N, R, plan))


if __name__ == "__main__":
    main()
