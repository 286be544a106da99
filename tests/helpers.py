"""Test-side helpers (no method arithmetic beyond the error norm of R12)."""
import numpy as np


def weights_parseval(n):
    w = np.full(n // 2 + 1, 2.0)
    w[0] = 1.0
    w[-1] = 1.0  # k = n/2
    return w


def rel_l2(a, b, n):
    """Relative L2 over the 3 fields (Parseval-weighted half spectrum, R12), per leading index."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    w = weights_parseval(n)[:, None]
    d = ((a - b) ** 2 * w).sum(axis=(-1, -2, -3))
    r = (b ** 2 * w).sum(axis=(-1, -2, -3))
    return np.sqrt(d / r)


def to_np(t):
    return t.detach().cpu().numpy()
