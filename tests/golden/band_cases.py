"""Seeded inputs of the band-route golden cases (shared by make_band_golden.py and tests)."""
import numpy as np

# (name, n, d, m, seed, spd)
CASES = [
    ("b1", 40, 3, 4, 1, True),
    ("b2", 37, 2, 5, 2, True),       # n not a multiple of m (identity padding)
    ("b3", 64, 4, 4, 3, False),      # unsymmetric, not SPD after symmetrization -> fallback
    ("b4", 9, 4, 4, 4, True),        # 2d+1 == n (widest probing)
    ("b5", 100, 1, 1, 5, True),      # tridiagonal, scalar blocks
    ("b6", 50, 0, 3, 6, True),       # diagonal
]


def dense_band(n, d, seed, spd):
    rng = np.random.default_rng(seed)
    a = np.zeros((n, n))
    for off in range(1, d + 1):
        lo = rng.uniform(-1, 1, n - off)
        up = lo if spd else rng.uniform(-1, 1, n - off)
        a[np.arange(off, n), np.arange(n - off)] = lo
        a[np.arange(n - off), np.arange(off, n)] = up
    if spd:
        np.fill_diagonal(a, np.abs(a).sum(axis=1) + 1.0 + rng.uniform(0, 1, n))
    else:
        np.fill_diagonal(a, rng.uniform(-0.5, 0.5, n))
    return a


def rhs(n, seed):
    return np.random.default_rng(100 + seed).standard_normal(n)
