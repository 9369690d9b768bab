"""CPU restatement of the reference band route -- TEST
INFRASTRUCTURE ONLY (tests/, never the product path).

Follows /root/reference/pkg/src/blocktri/bands.py:
  * band storage bands[k, j] = a(j + k - d, j)              (bands.py:18-41)
  * symmetrized (B + B^T)/2 in band storage                  (bands.py:73-84)
  * probing_build: 2d+1 class probes, band read-off, sym.   (bands.py:94-117)
  * band_as_blocktrid: order-m blocks, signs, identity pad   (bands.py:120-157)
Pinned against reference outputs in tests/golden/band_golden.npz
(tests/golden/make_band_golden.py).  Written vectorised; the arithmetic per
entry (one negation, one 0.5*(a+b)) is the reference's, so results are bitwise.
"""
from __future__ import annotations

import numpy as np


def from_dense(a, d):
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    bands = np.zeros((2 * d + 1, n))
    for off in range(-d, d + 1):
        j = np.arange(max(0, -off), min(n, n - off))
        bands[d + off, j] = a[j + off, j]
    return bands


def to_dense(bands, n, d):
    a = np.zeros((n, n))
    for off in range(-d, d + 1):
        j = np.arange(max(0, -off), min(n, n - off))
        a[j + off, j] = bands[d + off, j]
    return a


def symmetrized(bands, n, d):
    out = np.zeros_like(bands)
    for off in range(-d, d + 1):
        j = np.arange(max(0, -off), min(n, n - off))
        out[d + off, j] = 0.5 * (bands[d + off, j] + bands[d - off, j + off])
    return out


def probing_raw(apply_op, d, n):
    """Unsymmetrized band read off the 2d+1 class-probe responses."""
    w = 2 * d + 1
    raw = np.zeros((w, n))
    idx = np.arange(n)
    for cls_ in range(w):
        y = np.asarray(apply_op((idx % w == cls_).astype(np.float64)), dtype=np.float64)
        for j in idx[idx % w == cls_]:
            lo, hi = max(0, j - d), min(n, j + d + 1)
            raw[lo - j + d:hi - j + d, j] = y[lo:hi]
    return raw


def probing_build(apply_op, d, n):
    return symmetrized(probing_raw(apply_op, d, n), n, d)


def band_as_blocktrid(bands, n, d, m):
    nb = -(-n // m)
    diag = np.zeros((nb, m, m))
    lower = np.zeros((max(nb - 1, 0), m, m))
    upper = np.zeros((max(nb - 1, 0), m, m))
    for off in range(-d, d + 1):
        j = np.arange(max(0, -off), min(n, n - off))
        i = j + off
        v = bands[d + off, j]
        bi, r = np.divmod(i, m)
        bj, c = np.divmod(j, m)
        s = bi == bj
        diag[bi[s], r[s], c[s]] = v[s]
        s = bi == bj + 1
        lower[bj[s], r[s], c[s]] = -v[s]
        s = bi + 1 == bj
        upper[bi[s], r[s], c[s]] = -v[s]
    g = np.arange(n, nb * m)
    diag[g // m, g % m, g % m] = 1.0
    return diag, lower, upper
