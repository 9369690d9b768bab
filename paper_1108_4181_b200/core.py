"""Host-side block containers for the dichotomy path.

Mirrors the reference data types the path consumes and produces
(``pkg/src/blocktri/core.py:51-153``): an immutable block-tridiagonal matrix
with the *unsigned* storage convention -- row i reads
``-lower[i-1] x_{i-1} + diag[i] x_i - upper[i] x_{i+1} = f_i`` -- and a
block vector.  ``plan_build`` accepts either these or the reference's own
``blocktri.core.BlockTriMatrix`` (duck-typed on ``n, m, diag, lower, upper,
fingerprint``), so the package is a drop-in without the reference present.
"""

from __future__ import annotations

import hashlib

import numpy as np

from . import errors as _err


def _blocks(arr, count, m, name):
    a = np.array(arr, dtype=np.float64, order="C", copy=True)
    if count == 0 and a.size == 0:
        a = a.reshape(0, m, m)
    if a.shape != (count, m, m):
        raise _err.DimensionMismatch(f"{name}: expected shape {(count, m, m)}, got {a.shape}")
    return a


class BlockVector:
    """N blocks of length M stored as an (n, m) float64 array (ref core.py:51-81)."""

    __slots__ = ("data",)

    def __init__(self, data):
        data = np.ascontiguousarray(data, dtype=np.float64)
        if data.ndim != 2:
            raise _err.DimensionMismatch("BlockVector expects a 2-d (n, m) array")
        self.data = data

    @property
    def n(self):
        return self.data.shape[0]

    @property
    def m(self):
        return self.data.shape[1]


class BlockTriMatrix:
    """diag (n,m,m) = C_1..C_N, lower (n-1,m,m) = A_2..A_N, upper (n-1,m,m) =
    B_1..B_{N-1}; read-only after construction (ref core.py:84-153)."""

    __slots__ = ("n", "m", "diag", "lower", "upper", "_fp")

    def __init__(self, diag, lower=None, upper=None):
        diag = np.array(diag, dtype=np.float64, order="C", copy=True)
        if diag.ndim != 3 or diag.shape[1] != diag.shape[2]:
            raise _err.DimensionMismatch("diag must be (n, m, m)")
        n, m = diag.shape[0], diag.shape[1]
        if n < 1:
            raise _err.DimensionMismatch("need at least one block row")
        self.n, self.m = n, m
        self.diag = diag
        self.lower = _blocks(np.zeros((n - 1, m, m)) if lower is None else lower, n - 1, m, "lower")
        self.upper = _blocks(np.zeros((n - 1, m, m)) if upper is None else upper, n - 1, m, "upper")
        for a in (self.diag, self.lower, self.upper):
            a.flags.writeable = False
        self._fp = None

    def apply(self, x):
        """Assembled operator times an (n,m) or (n,m,k) array (ref core.py:118-127)."""
        return apply_blocktri(self.diag, self.lower, self.upper, x)

    def fingerprint(self) -> str:
        """sha256 over (n, m, diag, lower, upper) bytes, same recipe as ref core.py:145-153."""
        if self._fp is None:
            h = hashlib.sha256()
            h.update(np.int64([self.n, self.m]).tobytes())
            for a in (self.diag, self.lower, self.upper):
                h.update(a.tobytes())
            self._fp = h.hexdigest()
        return self._fp


def apply_blocktri(diag, lower, upper, x):
    x = np.asarray(x, dtype=np.float64)
    n, m = diag.shape[0], diag.shape[1]
    if x.shape[0] != n or x.shape[1] != m:
        raise _err.DimensionMismatch("vector does not match matrix layout")
    y = np.einsum("nij,nj...->ni...", diag, x)
    if n > 1:
        y[1:] -= np.einsum("nij,nj...->ni...", lower, x[:-1])
        y[:-1] -= np.einsum("nij,nj...->ni...", upper, x[1:])
    return y
