"""Row f3 (band route), CPU part: the oracle restatement and the host-side
BandMatrix utilities against the reference's own outputs (band_golden.npz,
written by tests/golden/make_band_golden.py), bitwise; argument errors."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
import bands_oracle as B  # noqa: E402
from band_cases import CASES, dense_band  # noqa: E402

from paper_1108_4181_b200 import bands, errors  # noqa: E402

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "band_golden.npz"))


def _same(a, b):
    return np.array_equal(a, b) and np.array_equal(np.signbit(a), np.signbit(b))


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_reference(case):
    name, n, d, m, seed, spd = case
    a = dense_band(n, d, seed, spd)
    bd = B.from_dense(a, d)
    assert _same(bd, G[f"{name}.bands"])
    assert _same(B.symmetrized(bd, n, d), G[f"{name}.sym"])
    for got, key in zip(B.band_as_blocktrid(bd, n, d, m), ("diag", "lower", "upper")):
        assert _same(got, G[f"{name}.{key}"])
    assert _same(B.probing_build(lambda v: a @ v, d, n), G[f"{name}.probe"])
    assert np.array_equal(B.to_dense(bd, n, d), a)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_band_matrix_host_utilities(case):
    name, n, d, m, seed, spd = case
    a = dense_band(n, d, seed, spd)
    b = bands.BandMatrix.from_dense(a, d)
    assert _same(b.bands, G[f"{name}.bands"])
    assert _same(b.symmetrized().bands, G[f"{name}.sym"]) and b.symmetrized().symmetric
    assert np.array_equal(b.to_dense(), a)
    x = np.random.default_rng(seed).standard_normal(n)
    assert np.allclose(b.matvec(x), a @ x, rtol=0, atol=1e-13)
    assert np.array_equal(b.diagonal(), np.diag(a))


def test_argument_errors():
    with pytest.raises(errors.DimensionMismatch):
        bands.BandMatrix(0, 1)
    with pytest.raises(errors.DimensionMismatch):
        bands.BandMatrix(5, 1, np.zeros((2, 5)))
    with pytest.raises(errors.BandTooWide):
        bands.probing_build(lambda v: v, 3, 6)
    with pytest.raises(errors.BlockTooSmall):
        bands.band_as_blocktrid(bands.BandMatrix(10, 3), 2)
