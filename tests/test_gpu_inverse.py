"""Preprocessing inverses D^{-1} with REAL row pivoting, on every inversion route:
one-CTA Gauss-Jordan (block order <= 64), the 8-CTA cluster Gauss-Jordan
(orders 128 / 256) and the blocked cluster-panel + DMMA-update Gauss-Jordan
(other orders above 64, e.g. 320 / 600 in mode 1).  The diagonally dominant
BASELINE configs never pivot, so these blocks are row-permuted on purpose;
the C oracle (reference pivot rule, ref _kernels.pyx:35-63) is the checker.
SingularPivot: the failing local row matches the oracle's when the singular
column comes late in the block (a duplicated row), not only at column 0."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

pytestmark = pytest.mark.gpu


def _permuted_blocks(n, m, k, seed):
    rng = np.random.default_rng(seed)
    diag = np.empty((n, m, m))
    for i in range(n):
        core = np.eye(m) + rng.uniform(-1, 1, (m, m)) * (0.4 / m)
        diag[i] = core[rng.permutation(m)]  # every column needs a row swap
    lower = rng.uniform(-1, 1, (n - 1, m, m)) * (0.05 / m)
    upper = rng.uniform(-1, 1, (n - 1, m, m)) * (0.05 / m)
    f = rng.standard_normal((n, m, k))
    return diag, lower, upper, f


@pytest.mark.parametrize("m", [24, 128, 200, 256, 320, 600])
def test_pivoting_blocks_match_oracle(m):
    import coracle
    import torch

    from paper_1108_4181_b200 import BlockTriMatrix, plan_build, plan_solve

    torch.cuda.set_device(0)
    n, k, ranks = 9, 6, 3
    d, lo, up, f = _permuted_blocks(n, m, k, seed=m)
    plan = plan_build(BlockTriMatrix(d, lo, up), ranks)
    x = plan_solve(plan, f)
    ref = coracle.CPlan(d, lo, up, ranks).solve(f)
    assert np.abs(x - ref).max() <= 1e-9 * np.abs(ref).max()
    y = np.einsum("nij,njk->nik", d, x)
    y[1:] -= np.einsum("nij,njk->nik", lo, x[:-1])
    y[:-1] -= np.einsum("nij,njk->nik", up, x[1:])
    assert np.abs(y - f).max() <= 1e-10 * np.abs(f).max()


@pytest.mark.parametrize("m", [40, 128, 256, 320])
@pytest.mark.parametrize("bad_row", [4, 7])
def test_singular_pivot_late_column(m, bad_row):
    import coracle
    import torch

    from paper_1108_4181_b200 import BlockTriMatrix, errors, plan_build

    torch.cuda.set_device(0)
    n, ranks = 12, 2
    d, lo, up, _ = _permuted_blocks(n, m, 1, seed=3 * m + bad_row)
    d[bad_row, -1] = d[bad_row, 0]  # duplicated row: singular at a late column
    lo[bad_row - 1] = 0.0
    up[bad_row] = 0.0
    with pytest.raises(errors.SingularPivot) as ref:
        coracle.CPlan(d, lo, up, ranks)
    with pytest.raises(errors.SingularPivot) as got:
        plan_build(BlockTriMatrix(d, lo, up), ranks)
    assert got.value.row == ref.value.row
