"""GPU: the host-memory solve (btd_plan_solve_host) column-chunk pipeline.

The host path cuts the K columns into chunks (narrow 32-column edge chunks, equal
middle chunks, two compute streams with separate scratch slots, up to four device
chunk buffers in flight).  Columns are independent in Algorithm 2 (ref
dichotomy.py:298-343 solves every column with the same factors), so every chunk plan
must give the oracle's answer; this covers the plan shapes and the graph-replay /
scratch-slot reuse across repeated and alternating calls.
"""
import numpy as np
import pytest

import blocktri_oracle as O
from paper_1108_4181_b200 import BlockTriMatrix, configs, plan_build, plan_solve

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k", [(m, k) for m in (16, 64) for k in (64, 96, 128, 160, 256, 320)]
                         + [(128, 256), (256, 256), (256, 64), (200, 128)])
def test_chunk_plans_match_oracle(m, k):
    """(m = 128 / 256 / 200: narrow host chunks take narrower chain tiles so a chunk's
    chains spread over the SMs -- every tile shape must give the oracle's answer.)"""
    n, ranks = 40, 5
    d, lo, up, f = configs.dominant_numpy(n, m, k, seed=k + m)
    plan = plan_build(BlockTriMatrix(d, lo, up), ranks)
    ref = O.plan_solve(O.plan_build(d, lo, up, ranks), f)
    first = plan_solve(plan, f)
    assert O.max_rel_err(first, ref) <= 1e-9
    assert O.rel_residual(d, lo, up, first, f) <= 1e-10
    for _ in range(3):  # eager, capture, replay
        assert np.array_equal(plan_solve(plan, f), first)


def test_alternating_widths_reuse_plan():
    n, m, ranks = 33, 32, 4
    d, lo, up, _ = configs.dominant_numpy(n, m, 1, seed=3)
    plan = plan_build(BlockTriMatrix(d, lo, up), ranks)
    oplan = O.plan_build(d, lo, up, ranks)
    rng = np.random.default_rng(7)
    for k in [256, 64, 256, 2, 192, 256, 1]:
        f = rng.standard_normal((n, m, k))
        x = plan_solve(plan, f)
        assert O.max_rel_err(x, O.plan_solve(oplan, f)) <= 1e-9


def test_large_host_batches_pinned_paths():
    """Batches >= 32 MB: the caller's buffer is page-locked on first use and reused,
    solutions come from the pinned pool, pinned_array inputs are used as they are;
    every path gives the same answer as the oracle, and repeated calls are bitwise equal."""
    import paper_1108_4181_b200 as btd
    from paper_1108_4181_b200 import _native, dichotomy

    n, m, k, ranks = 512, 64, 128, 8
    d, lo, up, f = configs.dominant_numpy(n, m, k, seed=5)
    assert f.nbytes >= dichotomy.PIN_MIN_BYTES
    plan = plan_build(BlockTriMatrix(d, lo, up), ranks)
    ref = O.plan_solve(O.plan_build(d, lo, up, ranks), f)
    x1 = plan_solve(plan, f)
    assert O.max_rel_err(x1, ref) <= 1e-9
    lib = _native.load()
    import ctypes

    assert lib.btd_host_is_pinned(ctypes.c_void_p(f.ctypes.data)) == 1  # registered for f's lifetime
    assert lib.btd_host_is_pinned(ctypes.c_void_p(x1.ctypes.data)) == 1  # from the pinned pool
    x2 = plan_solve(plan, f)
    assert np.array_equal(x1, x2)
    fp = btd.pinned_array(f)
    x3 = plan_solve(plan, fp)
    assert np.array_equal(x1, x3)
    del x1, x2, x3
    assert plan_solve(plan, f[:, :, :64].copy()).shape == (n, m, 64)
    assert any(dichotomy._pool.values())
    dichotomy.release_pinned_pool()
    assert not any(dichotomy._pool.values())
