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


@pytest.mark.parametrize("m", [16, 64])
@pytest.mark.parametrize("k", [64, 96, 128, 160, 256, 320])
def test_chunk_plans_match_oracle(m, k):
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
