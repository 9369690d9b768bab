"""Randomised GPU parity (hypothesis): random N, M (odd / padded block orders),
K (odd K takes the non-TMA path), P, split and sweep mode against the CPU
oracle -- the reference's property-test style (test_core.py:194-208) applied
to the whole dichotomy path.  Bars: max rel err <= 1e-9, rel residual <= 1e-10."""
import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import blocktri_oracle as O
from paper_1108_4181_b200 import BlockTriMatrix, configs, plan_build, plan_solve

pytestmark = pytest.mark.gpu


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(n=st.integers(1, 90), m=st.sampled_from([1, 2, 3, 5, 8, 13, 16, 24, 33, 64, 70, 128, 136, 256]),
       k=st.one_of(st.integers(1, 40), st.sampled_from([64, 128])), pfrac=st.floats(0.0, 1.0), split=st.sampled_from([1, 1, 2, 3]),
       mode=st.sampled_from(["0", "0", "1"]), seed=st.integers(0, 10_000))
def test_random_problems_match_oracle(n, m, k, pfrac, split, mode, seed):
    if m >= 128:
        n = min(n, 24)  # large blocks: keep the numpy oracle fast
    ranks = max(1, min(n, 1 + int(pfrac * (n - 1))))
    d, lo, up, f = configs.dominant_numpy(n, m, k, seed=seed)
    os.environ["BTD_FORCE_MODE"] = mode
    try:
        plan = plan_build(BlockTriMatrix(d, lo, up), ranks, split=split)
    finally:
        os.environ.pop("BTD_FORCE_MODE", None)
    x = plan_solve(plan, f)
    ref = O.plan_solve(O.plan_build(d, lo, up, ranks), f)
    assert O.max_rel_err(x, ref) <= 1e-9
    assert O.rel_residual(d, lo, up, x, f) <= 1e-10
