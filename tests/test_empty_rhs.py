"""Zero-column batches and empty right-hand-side lists: the reference fails inside
numpy with ValueError (dichotomy.py:364-378); the mirror raises an error that is both
DimensionMismatch and ValueError, before any device work (no GPU needed here)."""
import numpy as np
import pytest

from paper_1108_4181_b200 import dichotomy, errors


class _StubPlan:
    n, m, device = 20, 3, 0


def test_zero_columns_raise_dimension_mismatch_and_value_error():
    for exc in (errors.DimensionMismatch, ValueError):
        with pytest.raises(exc):
            dichotomy.plan_solve(_StubPlan(), np.zeros((20, 3, 0)))


def test_empty_list_raises_dimension_mismatch_and_value_error():
    for exc in (errors.DimensionMismatch, ValueError):
        with pytest.raises(exc):
            dichotomy.plan_solve(_StubPlan(), [])


def test_wrong_layout_is_plain_dimension_mismatch():
    with pytest.raises(errors.DimensionMismatch) as info:
        dichotomy.plan_solve(_StubPlan(), np.zeros((19, 3, 2)))
    assert not isinstance(info.value, ValueError)


def test_empty_rhs_follows_rebound_classes():
    class RefDM(Exception):
        pass

    saved = errors.DimensionMismatch
    try:
        errors.DimensionMismatch = RefDM
        e = errors.empty_rhs("x")
        assert isinstance(e, RefDM) and isinstance(e, ValueError)
    finally:
        errors.DimensionMismatch = saved
