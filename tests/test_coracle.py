"""The C restatement (CPU baseline arm) against the reference goldens."""
import pytest

import blocktri_oracle as O
import coracle
from golden_cases import case_inputs, load, singular_inputs
from paper_1108_4181_b200 import errors

META, NPZ = load()


@pytest.mark.parametrize("name", sorted(k for k in META["cases"] if k != "thomas"))
def test_c_oracle_matches_reference(name):
    c = META["cases"][name]
    d, lo, up, f = case_inputs(c)
    x = coracle.CPlan(d, lo, up, c["ranks"]).solve(f)
    assert O.max_rel_err(x, NPZ["compiled"][f"{name}.x"]) <= 1e-12
    assert O.rel_residual(d, lo, up, x, f) <= 1e-12


@pytest.mark.parametrize("name", sorted(k for k in META["errors"] if k.startswith("sing")))
def test_c_oracle_singular_row(name):
    e = META["errors"][name]
    d, lo, up = singular_inputs(e["n"], e["m"], e["singular_row"])
    with pytest.raises(errors.SingularPivot) as info:
        coracle.CPlan(d, lo, up, e["ranks"])
    assert info.value.row == e["row"]


def test_c_oracle_invalid_ranks():
    d, lo, up, _ = case_inputs(META["cases"]["p2"])
    with pytest.raises(errors.InvalidRankCount):
        coracle.CPlan(d, lo, up, 0)
