"""Pins the CPU oracle to the reference's own outputs (golden fixtures).

The oracle must be bitwise equal to the reference run with its numpy kernel
backend and within 1e-13 of its Cython backend (the two reference backends
differ by ~1e-15 themselves).
"""
import numpy as np
import pytest

import blocktri_oracle as O
from golden_cases import case_inputs, load, sha, singular_inputs
from paper_1108_4181_b200 import errors

META, NPZ = load()
CASES = sorted(k for k in META["cases"] if k != "thomas")


@pytest.mark.parametrize("name", CASES)
def test_inputs_regenerate_exactly(name):
    c = META["cases"][name]
    assert sha(*case_inputs(c)) == c["sha_inputs"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference(name):
    c = META["cases"][name]
    diag, lower, upper, f = case_inputs(c)
    if c["n"] * c["m"] * max(c["k"], 1) > 40000 and c["m"] >= 64:
        pytest.skip("large-m case is covered on the GPU box")
    plan = O.plan_build(diag, lower, upper, c["ranks"])
    assert plan.L == c["L"] and plan.npad == c["npad"]
    assert [list(t) for t in plan.tree] == c["tree"]
    assert O.tree_depth(c["ranks"]) == c["depth"]
    x = O.plan_solve(plan, f)
    assert np.array_equal(x, NPZ["python"][f"{name}.x"]), "not bitwise equal to reference (numpy backend)"
    assert O.max_rel_err(x, NPZ["compiled"][f"{name}.x"]) <= 1e-13
    assert np.array_equal(plan.rdiag, NPZ["python"][f"{name}.xt_rdiag"])
    assert O.rel_residual(diag, lower, upper, x, f) <= 1e-12


def test_thomas_seam_matches_reference():
    from paper_1108_4181_b200 import configs

    diag, lower, upper, f = configs.dominant_numpy(20, 5, 3, 31)
    assert sha(diag, lower, upper, f) == META["cases"]["thomas"]["sha_inputs"]
    dlu, dpiv, sup = O.thomas_factor(diag, lower, upper)
    g = NPZ["python"]
    assert np.array_equal(dlu, g["thomas.dlu"]) and np.array_equal(dpiv, g["thomas.dpiv"])
    assert np.array_equal(sup, g["thomas.supper"])
    assert np.array_equal(O.thomas_solve(dlu, dpiv, sup, lower, f), g["thomas.x"])
    assert np.abs(dlu - NPZ["compiled"]["thomas.dlu"]).max() <= 1e-14


@pytest.mark.parametrize("name", sorted(k for k in META["errors"] if k.startswith("sing")))
def test_oracle_singular_pivot_row(name):
    e = META["errors"][name]
    d, lo, up = singular_inputs(e["n"], e["m"], e["singular_row"])
    with pytest.raises(errors.SingularPivot) as info:
        O.plan_build(d, lo, up, e["ranks"])
    assert info.value.row == e["row"]


@pytest.mark.parametrize("ranks", [0, 25])
def test_oracle_invalid_ranks(ranks):
    from paper_1108_4181_b200 import configs

    d, lo, up, _ = configs.dominant_numpy(24, 2, 1, 3)
    with pytest.raises(errors.InvalidRankCount):
        O.plan_build(d, lo, up, ranks)
    assert META["errors"][f"ranks{ranks}"]["error"] == "InvalidRankCount"
