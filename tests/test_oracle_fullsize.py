"""The C oracle against the reference-written FULL-SIZE goldens
(tests/golden/fullsize_*.npz, written by the unmodified reference through
tests/golden/make_fullsize_golden.py) on identical inputs: pins the checker
that the GPU full-size parity tests and bench.py's parity report run live.
c2 by default (~30 s); BTD_ORACLE_FULLSIZE=all adds c1 and c4."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

NAMES = ["c2"] + (["c1", "c4"] if os.environ.get("BTD_ORACLE_FULLSIZE") == "all" else [])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_at_full_size(name):
    import parity

    from paper_1108_4181_b200 import configs

    g, meta = parity.golden(name)
    assert g is not None
    d, lo, up, f = configs.generate_columns(name, meta["cols"])
    assert parity.sha_inputs(d, lo, up, f) == meta["sha_inputs"]
    x = parity.oracle_columns(d, lo, up, f, configs.CONFIGS[name]["ranks"])
    rep = parity.compare_golden(name, x)
    assert rep["max_rel_err_sampled_rows"] <= 1e-12 and rep["checksum_rel_err"] <= 1e-12, rep
