"""Drop-in installation into the reference package (runs where the reference
is importable, i.e. the build container; the GPU box has no /root/reference)."""
import os
import sys

import pytest

REF_SRC = "/tmp/blocktri_ref_golden/src"


def _ref():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not built here (tests/golden/make_golden.py builds it)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import blocktri.dichotomy as d

    return d


def test_install_swaps_entry_points_and_error_classes():
    d = _ref()
    import blocktri.errors as refe

    from paper_1108_4181_b200 import errors, install

    orig = d.plan_build, d.plan_solve
    try:
        install.install()
        assert d.plan_solve.__module__ == "paper_1108_4181_b200.dichotomy"
        assert d.plan_build is not orig[0]
        assert errors.SingularPivot is refe.SingularPivot
        # the reference's own validation semantics are preserved before any GPU work
        from blocktri.core import BlockTriMatrix
        import numpy as np

        with pytest.raises(refe.InvalidRankCount):
            d.plan_build(BlockTriMatrix(np.tile(np.eye(2), (4, 1, 1))), 9)
    finally:
        install.uninstall()
    assert (d.plan_build, d.plan_solve) == orig
    assert errors.SingularPivot is not refe.SingularPivot
