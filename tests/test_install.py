"""Drop-in installation into the reference package (oracle/_ref, built by
oracle/build_ref.sh from the unmodified reference).  Host-only checks: which
attributes install() swaps and restores, error-class rebinding, and the
DevicePlan's explicit refusal of the reference plan internals."""
import numpy as np
import pytest

import refpkg


@pytest.fixture()
def ref():
    if not refpkg.available():
        pytest.skip("reference package not built (oracle/build_ref.sh)")
    return refpkg.import_blocktri()


def test_install_swaps_entry_points_and_error_classes(ref):
    import blocktri.dichotomy as d
    import blocktri.errors as refe
    import blocktri.harness as h
    import blocktri.io as rio

    from paper_1108_4181_b200 import errors, install
    from paper_1108_4181_b200 import io as bio

    orig = d.plan_build, d.plan_solve, h.harness_solve, rio.write_plan, rio.read_plan
    try:
        install.install()
        assert d.plan_solve.__module__ == "paper_1108_4181_b200.dichotomy"
        assert d.plan_build is not orig[0]
        assert (h.harness_solve, rio.write_plan, rio.read_plan) != orig[2:]
        assert errors.SingularPivot is refe.SingularPivot
        assert errors.FileFormatError is refe.FileFormatError and bio.FileFormatError is refe.FileFormatError
        assert errors.ConfigError is refe.ConfigError
        # DeviceError has no reference analogue: re-parented under the reference root
        assert issubclass(errors.DeviceError, refe.BlocktriError)
        # the reference's own validation semantics are preserved before any GPU work
        from blocktri.core import BlockTriMatrix

        with pytest.raises(refe.InvalidRankCount):
            d.plan_build(BlockTriMatrix(np.tile(np.eye(2), (4, 1, 1))), 9)
    finally:
        install.uninstall()
    assert (d.plan_build, d.plan_solve, h.harness_solve, rio.write_plan, rio.read_plan) == orig
    assert errors.SingularPivot is not refe.SingularPivot
    assert not issubclass(errors.DeviceError, refe.BlocktriError)


def test_device_plan_refuses_reference_internals():
    from paper_1108_4181_b200.dichotomy import DevicePlan

    p = DevicePlan.__new__(DevicePlan)
    for name in ("padded", "ranges", "reduced", "tree", "inverse_rows"):
        with pytest.raises(AttributeError, match="HBM"):
            getattr(p, name)


def test_reference_protocol_trace_matches_harness(ref):
    """The trace the installed harness_solve returns equals the one the
    reference harness logs for the same plan (stages, records, bytes)."""
    from blocktri import core, dichotomy, harness

    from paper_1108_4181_b200 import configs, trace

    for (n, m, k, p) in ((24, 3, 2, 5), (40, 4, 1, 8), (16, 2, 3, 1)):
        d_, lo, up, f = configs.dominant_numpy(n, m, k, seed=n)
        plan = dichotomy.plan_build(core.BlockTriMatrix(d_, lo, up), p)
        _x, tr = harness.harness_solve(plan, f if k > 1 else f[:, :, 0])
        mine = trace.reference_protocol_trace(p, m, k)
        assert tr.records == mine.records and tr.stages == mine.stages
