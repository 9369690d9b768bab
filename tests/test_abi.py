"""CPU checks of the C-ABI boundary: the library builds for sm_100a, loads,
and exports every entry point include/blocktri_b200.h declares (no compute
call is made without a GPU)."""
import ctypes
import os
import re
import subprocess

from paper_1108_4181_b200 import _native, build

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "blocktri_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(btd_[a-z_]+)\s*\(", text)))


def test_library_builds_and_loads():
    path = build.build()
    assert os.path.exists(path)
    lib = _native.load()
    assert lib.btd_version() == 1
    assert lib.btd_launch_count() >= 0
    assert isinstance(_native.last_error(), str)


def test_every_declared_symbol_is_exported():
    build.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    declared = _declared()
    assert declared and set(declared) == set(_native.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", nm), name


def test_sass_is_sm100a_with_dmma():
    build.build()
    out = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", _native.LIB_PATH], capture_output=True,
                                       text=True).stdout
    assert "DMMA" in out, "fp64 tensor-core path missing from SASS"


def test_status_codes_map_to_reference_errors():
    from paper_1108_4181_b200 import errors
    import pytest

    with pytest.raises(errors.DimensionMismatch):
        _native.check(1)
    with pytest.raises(errors.SingularPivot) as info:
        _native.check(2, 7)
    assert info.value.row == 7
    with pytest.raises(errors.InvalidRankCount):
        _native.check(3)
    with pytest.raises(errors.DeviceError):
        _native.check(4)


def test_sass_has_tma_bulk_copies_and_mbarriers():
    build.build()
    out = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in out, "TMA bulk-copy path missing from SASS"
    assert "SYNCS" in out, "mbarrier path missing from SASS"
