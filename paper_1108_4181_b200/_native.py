"""ctypes binding of the C ABI in include/blocktri_b200.h.

The shared library is built in-tree (``python -m paper_1108_4181_b200.build``
or ``__graft_entry__.build()``) into ``paper_1108_4181_b200/_lib``.  There is
no fallback: a missing library or a machine without a CUDA device raises
:class:`~paper_1108_4181_b200.errors.DeviceError`.
"""

from __future__ import annotations

import ctypes
import os

from . import errors as _err

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
# BTD_LIB_PATH: an alternative in-tree build of the same library (A/B tuning runs)
LIB_PATH = os.environ.get("BTD_LIB_PATH") or os.path.join(LIB_DIR, "libblocktri_b200.so")

BTD_OK = 0
BTD_ERR_DIMENSION = 1
BTD_ERR_SINGULAR_PIVOT = 2
BTD_ERR_INVALID_RANKS = 3
BTD_ERR_CUDA = 4
BTD_ERR_NCCL = 5
BTD_ERR_OOM = 6
BTD_ERR_INVALID_ARG = 7
BTD_ERR_UNSUPPORTED = 8
BTD_MATRIX_ON_DEVICE = 1

# Every symbol include/blocktri_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "btd_plan_create",
    "btd_plan_solve",
    "btd_plan_solve_host",
    "btd_plan_destroy",
    "btd_plan_query",
    "btd_plan_export",
    "btd_plan_import",
    "btd_band_to_blocktri",
    "btd_band_from_probes",
    "btd_blocktri_apply",
    "btd_csr_spmm",
    "btd_plan_create_shard",
    "btd_shard_contrib",
    "btd_shard_finish",
    "btd_shard_exchange_size",
    "btd_shard_solve_a",
    "btd_shard_solve_b",
    "btd_shard_solve_c",
    "btd_plan_set_profiling",
    "btd_plan_phase_times",
    "btd_copy_columns",
    "btd_host_pin",
    "btd_host_is_pinned",
    "btd_host_unpin",
    "btd_host_alloc",
    "btd_host_free",
    "btd_launch_count",
    "btd_last_error",
    "btd_version",
)


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("m", ctypes.c_int64), ("mp", ctypes.c_int64),
        ("ranks", ctypes.c_int64), ("split", ctypes.c_int64), ("nranges", ctypes.c_int64),
        ("L", ctypes.c_int64), ("tree_nodes", ctypes.c_int64), ("tree_depth", ctypes.c_int64),
        ("factor_bytes", ctypes.c_int64), ("row_lo", ctypes.c_int64), ("row_hi", ctypes.c_int64),
        ("device", ctypes.c_int32), ("mode", ctypes.c_int32),
        ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
        ("range_lo", ctypes.c_int64), ("range_hi", ctypes.c_int64),
        ("scalar_coupling", ctypes.c_int64),
    ]


_lib = None


def load():
    """Load the library once; raise DeviceError (never fall back) if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise _err.DeviceError(
            f"native library missing: {LIB_PATH} (run `python -m paper_1108_4181_b200.build`)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    lib.btd_plan_create.argtypes = [dp, dp, dp, i64, i64, i64, i64, i32, i32, vp,
                                    ctypes.POINTER(vp), ctypes.POINTER(i64)]
    lib.btd_plan_create.restype = i32
    lib.btd_plan_solve.argtypes = [vp, dp, dp, i64, vp]
    lib.btd_plan_solve.restype = i32
    lib.btd_plan_solve_host.argtypes = [vp, dp, dp, i64, vp]
    lib.btd_plan_solve_host.restype = i32
    lib.btd_plan_destroy.argtypes = [vp]
    lib.btd_plan_destroy.restype = i32
    lib.btd_plan_query.argtypes = [vp, ctypes.POINTER(PlanInfo)]
    lib.btd_plan_query.restype = i32
    lib.btd_plan_export.argtypes = [vp, vp, ctypes.POINTER(i64), vp]
    lib.btd_plan_export.restype = i32
    lib.btd_plan_import.argtypes = [vp, i64, i32, vp, ctypes.POINTER(vp)]
    lib.btd_plan_import.restype = i32
    lib.btd_band_to_blocktri.argtypes = [dp, i64, i64, i64, dp, dp, dp, vp]
    lib.btd_band_to_blocktri.restype = i32
    lib.btd_band_from_probes.argtypes = [dp, i64, i64, i64, dp, vp]
    lib.btd_band_from_probes.restype = i32
    lib.btd_blocktri_apply.argtypes = [dp, dp, dp, i64, i64, dp, dp, i64, vp]
    lib.btd_blocktri_apply.restype = i32
    lib.btd_csr_spmm.argtypes = [dp, dp, dp, i64, i64, dp, ctypes.c_double, ctypes.c_double, dp, vp]
    lib.btd_csr_spmm.restype = i32
    lib.btd_plan_create_shard.argtypes = [dp, dp, dp, i64, i64, i64, i64, i32, i32, i32, i32, vp,
                                          ctypes.POINTER(vp), ctypes.POINTER(i64)]
    lib.btd_plan_create_shard.restype = i32
    lib.btd_shard_contrib.argtypes = [vp, dp, ctypes.POINTER(i64), vp]
    lib.btd_shard_contrib.restype = i32
    lib.btd_shard_finish.argtypes = [vp, dp, vp, ctypes.POINTER(i64)]
    lib.btd_shard_finish.restype = i32
    lib.btd_shard_exchange_size.argtypes = [vp, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.btd_shard_exchange_size.restype = i32
    lib.btd_shard_solve_a.argtypes = [vp, dp, dp, i64, dp, vp]
    lib.btd_shard_solve_a.restype = i32
    lib.btd_shard_solve_b.argtypes = [vp, dp, dp, i64, vp]
    lib.btd_shard_solve_b.restype = i32
    lib.btd_shard_solve_c.argtypes = [vp, dp, dp, dp, i64, vp]
    lib.btd_shard_solve_c.restype = i32
    lib.btd_plan_set_profiling.argtypes = [vp, i32]
    lib.btd_plan_set_profiling.restype = i32
    lib.btd_plan_phase_times.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64), i32]
    lib.btd_plan_phase_times.restype = i32
    lib.btd_copy_columns.argtypes = [dp, i64, i64, i64, i64, dp, i32, vp]
    lib.btd_copy_columns.restype = i32
    lib.btd_host_pin.argtypes = [vp, i64, ctypes.POINTER(i32)]
    lib.btd_host_pin.restype = i32
    lib.btd_host_is_pinned.argtypes = [vp]
    lib.btd_host_is_pinned.restype = i32
    lib.btd_host_unpin.argtypes = [vp]
    lib.btd_host_unpin.restype = i32
    lib.btd_host_alloc.argtypes = [i64, ctypes.POINTER(vp)]
    lib.btd_host_alloc.restype = i32
    lib.btd_host_free.argtypes = [vp]
    lib.btd_host_free.restype = i32
    lib.btd_launch_count.argtypes = []
    lib.btd_launch_count.restype = i64
    lib.btd_last_error.argtypes = []
    lib.btd_last_error.restype = ctypes.c_char_p
    lib.btd_version.argtypes = []
    lib.btd_version.restype = i32
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().btd_last_error()
    return msg.decode() if msg else ""


def check(status: int, err_row: int = -1) -> None:
    """Map a C status to the reference exception classes (ref errors.py)."""
    if status == BTD_OK:
        return
    msg = last_error()
    if status == BTD_ERR_DIMENSION:
        raise _err.DimensionMismatch(msg)
    if status == BTD_ERR_SINGULAR_PIVOT:
        raise _err.SingularPivot(int(err_row), msg)
    if status == BTD_ERR_INVALID_RANKS:
        raise _err.InvalidRankCount(msg)
    raise _err.DeviceError(f"status {status}: {msg}")


def launch_count() -> int:
    return int(load().btd_launch_count())
