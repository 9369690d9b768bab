"""ctypes wrapper of oracle/liboracle.so (C restatement of the reference path).
TEST / BASELINE INFRASTRUCTURE ONLY."""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_lib = None


def load():
    global _lib
    if _lib is None:
        src = os.path.join(HERE, "blocktri_oracle.c")
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        lib = ctypes.CDLL(LIB)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        lib.oracle_plan_build.argtypes = [vp, vp, vp, i64, i64, i64, ctypes.POINTER(vp), ctypes.POINTER(i64)]
        lib.oracle_plan_build.restype = ctypes.c_int
        lib.oracle_plan_solve.argtypes = [vp, vp, vp, i64]
        lib.oracle_plan_solve.restype = ctypes.c_int
        lib.oracle_plan_free.argtypes = [vp]
        lib.oracle_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


class CPlan:
    def __init__(self, diag, lower, upper, ranks):
        from paper_1108_4181_b200 import errors

        lib = load()
        self.d = np.ascontiguousarray(diag, dtype=np.float64)
        n, m = self.d.shape[0], self.d.shape[1]
        self.lo = np.ascontiguousarray(lower, dtype=np.float64).reshape(max(n - 1, 0), m, m)
        self.up = np.ascontiguousarray(upper, dtype=np.float64).reshape(max(n - 1, 0), m, m)
        self.n, self.m = n, m
        h = ctypes.c_void_p()
        row = ctypes.c_int64(-1)
        st = lib.oracle_plan_build(self.d.ctypes.data, self.lo.ctypes.data, self.up.ctypes.data, n, m, ranks,
                                   ctypes.byref(h), ctypes.byref(row))
        if st == 3:
            raise errors.InvalidRankCount(f"ranks={ranks} outside [1, N={n}]")
        if st == 2:
            raise errors.SingularPivot(row.value)
        self.h = h

    def solve(self, f):
        f = np.ascontiguousarray(f, dtype=np.float64)
        squeeze = f.ndim == 2
        fk = f[:, :, None] if squeeze else f
        fk = np.ascontiguousarray(fk)
        x = np.empty_like(fk)
        load().oracle_plan_solve(self.h, fk.ctypes.data, x.ctypes.data, fk.shape[2])
        return x[:, :, 0] if squeeze else x

    def __del__(self):
        if getattr(self, "h", None):
            load().oracle_plan_free(self.h)
            self.h = None


def threads():
    return int(load().oracle_threads())
