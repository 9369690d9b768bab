"""BTR1 / BVC1 / DPLN binary containers around the path.

Same on-disk layout as the reference (``io.py:1-99``): little-endian,
``BTR1`` = magic, u64 N, u64 M, C blocks (N*M*M), A blocks ((N-1)*M*M),
B blocks ((N-1)*M*M); ``BVC1`` = magic, u64 N, u64 M, N*M doubles.  Files are
written atomically (temp file + rename, ref io.py:29-40).
"""

from __future__ import annotations

import ctypes
import os
import struct
import tempfile

import numpy as np

from . import errors as _err
from .core import BlockTriMatrix, BlockVector


def __getattr__(name):
    # io.FileFormatError is errors.FileFormatError as currently bound (the
    # reference's own class after install(), ref errors.py:88)
    if name == "FileFormatError":
        return _err.FileFormatError
    raise AttributeError(name)


def atomic_write(path, data: bytes):
    d = os.path.dirname(os.path.abspath(path)) or "."
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".tmp-b200-")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(data)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _take(fh, nbytes, what):
    buf = fh.read(nbytes)
    if len(buf) != nbytes:
        raise _err.FileFormatError(f"truncated file while reading {what}")
    return buf


def _header(fh, magic):
    got = fh.read(4)
    if got != magic:
        raise _err.FileFormatError(f"bad magic {got!r}, expected {magic!r}")
    return struct.unpack("<QQ", _take(fh, 16, "header"))


def _f64(fh, count, what):
    return np.frombuffer(_take(fh, count * 8, what), dtype="<f8").astype(np.float64)


def write_matrix(path, p):
    blobs = [b"BTR1", struct.pack("<QQ", p.n, p.m)]
    blobs += [np.ascontiguousarray(a, dtype="<f8").tobytes() for a in (p.diag, p.lower, p.upper)]
    atomic_write(path, b"".join(blobs))


def read_matrix(path) -> BlockTriMatrix:
    with open(path, "rb") as fh:
        n, m = _header(fh, b"BTR1")
        diag = _f64(fh, n * m * m, "diag blocks").reshape(n, m, m)
        lower = _f64(fh, (n - 1) * m * m, "lower blocks").reshape(n - 1, m, m)
        upper = _f64(fh, (n - 1) * m * m, "upper blocks").reshape(n - 1, m, m)
        if fh.read(1):
            raise _err.FileFormatError("trailing bytes after BTR1 payload")
    return BlockTriMatrix(diag, lower, upper)


def write_vector(path, v):
    data = v.data if hasattr(v, "data") else np.asarray(v)
    atomic_write(path, b"BVC1" + struct.pack("<QQ", data.shape[0], data.shape[1])
                 + np.ascontiguousarray(data, dtype="<f8").tobytes())


def read_vector(path) -> BlockVector:
    with open(path, "rb") as fh:
        n, m = _header(fh, b"BVC1")
        data = _f64(fh, n * m, "vector payload").reshape(n, m)
        if fh.read(1):
            raise _err.FileFormatError("trailing bytes after BVC1 payload")
    return BlockVector(data)


# -- DPLN (plan cache) -----------------------------------------------------------
#
# Same container as the reference (ref io.py:125-203): magic "DPLN", u64 version,
# u64 n, m, ranks, L, npad, u64 fingerprint length + ASCII sha256 of the matrix.
# Version 1 is the reference's CPU plan (LU + pivots + U/V superposition factors);
# GPU_PLAN_VERSION is this package's plan: u64 split, u64 image bytes, then the
# device image of btd_plan_export (factor pool, tree inverse rows, E/H blocks).

REF_PLAN_VERSION = 1
GPU_PLAN_VERSION = 0x42320001  # "B2" tag, image version 1


def write_plan(path, plan):
    """Write a GPU plan (DevicePlan) as a DPLN container, atomically."""
    from . import _native

    lib = _native.load()
    need = ctypes.c_int64(0)
    _native.check(lib.btd_plan_export(plan.handle, None, ctypes.byref(need), None))
    image = np.empty(need.value, dtype=np.uint8)
    _native.check(lib.btd_plan_export(plan.handle, ctypes.c_void_p(image.ctypes.data), ctypes.byref(need), None))
    fp = plan.matrix_fingerprint.encode("ascii") if plan.matrix_fingerprint else b""
    head = b"".join([b"DPLN", struct.pack("<Q", GPU_PLAN_VERSION),
                     struct.pack("<QQQQQ", plan.n, plan.m, plan.ranks, plan.L, plan.npad),
                     struct.pack("<Q", len(fp)), fp, struct.pack("<QQ", plan.split, image.size)])
    d = os.path.dirname(os.path.abspath(path)) or "."
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".tmp-b200-")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(head)
            fh.write(memoryview(image))
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _ref_plan_payload_bytes(n, m, ranks, L):
    """Payload size of a reference DPLN v1 file (ref io.py:132-146)."""
    from .dichotomy import tree_node_sizes

    f8 = 8
    size = (ranks + 2 * max(ranks - 1, 0)) * m * m * f8
    per_range = 2 * (L + 1) * m * m * f8
    if L >= 2:
        per_range += (L - 1) * m * m * f8 + (L - 1) * m * 8 + max(L - 2, 0) * m * m * f8
    size += ranks * per_range
    size += sum(m * s * m * f8 for s in tree_node_sizes(ranks))
    return size


def read_plan(path, matrix, *, device=None, split=1):
    """Load a DPLN plan and bind it to ``matrix`` (fingerprint-checked, ref io.py:149-203).

    GPU plan files are imported onto ``device`` without redoing the preprocessing.
    Reference CPU plan files (version 1) are validated (header, fingerprint,
    payload length) and the GPU plan is rebuilt from ``matrix``: their LU/pivot
    and U/V factor set is not the GPU plan's factor set (f2).
    """
    from . import _native, dichotomy

    with open(path, "rb") as fh:
        if fh.read(4) != b"DPLN":
            raise _err.FileFormatError("bad magic, expected b'DPLN'")
        (version,) = struct.unpack("<Q", _take(fh, 8, "version"))
        if version not in (REF_PLAN_VERSION, GPU_PLAN_VERSION):
            raise _err.FileFormatError(f"unsupported plan version {version}")
        n, m, ranks, L, npad = struct.unpack("<QQQQQ", _take(fh, 40, "plan dims"))
        (fplen,) = struct.unpack("<Q", _take(fh, 8, "fingerprint length"))
        fingerprint = _take(fh, fplen, "fingerprint").decode("ascii")
        if matrix.fingerprint() != fingerprint:
            raise _err.FileFormatError("plan does not belong to this matrix")
        if matrix.n != n or matrix.m != m:
            raise _err.FileFormatError("plan dimensions disagree with the matrix")
        if version == REF_PLAN_VERSION:
            body = fh.seek(0, os.SEEK_END) - (4 + 8 + 40 + 8 + fplen)
            if body != _ref_plan_payload_bytes(n, m, ranks, L):
                raise _err.FileFormatError("DPLN payload length does not match its header")
            return dichotomy.plan_build(matrix, ranks, split=split, device=device)
        split, nbytes = struct.unpack("<QQ", _take(fh, 16, "image header"))
        image = np.fromfile(fh, dtype=np.uint8, count=nbytes)
        if image.size != nbytes:
            raise _err.FileFormatError("truncated file while reading plan image")
        if fh.read(1):
            raise _err.FileFormatError("trailing bytes after DPLN payload")
    lib = _native.load()
    dev = dichotomy._resolve_device(device)
    handle = ctypes.c_void_p()
    status = lib.btd_plan_import(ctypes.c_void_p(image.ctypes.data), int(nbytes), dev, None, ctypes.byref(handle))
    if status == _native.BTD_ERR_INVALID_ARG or status == _native.BTD_ERR_UNSUPPORTED:
        raise _err.FileFormatError(f"plan image rejected: {_native.last_error()}")
    _native.check(status)
    plan = dichotomy.DevicePlan(handle, n, m, int(ranks), int(split), dev, fingerprint)
    if plan.L != L or plan.npad != npad:
        plan.close()
        raise _err.FileFormatError("plan image disagrees with its DPLN header")
    return plan
