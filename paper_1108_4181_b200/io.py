"""BTR1 / BVC1 binary containers around the path.

Same on-disk layout as the reference (``io.py:1-99``): little-endian,
``BTR1`` = magic, u64 N, u64 M, C blocks (N*M*M), A blocks ((N-1)*M*M),
B blocks ((N-1)*M*M); ``BVC1`` = magic, u64 N, u64 M, N*M doubles.  Files are
written atomically (temp file + rename, ref io.py:29-40).
"""

from __future__ import annotations

import os
import struct
import tempfile

import numpy as np

from .core import BlockTriMatrix, BlockVector
from .errors import BlocktriError


class FileFormatError(BlocktriError):
    """Malformed binary container (ref errors.py:84-85)."""


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
        raise FileFormatError(f"truncated file while reading {what}")
    return buf


def _header(fh, magic):
    got = fh.read(4)
    if got != magic:
        raise FileFormatError(f"bad magic {got!r}, expected {magic!r}")
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
            raise FileFormatError("trailing bytes after BTR1 payload")
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
            raise FileFormatError("trailing bytes after BVC1 payload")
    return BlockVector(data)
