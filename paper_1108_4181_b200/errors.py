"""Exception types raised by the B200 dichotomy path.

The names, base class and ``SingularPivot.row`` attribute follow the
reference hierarchy (``pkg/src/blocktri/errors.py:4-33``) so code written
against ``blocktri`` catches the same failures.  When the reference package
is importable, :mod:`paper_1108_4181_b200.install` swaps these for the
reference classes themselves so ``except blocktri.errors.X`` keeps working.
"""


class BlocktriError(Exception):
    """Root of every error this package raises (ref errors.py:4)."""


class DimensionMismatch(BlocktriError):
    """Block counts / block orders of the operands disagree (ref errors.py:8)."""


class SingularBlock(BlocktriError):
    """A dense block is singular to working precision (ref errors.py:12)."""


class SingularPivot(BlocktriError):
    """Singular pivot block inside a sweep; ``row`` is the block row local to
    the factored (sub)matrix, exactly as the reference reports it
    (ref errors.py:16-21, _kernels.pyx:159-160)."""

    def __init__(self, row, message=None):
        self.row = row
        super().__init__(message or f"singular pivot block at block row {row}")


class IndexOutOfRange(BlocktriError):
    """Block-row index outside the valid range (ref errors.py:28)."""


class InvalidRankCount(BlocktriError):
    """ranks < 1 or ranks > N (ref errors.py:32, dichotomy.py:326-327)."""


class InconsistentRanges(BlocktriError):
    """Ranges do not tile the matrix (ref errors.py:36)."""


class DeadlockDetected(BlocktriError):
    """A rank waits on a message no rank will send (ref errors.py:40)."""


class StageViolation(BlocktriError):
    """An execution trace violates the dichotomy stage structure (ref errors.py:44)."""


class Breakdown(BlocktriError):
    """Conjugate-gradient breakdown (ref errors.py:56)."""


class UnlabeledNode(BlocktriError):
    """A mesh node is neither interior nor interface (ref errors.py:48)."""


class SubdomainSolveFailure(BlocktriError):
    """An interior solve inside the Schur complement failed (ref errors.py:52)."""


class BandTooWide(BlocktriError):
    """Probing bandwidth does not fit the operator order (ref errors.py:60)."""


class BlockTooSmall(BlocktriError):
    """Block order smaller than the band half-width (ref errors.py:64)."""


class ConfigError(BlocktriError):
    """Invalid CLI configuration (ref errors.py:84)."""


class FileFormatError(BlocktriError):
    """Malformed binary container (ref errors.py:88)."""


class DeviceError(BlocktriError):
    """CUDA / NCCL failure or missing native library (no reference analogue:
    the reference never leaves the host)."""


_BY_NAME = {
    c.__name__: c
    for c in (BlocktriError, DimensionMismatch, SingularBlock, SingularPivot,
              IndexOutOfRange, InvalidRankCount, InconsistentRanges, DeadlockDetected,
              StageViolation, Breakdown, UnlabeledNode, SubdomainSolveFailure, BandTooWide, BlockTooSmall,
              ConfigError, FileFormatError, DeviceError)
}


_ORIGINAL = dict(_BY_NAME)
_REPARENTED = {}


def restore() -> None:
    """Undo :func:`rebind`."""
    globals().update(_ORIGINAL)
    _BY_NAME.update(_ORIGINAL)


def rebind(module) -> None:
    """Use another module's same-named exception classes (e.g. blocktri.errors).

    Names the other module lacks (``DeviceError``: the reference never leaves
    the host) are re-created under that module's ``BlocktriError``, so one
    ``except blocktri.errors.BlocktriError`` catches every failure of the path.
    Code must therefore look classes up through this module at raise time
    (``errors.X`` / :func:`get`), never bind them at import."""
    g = globals()
    root = getattr(module, "BlocktriError", None)
    for name in list(_BY_NAME):
        cls = getattr(module, name, None)
        if isinstance(cls, type) and issubclass(cls, Exception):
            g[name] = cls
            _BY_NAME[name] = cls
        elif isinstance(root, type) and issubclass(root, Exception):
            key = (name, root)
            if key not in _REPARENTED:
                orig = _ORIGINAL[name]
                _REPARENTED[key] = type(name, (root, orig), {"__module__": __name__, "__doc__": orig.__doc__})
            g[name] = _REPARENTED[key]
            _BY_NAME[name] = _REPARENTED[key]


def get(name):
    return _BY_NAME[name]


_EMPTY = {}


def empty_rhs(message):
    """Error for a zero-column batch or an empty list of right-hand sides.  The
    reference fails there inside numpy with a ``ValueError`` (``np.stack`` of an
    empty list, a reshape of a size-0 array; ref dichotomy.py:364-378); this one
    is both the (current) ``DimensionMismatch`` and a ``ValueError`` so either
    ``except`` clause keeps working."""
    base = globals()["DimensionMismatch"]
    cls = _EMPTY.get(base)
    if cls is None:
        cls = _EMPTY[base] = type("EmptyRightHandSide", (base, ValueError), {"__module__": __name__})
    return cls(message)
