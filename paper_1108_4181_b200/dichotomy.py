"""Drop-in ``plan_build`` / ``plan_solve`` on B200 (Algorithm 2 of arXiv 1108.4181).

Same call shapes, accepted input forms, return forms and exceptions as the
reference entry points ``blocktri.dichotomy.plan_build`` (dichotomy.py:318-338)
and ``plan_solve`` (dichotomy.py:358-390); the work runs in the sm_100a
library through the C ABI of ``include/blocktri_b200.h``.

* ``ranks`` is the reference's P (ranges), validated 1 <= P <= N
  (InvalidRankCount); the device plan uses the reference's ranges, identity
  padding, reduced system and partition tree.  ``split`` (keyword, default 1)
  optionally subdivides each range into that many device ranges -- the
  on-device second level of the dichotomy (hard part 1); results
  stay within the parity tolerance, and errors are reported for the
  subdivided partition.
* ``plan_solve`` takes a BlockVector, an (n, m) array, an (n, m, k) batch or a
  list of BlockVectors and returns the matching form, as a new float64 array.
  A ``torch`` CUDA tensor (n, m[, k]) stays on the device (no host copies).
* No block is factorized during a solve.  Numpy inputs are copied to the
  device and back inside the call (the reference's host-memory contract).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from . import errors as _err
from .core import BlockTriMatrix, BlockVector


def _torch():
    try:
        import torch
    except ImportError:  # pragma: no cover - torch is part of the image
        return None
    return torch


def _is_tensor(x):
    t = _torch()
    return t is not None and isinstance(x, t.Tensor)


def _current_stream(device):
    t = _torch()
    if t is None or not t.cuda.is_available():
        return None
    return ctypes.c_void_p(t.cuda.current_stream(device).cuda_stream)


def _resolve_device(device):
    t = _torch()
    if t is None or not t.cuda.is_available():
        raise _err.DeviceError("no CUDA device visible: the B200 path has no CPU fallback")
    if device is None:
        return t.cuda.current_device()
    if isinstance(device, str):
        device = t.device(device)
    if hasattr(device, "index"):
        return device.index if device.index is not None else t.cuda.current_device()
    return int(device)


def build_partition_tree(count):
    """Algorithm 1's partition tree over ``count`` reduced blocks, BFS order.

    Same node list as ref dichotomy.py:28-57: queue from (0, count-1), split at
    k = lo + (hi - lo + 1) // 2, children (lo, k-1) and (k+1, hi) when non-empty.
    Returns [(lo, hi, k, level)].  (The device plan builds the same tree in C++,
    btd_api.cu partition_tree.)"""
    nodes, queue = [], [(0, count - 1, 0)] if count > 0 else []
    head = 0
    while head < len(queue):
        lo, hi, level = queue[head]
        head += 1
        k = lo + (hi - lo + 1) // 2
        nodes.append((lo, hi, k, level))
        if k - 1 >= lo:
            queue.append((lo, k - 1, level + 1))
        if hi >= k + 1:
            queue.append((k + 1, hi, level + 1))
    return nodes


def tree_node_sizes(count):
    return [hi - lo + 1 for lo, hi, _k, _lev in build_partition_tree(count)]


class DevicePlan:
    """Preprocessing product bound to one matrix (mirrors ref DichotomyPlan,
    dichotomy.py:99-131).  Factors live in HBM of ``device``."""

    def __init__(self, handle, n, m, ranks, split, device, fingerprint):
        self._h = handle
        self.n, self.m, self.ranks, self.split, self.device = n, m, ranks, split, device
        self.matrix_fingerprint = fingerprint
        info = _native.PlanInfo()
        _native.check(_native.load().btd_plan_query(self._h, ctypes.byref(info)))
        self.info = info
        self.L = int(info.L)
        self.nranges = int(info.nranges)
        self.npad = self.L * self.nranges
        self.mode = int(info.mode)
        # every interior lower coupling is a scalar multiple of I: two-product forward sweep (8 M^2 K flops per row)
        self.scalar_coupling = bool(info.scalar_coupling)
        self.factor_bytes = int(info.factor_bytes)
        self.tree_depth = int(info.tree_depth)

    def matches(self, matrix) -> bool:
        return matrix.fingerprint() == self.matrix_fingerprint

    # host-side internals of the reference DichotomyPlan (dichotomy.py:99-131) that
    # its harness / io read; a GPU plan keeps their equivalents in HBM
    _REF_INTERNALS = ("padded", "ranges", "reduced", "tree", "inverse_rows")

    def __getattr__(self, name):
        if name in DevicePlan._REF_INTERNALS:
            raise AttributeError(
                f"DevicePlan has no host '{name}': its factors live in HBM. Solve with plan_solve; after "
                "install.install() the reference's harness.harness_solve and io.write_plan/read_plan "
                "accept GPU plans")
        raise AttributeError(name)

    def close(self):
        if getattr(self, "_h", None):
            _native.load().btd_plan_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        if not self._h:
            raise _err.DeviceError("plan was closed")
        return self._h


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr())


def plan_build_arrays(diag, lower, upper, ranks, *, split=1, device=None, fingerprint=None):
    """plan_build on raw (n,m,m)/(n-1,m,m) arrays: numpy (host) or torch CUDA
    tensors (device-resident, no host copy)."""
    lib = _native.load()
    dev = _resolve_device(device)
    if _is_tensor(diag):
        t = _torch()
        n, m = int(diag.shape[0]), int(diag.shape[1])
        arrs = [a.to(device=f"cuda:{dev}", dtype=t.float64).contiguous() for a in (diag, lower, upper)]
        flags = _native.BTD_MATRIX_ON_DEVICE
    else:
        diag = np.ascontiguousarray(diag, dtype=np.float64)
        if diag.ndim != 3 or diag.shape[1] != diag.shape[2]:
            raise _err.DimensionMismatch("diag must be (n, m, m)")
        n, m = diag.shape[0], diag.shape[1]
        lower = np.ascontiguousarray(lower, dtype=np.float64).reshape(max(n - 1, 0), m, m)
        upper = np.ascontiguousarray(upper, dtype=np.float64).reshape(max(n - 1, 0), m, m)
        arrs = [diag, lower, upper]
        flags = 0
    if n > 1:
        for a in arrs[1:]:
            if tuple(a.shape) != (n - 1, m, m):
                raise _err.DimensionMismatch(f"couplings must be {(n - 1, m, m)}, got {tuple(a.shape)}")
    handle = ctypes.c_void_p()
    err_row = ctypes.c_int64(-1)
    t = _torch()
    if t is not None and t.cuda.is_available():
        with t.cuda.device(dev):
            stream = _current_stream(dev)
            status = lib.btd_plan_create(_ptr(arrs[0]), _ptr(arrs[1]), _ptr(arrs[2]), n, m, int(ranks),
                                         int(split), dev, flags, stream, ctypes.byref(handle),
                                         ctypes.byref(err_row))
    else:  # pragma: no cover - _resolve_device already raised
        raise _err.DeviceError("no CUDA device")
    _native.check(status, err_row.value)
    return DevicePlan(handle, n, m, int(ranks), int(split), dev, fingerprint)


def plan_build(p_matrix, ranks, *, split=1, device=None):
    """Algorithm 2 step 1 (ref dichotomy.py:318-338) on the GPU.

    ``p_matrix`` is a BlockTriMatrix (this package's or the reference's).
    Raises InvalidRankCount unless 1 <= ranks <= N, SingularPivot(row) with the
    reference's range-local row."""
    n = p_matrix.n
    if ranks < 1 or ranks > n:
        raise _err.InvalidRankCount(f"ranks={ranks} outside [1, N={n}]")
    return plan_build_arrays(p_matrix.diag, p_matrix.lower, p_matrix.upper, ranks, split=split,
                             device=device, fingerprint=p_matrix.fingerprint())


def _solve_tensor(plan, f):
    t = _torch()
    squeeze = f.dim() == 2
    if f.dim() not in (2, 3) or f.shape[0] != plan.n or f.shape[1] != plan.m:
        raise _err.DimensionMismatch(
            f"rhs layout {tuple(f.shape[:2])} does not match plan ({plan.n}, {plan.m})")
    if not squeeze and f.shape[2] == 0:
        raise _err.empty_rhs("right-hand-side batch with zero columns")
    fk = f.unsqueeze(2) if squeeze else f
    fk = fk.to(device=f"cuda:{plan.device}", dtype=t.float64).contiguous()
    x = t.empty_like(fk)
    with t.cuda.device(plan.device):
        stream = _current_stream(plan.device)
        _native.check(_native.load().btd_plan_solve(plan.handle, _ptr(fk), _ptr(x), int(fk.shape[2]), stream))
    return x.squeeze(2) if squeeze else x


# ---- host memory for the numpy path ------------------------------------------
# The reference's plan_solve takes and returns numpy arrays (dichotomy.py:358-390).
# The library's host pipeline (btd_plan_solve_host) overlaps H2D, solve and D2H
# only on page-locked memory (pageable 2-D copies run at 1.5-6.5 GB/s: a c4 solve
# from pageable buffers takes ~6 s, measured), so large host solves
#   * page-lock the caller's input buffer (cudaHostRegister via btd_host_pin) for
#     the lifetime of the array that owns it -- a repeated solve of the same batch
#     pays nothing more;
#   * return their solution in a page-locked array drawn from a small pool
#     (btd_host_alloc); a block returns to the pool when its array dies (two per
#     size: the caller's previous result + the next).
# Small batches are latency-bound and take the plain path.
PIN_MIN_BYTES = 32 << 20
_POOL_KEEP = 2            # free blocks kept per size
_pinned_owners = {}       # id(owner) -> weakref.finalize
_pool = {}                # nbytes -> [ptr, ...]


class _PinnedBlock:
    __slots__ = ("ptr", "nbytes", "__weakref__")

    def __init__(self, nbytes):
        ptr = ctypes.c_void_p()
        _native.check(_native.load().btd_host_alloc(nbytes, ctypes.byref(ptr)))
        self.ptr, self.nbytes = ptr.value, nbytes

    def __del__(self):  # back to the pool (or freed past the pool's depth)
        try:
            free = _pool.setdefault(self.nbytes, [])
            if len(free) < _POOL_KEEP:
                free.append(self.ptr)
            else:
                _native.load().btd_host_free(ctypes.c_void_p(self.ptr))
        except Exception:  # pragma: no cover - interpreter teardown
            pass


def release_pinned_pool():
    """Free the page-locked solution blocks kept for reuse (arrays still alive keep theirs)."""
    lib = _native.load()
    for free in _pool.values():
        while free:
            lib.btd_host_free(ctypes.c_void_p(free.pop()))


def _pinned_empty(shape):
    """Uninitialised float64 C-contiguous array in page-locked memory."""
    count = int(np.prod(shape))
    nbytes = count * 8
    free = _pool.get(nbytes)
    if free:
        blk = _PinnedBlock.__new__(_PinnedBlock)
        blk.ptr, blk.nbytes = free.pop(), nbytes
    else:
        blk = _PinnedBlock(nbytes)
    buf = (ctypes.c_double * count).from_address(blk.ptr)
    buf._owner = blk
    return np.frombuffer(buf, dtype=np.float64).reshape(shape)


def pinned_empty(shape):
    """A float64 C-contiguous numpy array in page-locked host memory (cudaHostAlloc),
    for right-hand-side batches that are solved from the host repeatedly: its
    copies run at the full copy-engine rate (cudaHostRegister'ed pageable memory
    streams ~20% slower, profiles/r02_e2e.txt)."""
    return _pinned_empty(tuple(int(v) for v in shape))


def pinned_array(a):
    """Copy of ``a`` (float64, C order) in page-locked host memory."""
    a = np.asarray(a, dtype=np.float64)
    out = _pinned_empty(a.shape)
    np.copyto(out, a)
    return out


def _unpin(ptr):
    try:
        _native.load().btd_host_unpin(ctypes.c_void_p(ptr))
    except Exception:  # pragma: no cover - interpreter teardown
        pass


def _pin_input(a):
    """Page-lock the buffer behind ``a`` until the array owning it is collected.
    Returns True when the buffer is page-locked."""
    import weakref

    if _native.load().btd_host_is_pinned(ctypes.c_void_p(a.ctypes.data)):
        return True  # already page-locked: pinned_array / pinned_empty, a pinned torch tensor's view
    owner = a
    while isinstance(owner.base, np.ndarray):
        owner = owner.base
    if not (owner.flags.c_contiguous and owner.flags.owndata) or owner.nbytes < PIN_MIN_BYTES:
        return False
    key = id(owner)
    fin = _pinned_owners.get(key)
    if fin is not None and fin.alive:
        return True
    was = ctypes.c_int(0)
    st = _native.load().btd_host_pin(ctypes.c_void_p(owner.ctypes.data), owner.nbytes, ctypes.byref(was))
    if st != _native.BTD_OK:
        return False  # not lockable: plain copies
    if was.value:
        return True  # already page-locked (e.g. a pinned torch tensor's view)

    def drop(k=key, ptr=owner.ctypes.data):
        _pinned_owners.pop(k, None)
        _unpin(ptr)

    _pinned_owners[key] = weakref.finalize(owner, drop)
    return True


def _solve_host(plan, data):
    squeeze = data.ndim == 2
    fk = data[:, :, None] if squeeze else data
    fk = np.ascontiguousarray(fk, dtype=np.float64)
    pinned = (fk.nbytes >= PIN_MIN_BYTES and np.may_share_memory(fk, data)  # never lock a temporary copy
              and _pin_input(fk))
    x = _pinned_empty(fk.shape) if pinned else np.empty_like(fk)
    t = _torch()
    with t.cuda.device(plan.device):
        stream = _current_stream(plan.device)
        _native.check(_native.load().btd_plan_solve_host(plan.handle, _ptr(fk), _ptr(x), int(fk.shape[2]),
                                                         stream))
    return x[:, :, 0] if squeeze else x


def plan_solve(plan, f_batch):
    """Algorithm 2 step 2 (ref dichotomy.py:358-390); zero block factorizations.

    Accepts a BlockVector, an (n,m) array, an (n,m,k) batch or a list of
    BlockVectors (returned as a list), or a torch CUDA tensor (returned on
    the device)."""
    if isinstance(f_batch, (list, tuple)):
        if not f_batch:
            raise _err.empty_rhs("empty right-hand-side list")
        cls = type(f_batch[0])
        stacked = np.stack([bv.data for bv in f_batch], axis=2)
        out = plan_solve(plan, stacked)
        return [cls(np.ascontiguousarray(out[:, :, i])) for i in range(out.shape[2])]
    if _is_tensor(f_batch):
        return _solve_tensor(plan, f_batch)
    is_bv = hasattr(f_batch, "data") and type(f_batch).__name__ == "BlockVector"
    data = f_batch.data if is_bv else np.asarray(f_batch, dtype=np.float64)
    if data.ndim not in (2, 3) or data.shape[0] != plan.n or data.shape[1] != plan.m:
        raise _err.DimensionMismatch(
            f"rhs layout {data.shape[:2]} does not match plan ({plan.n}, {plan.m})")
    if data.ndim == 3 and data.shape[2] == 0:
        raise _err.empty_rhs("right-hand-side batch with zero columns")
    x = _solve_host(plan, data)
    return type(f_batch)(x) if is_bv else x


__all__ = ["DevicePlan", "plan_build", "plan_build_arrays", "plan_solve", "pinned_array", "pinned_empty",
           "release_pinned_pool",
           "BlockTriMatrix", "BlockVector"]
