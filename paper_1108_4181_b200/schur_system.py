"""Generic Schur-complement domain decomposition on the GPU.

Mirrors the reference's matrix-free Schur API (``schur.py:29-378``):
``partition_numbering``, ``CgStats``, ``cg_solve``, ``BlocktriOperator``,
``SubdomainBlock``, ``SchurSystem``, ``schur_apply``, ``schur_rhs``,
``recover_interiors``, ``solve_interface``, ``solve_schur``,
``probing_preconditioner`` -- with every vector resident on the device:

* interior solves ``A_ii^{-1}`` are dichotomy plan solves (``btd_plan_solve``,
  persistent buffers per column count, so repeated solves replay the plan's
  CUDA graph);
* couplings ``A_iG``, ``A_iG^T`` and ``A_GG`` are CSR matrices in HBM applied by
  ``btd_csr_spmm``; ``BlocktriOperator.apply`` is ``btd_blocktri_apply``;
* CG runs on device vectors (two scalar reads per iteration for the step
  lengths, exactly the reference's recurrence, ``schur.py:81-121``); the
  unsymmetric interface goes through a device restarted GMRES (CGS2
  orthogonalisation, left preconditioning, ``restart = min(50, n)`` and
  ``maxit`` restart cycles like the reference's scipy call, ``schur.py:347-360``);
* ``probing_preconditioner`` applies S to all 2d+1 probes as ONE batched
  application (every subdomain solve has K = 2d+1 columns) instead of 2d+1
  single-vector applications.

Inputs may be numpy arrays or CUDA tensors; results come back in the input's
kind.  The config-3 pipeline with the explicit S is :class:`.schur.HelmholtzDD`.
Out of scope here: the reference's ``DenseOperator`` / ``SparseLUOperator`` /
``SeparableOperator`` interiors (scipy factorisations on the host) -- interiors
are block-tridiagonal dichotomy plans.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native
from . import errors as _err
from .bands import BandPreconditioner, probing_build
from .dichotomy import _current_stream, _resolve_device, _torch, plan_build_arrays

INTERFACE_LABEL = -1


def partition_numbering(labels):
    """Permutation to interior-then-interface ordering (ref schur.py:29-56).

    Returns ``(perm, inverse, slices)``: ``perm`` lists old indices in the new
    order (domain 0, domain 1, ..., interface last), ``slices[label]`` the
    label's slice of the new ordering."""
    labels = np.asarray(labels)
    if labels.ndim != 1 or labels.size == 0:
        raise _err.DimensionMismatch("labels must be a flat nonempty sequence")
    if not np.issubdtype(labels.dtype, np.integer):
        raise _err.UnlabeledNode("labels must be integers (subdomain id or -1)")
    bad = np.flatnonzero(labels < INTERFACE_LABEL)
    if bad.size:
        raise _err.UnlabeledNode(f"node {bad[0]} has label {labels[bad[0]]}")
    order = sorted(int(v) for v in np.unique(labels) if v != INTERFACE_LABEL) + [INTERFACE_LABEL]
    perm, slices, pos = [], {}, 0
    for lab in order:
        idx = np.flatnonzero(labels == lab)
        perm.append(idx)
        slices[lab] = slice(pos, pos + idx.size)
        pos += idx.size
    perm = np.concatenate(perm)
    inverse = np.empty_like(perm)
    inverse[perm] = np.arange(perm.size)
    return perm, inverse, slices


class CgStats:
    """Iteration report of one interface solve (ref schur.py:59-78)."""

    __slots__ = ("iterations", "relative_residual", "breakdown", "converged", "history")

    def __init__(self, iterations, relative_residual, breakdown, converged, history):
        self.iterations = iterations
        self.relative_residual = relative_residual
        self.breakdown = breakdown
        self.converged = converged
        self.history = history

    def __repr__(self):
        return (f"CgStats(iterations={self.iterations}, relative_residual={self.relative_residual:.3e}, "
                f"converged={self.converged})")


# ------------------------------------------------------------------- vectors
def _device():
    t = _torch()
    if t is None or not t.cuda.is_available():
        raise _err.DeviceError("the Schur DD path runs on a CUDA device")
    return t


def _to_dev(x, dev):
    """(tensor on cuda:dev, came_from_numpy)."""
    t = _device()
    if isinstance(x, t.Tensor):
        return x.to(device=f"cuda:{dev}", dtype=t.float64), False
    return t.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(f"cuda:{dev}"), True


def _back(x, was_numpy):
    return x.cpu().numpy() if was_numpy else x


def cg_solve(apply_op, rhs, precond=None, tol=1e-8, maxit=None, *, device=None):
    """Preconditioned CG on an SPD operator (ref schur.py:81-121), on device vectors.

    ``apply_op`` / ``precond`` receive and return CUDA tensors.  Stops when the
    relative preconditioned residual sqrt(r.z)/sqrt(r0.z0) <= tol or after
    ``maxit`` (default 10 sqrt(n) + 1) iterations; raises Breakdown on
    nonpositive curvature or an indefinite preconditioner."""
    t = _device()
    dev = _resolve_device(device) if not isinstance(rhs, t.Tensor) else rhs.device.index
    b, was_np = _to_dev(rhs, dev)
    n = b.numel()
    if maxit is None:
        maxit = int(10 * math.sqrt(n)) + 1
    x = t.zeros_like(b)
    if not bool(t.any(b != 0)):
        return _back(x, was_np), CgStats(0, 0.0, False, True, [0.0])
    r = b.clone()
    z = precond(r) if precond is not None else r.clone()
    rz = float(t.dot(r.reshape(-1), z.reshape(-1)))
    if rz <= 0:
        raise _err.Breakdown("preconditioner produced a nonpositive inner product")
    norm0 = math.sqrt(rz)
    p = z.clone()
    history = [1.0]
    for it in range(1, maxit + 1):
        ap = apply_op(p)
        pap = float(t.dot(p.reshape(-1), ap.reshape(-1)))
        if pap <= 0:
            raise _err.Breakdown(f"nonpositive curvature at iteration {it}")
        alpha = rz / pap
        x.add_(p, alpha=alpha)
        r.add_(ap, alpha=-alpha)
        z = precond(r) if precond is not None else r.clone()
        rz_new = float(t.dot(r.reshape(-1), z.reshape(-1)))
        if rz_new < 0:
            raise _err.Breakdown(f"indefinite preconditioner at iteration {it}")
        res = math.sqrt(rz_new) / norm0
        history.append(res)
        if res <= tol:
            return _back(x, was_np), CgStats(it, res, False, True, history)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return _back(x, was_np), CgStats(maxit, history[-1], False, False, history)


def gmres_solve(apply_op, rhs, precond=None, tol=1e-8, restart=None, maxit=None, *, device=None):
    """Restarted, left-preconditioned GMRES on device vectors with the stopping
    semantics of the reference's call ``scipy.sparse.linalg.gmres(rtol=tol,
    atol=0, restart, maxiter, M, callback_type="pr_norm")`` (ref
    schur.py:349-358; SciPy's published algorithm, restated):

    * converged iff the TRUE residual ||b - A x|| <= tol ||b|| after a cycle;
    * inside a cycle (modified Gram-Schmidt Arnoldi on M A, Givens QR) the
      preconditioned residual estimate |g_{j+1}| stops the cycle once it is
      <= ptol, where ptol starts at ||M b|| min(1, atol/||b||) and adapts after
      every cycle from the true residual (tightened 4x when the estimate passed
      but the true residual did not, loosened 1.5x otherwise);
    * ``maxit`` counts restart cycles; ``history`` holds |g_{j+1}| / ||b|| per
      inner iteration (the reference's "pr_norm" callback values).

    Returns (x, converged, history)."""
    t = _device()
    dev = _resolve_device(device) if not isinstance(rhs, t.Tensor) else rhs.device.index
    b, was_np = _to_dev(rhs, dev)
    b = b.reshape(-1)
    n = b.numel()
    restart = min(50, n) if restart is None else restart
    maxit = n if maxit is None else maxit
    M = precond if precond is not None else (lambda v: v)
    x = t.zeros_like(b)
    history = []
    bnrm = float(t.linalg.vector_norm(b))
    if bnrm == 0.0:
        return _back(x, was_np), True, history
    eps = np.finfo(np.float64).eps
    atol = tol * bnrm
    ptol_max = 1.0
    ptol = float(t.linalg.vector_norm(M(b))) * min(1.0, atol / bnrm)
    r = b.clone()
    rnorm = bnrm
    for _cycle in range(maxit):
        v0 = M(r)
        beta = float(t.linalg.vector_norm(v0))
        V = t.zeros((restart + 1, n), dtype=t.float64, device=b.device)
        V[0] = v0 / beta
        H = np.zeros((restart + 1, restart))
        cs, sn = np.zeros(restart), np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        breakdown = False
        j_done = 0
        presid = beta
        for j in range(restart):
            w = M(apply_op(V[j]))
            h0 = float(t.linalg.vector_norm(w))
            for i in range(j + 1):  # modified Gram-Schmidt
                hij = float(t.dot(V[i], w))
                H[i, j] = hij
                w = w - hij * V[i]
            hn = float(t.linalg.vector_norm(w))
            H[j + 1, j] = hn
            if hn <= eps * h0:  # exact-solution indicator
                H[j + 1, j] = 0.0
                breakdown = True
            else:
                V[j + 1] = w / hn
            for i in range(j):  # previous Givens rotations
                a_, c_ = H[i, j], H[i + 1, j]
                H[i, j], H[i + 1, j] = cs[i] * a_ + sn[i] * c_, -sn[i] * a_ + cs[i] * c_
            den = math.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if den == 0 else (H[j, j] / den, H[j + 1, j] / den)
            H[j, j], H[j + 1, j] = den, 0.0
            g[j + 1], g[j] = -sn[j] * g[j], cs[j] * g[j]
            j_done = j + 1
            presid = abs(g[j + 1])
            history.append(presid / bnrm)
            if presid <= ptol or breakdown:
                break
        y = np.linalg.lstsq(np.triu(H[:j_done, :j_done]), g[:j_done], rcond=None)[0] if j_done else np.zeros(0)
        x = x + V[:j_done].T @ t.from_numpy(y).to(b.device)
        r = b - apply_op(x)
        rnorm = float(t.linalg.vector_norm(r))
        if rnorm <= atol or breakdown:
            break
        if presid <= ptol:
            ptol_max = max(eps, 0.25 * ptol_max)
        else:
            ptol_max = min(1.0, 1.5 * ptol_max)
        ptol = presid * min(ptol_max, atol / rnorm)
    return _back(x, was_np), rnorm <= atol, history


# ------------------------------------------------------------------- operators
class _DeviceCSR:
    """A scipy sparse matrix in HBM (int64 CSR), applied by btd_csr_spmm."""

    def __init__(self, s, dev):
        import scipy.sparse

        t = _device()
        csr = scipy.sparse.csr_matrix(s)
        csr.sort_indices()
        self.shape = csr.shape
        self.dev = dev
        self.rowptr = t.from_numpy(csr.indptr.astype(np.int64)).to(f"cuda:{dev}")
        self.col = t.from_numpy(csr.indices.astype(np.int64)).to(f"cuda:{dev}")
        self.val = t.from_numpy(csr.data.astype(np.float64)).to(f"cuda:{dev}")

    def mm(self, x):
        t = _device()
        if x.shape[0] != self.shape[1]:
            raise _err.DimensionMismatch(f"operand has {x.shape[0]} rows, matrix has {self.shape[1]} columns")
        xc = x.contiguous()
        k = 1 if x.dim() == 1 else int(x.shape[1])
        y = t.empty((self.shape[0],) + tuple(x.shape[1:]), dtype=t.float64, device=x.device)
        with t.cuda.device(self.dev):
            _native.check(_native.load().btd_csr_spmm(
                ctypes.c_void_p(self.rowptr.data_ptr()), ctypes.c_void_p(self.col.data_ptr()),
                ctypes.c_void_p(self.val.data_ptr()), self.shape[0], k, ctypes.c_void_p(xc.data_ptr()),
                1.0, 0.0, ctypes.c_void_p(y.data_ptr()), _current_stream(self.dev)))
        return y


class BlocktriOperator:
    """Block-tridiagonal interior solved through a GPU dichotomy plan built once
    (ref schur.py:168-195).  ``n`` = unpadded order (the first n entries of the
    n_blocks x m vector); vectors may be numpy or CUDA tensors, (n,) or (n, K)."""

    kind = "blocktri"

    def __init__(self, mat, ranks=1, unpadded=None, *, split=1, device=None):
        t = _device()
        dev = _resolve_device(device)
        self.mat, self.device = mat, dev
        self.nb, self.m = int(mat.n), int(mat.m)
        self.n = int(unpadded) if unpadded is not None else self.nb * self.m
        self._blocks = [t.as_tensor(np.array(a) if not isinstance(a, t.Tensor) else a,
                                    dtype=t.float64).to(f"cuda:{dev}").contiguous()
                        for a in (mat.diag, mat.lower, mat.upper)]
        fp = mat.fingerprint() if hasattr(mat, "fingerprint") else None
        self.plan = plan_build_arrays(*self._blocks, ranks, split=split, device=dev, fingerprint=fp)
        self._bufs = {}

    def _buffers(self, k):
        if k not in self._bufs:
            t = _torch()
            shape = (self.nb, self.m, k)
            self._bufs[k] = (t.zeros(shape, dtype=t.float64, device=f"cuda:{self.device}"),
                             t.empty(shape, dtype=t.float64, device=f"cuda:{self.device}"))
        return self._bufs[k]

    def _stage(self, r):
        rd, was_np = _to_dev(r, self.device)
        single = rd.dim() == 1
        k = 1 if single else int(rd.shape[1])
        if rd.shape[0] != self.n:
            raise _err.DimensionMismatch(f"vector has {rd.shape[0]} rows, operator order {self.n}")
        f, x = self._buffers(k)
        f.view(self.nb * self.m, k)[: self.n].copy_(rd.reshape(self.n, k))
        return f, x, k, single, was_np

    def solve(self, r):
        t = _torch()
        f, x, k, single, was_np = self._stage(r)
        with t.cuda.device(self.device):
            _native.check(_native.load().btd_plan_solve(self.plan.handle, ctypes.c_void_p(f.data_ptr()),
                                                        ctypes.c_void_p(x.data_ptr()), k,
                                                        _current_stream(self.device)))
        out = x.view(self.nb * self.m, k)[: self.n].clone()
        return _back(out[:, 0] if single else out, was_np)

    def apply(self, xin):
        t = _torch()
        f, y, k, single, was_np = self._stage(xin)
        d, lo, up = self._blocks
        with t.cuda.device(self.device):
            _native.check(_native.load().btd_blocktri_apply(
                ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(lo.data_ptr() if lo.numel() else 0),
                ctypes.c_void_p(up.data_ptr() if up.numel() else 0), self.nb, self.m,
                ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(y.data_ptr()), k, _current_stream(self.device)))
        out = y.view(self.nb * self.m, k)[: self.n].clone()
        return _back(out[:, 0] if single else out, was_np)


class SubdomainBlock:
    """One subdomain: interior operator plus its interface couplings (ref schur.py:198-259).

    ``coupling`` = A_iG (interior rows x interface columns); ``coupling_t`` the
    interface-equation side (default A_iG^T)."""

    __slots__ = ("label", "op", "coupling", "coupling_t", "symmetric", "fast_schur", "_c", "_ct")

    def __init__(self, label, op, coupling, coupling_t=None, symmetric=True, fast_schur=False):
        import scipy.sparse

        if fast_schur:
            raise NotImplementedError("fast_schur (separable interiors) is not part of the GPU path")
        self.label, self.op, self.symmetric, self.fast_schur = label, op, symmetric, False
        self.coupling = scipy.sparse.csr_matrix(coupling)
        self.coupling_t = (scipy.sparse.csr_matrix(coupling_t) if coupling_t is not None
                           else self.coupling.T.tocsr())
        if self.coupling.shape[0] != op.n:
            raise _err.DimensionMismatch(f"coupling rows {self.coupling.shape[0]} != interior size {op.n}")
        dev = getattr(op, "device", 0)
        self._c = _DeviceCSR(self.coupling, dev)
        self._ct = _DeviceCSR(self.coupling_t, dev)

    @property
    def n(self):
        return self.op.n

    def solve(self, r):
        try:
            return self.op.solve(r)
        except _err.DeviceError:
            raise
        except Exception as exc:  # noqa: BLE001 - uniform failure surface (ref schur.py:247-253)
            raise _err.SubdomainSolveFailure(f"subdomain {self.label}: {exc}") from exc

    def schur_term(self, xg):
        """A_iG^T A_ii^{-1} A_iG xg on the device."""
        return self._ct.mm(self.solve(self._c.mm(xg)))


class SchurSystem:
    """Interior blocks + interface block of the partitioned system (ref schur.py:262-310)."""

    __slots__ = ("blocks", "a_gamma", "ngamma", "symmetric", "_ag", "device")

    def __init__(self, blocks, a_gamma, symmetric=None):
        import scipy.sparse

        self.blocks = list(blocks)
        self.a_gamma = scipy.sparse.csr_matrix(a_gamma)
        self.ngamma = self.a_gamma.shape[0]
        for blk in self.blocks:
            if blk.coupling.shape[1] != self.ngamma:
                raise _err.DimensionMismatch(f"subdomain {blk.label} coupling has {blk.coupling.shape[1]} "
                                             f"interface columns, expected {self.ngamma}")
        self.symmetric = all(b.symmetric for b in self.blocks) if symmetric is None else symmetric
        self.device = getattr(self.blocks[0].op, "device", 0) if self.blocks else _resolve_device(None)
        self._ag = _DeviceCSR(self.a_gamma, self.device)

    @property
    def interior_sizes(self):
        return [b.n for b in self.blocks]

    def split_rhs(self, f):
        total = sum(self.interior_sizes) + self.ngamma
        if f.shape[0] != total:
            raise _err.DimensionMismatch(f"rhs length {f.shape[0]}, system order {total}")
        parts, pos = [], 0
        for n in self.interior_sizes:
            parts.append(f[pos:pos + n])
            pos += n
        return parts, f[pos:]

    def assemble_solution(self, x_is, xg):
        return _torch().cat(list(x_is) + [xg])

    def apply_full(self, x):
        """Saddle operator applied to a full interior-then-interface vector."""
        xd, was_np = _to_dev(x, self.device)
        parts, xg = self.split_rhs(xd)
        out = [blk.op.apply(xi) + blk._c.mm(xg) for blk, xi in zip(self.blocks, parts)]
        yg = self._ag.mm(xg)
        for blk, xi in zip(self.blocks, parts):
            yg = yg + blk._ct.mm(xi)
        return _back(_torch().cat(out + [yg]), was_np)


def schur_apply(sys: SchurSystem, xg):
    """S xg = A_GG xg - sum_i A_iG^T A_ii^{-1} A_iG xg, matrix-free (ref schur.py:313-319)."""
    xd, was_np = _to_dev(xg, sys.device)
    y = sys._ag.mm(xd)
    for blk in sys.blocks:
        y = y - blk.schur_term(xd)
    return _back(y, was_np)


def schur_rhs(sys: SchurSystem, f):
    """f_G - sum_i A_iG^T A_ii^{-1} f_i (ref schur.py:322-328)."""
    fd, was_np = _to_dev(f, sys.device)
    parts, fg = sys.split_rhs(fd)
    y = fg.clone()
    for blk, fi in zip(sys.blocks, parts):
        y = y - blk._ct.mm(blk.solve(fi))
    return _back(y, was_np)


def recover_interiors(sys: SchurSystem, xg, f):
    """x_i = A_ii^{-1} (f_i - A_iG x_G) (ref schur.py:331-335)."""
    fd, was_np = _to_dev(f, sys.device)
    xd, _ = _to_dev(xg, sys.device)
    parts, _ = sys.split_rhs(fd)
    return [_back(blk.solve(fi - blk._c.mm(xd)), was_np) for blk, fi in zip(sys.blocks, parts)]


def solve_interface(sys: SchurSystem, f, tol=1e-8, maxit=None, precond=None):
    """Interface solve: CG when symmetric, restarted GMRES otherwise (ref schur.py:338-362)."""
    t = _device()
    fd, was_np = _to_dev(f, sys.device)
    rhs = schur_rhs(sys, fd)
    if maxit is None:
        maxit = int(10 * math.sqrt(max(sys.ngamma, 1))) + 1
    pc = None
    if precond is not None:
        pc = precond.apply if hasattr(precond, "apply") else precond
    apply_op = lambda v: schur_apply(sys, v)  # noqa: E731
    if sys.symmetric:
        xg, stats = cg_solve(apply_op, rhs, precond=pc, tol=tol, maxit=maxit)
        return _back(xg, was_np), stats
    xg, ok, history = gmres_solve(apply_op, rhs, precond=pc, tol=tol, restart=min(50, sys.ngamma), maxit=maxit)
    rnorm = float(t.linalg.vector_norm(rhs - apply_op(xg)))
    denom = float(t.linalg.vector_norm(rhs)) or 1.0
    return _back(xg, was_np), CgStats(len(history), rnorm / denom, False, ok, history)


def solve_schur(sys: SchurSystem, f, tol=1e-8, maxit=None, precond=None):
    """Interface solve then interior recovery (ref schur.py:365-372); returns
    (x_full in interior-then-interface ordering, stats)."""
    fd, was_np = _to_dev(f, sys.device)
    xg, stats = solve_interface(sys, fd, tol=tol, maxit=maxit, precond=precond)
    x_is = recover_interiors(sys, xg, fd)
    return _back(sys.assemble_solution(x_is, xg), was_np), stats


def probing_preconditioner(sys: SchurSystem, d, ranks=None):
    """Probe S to bandwidth d (one batched application of S to the 2d+1 probes)
    and wrap the band solve as a preconditioner (ref schur.py:375-378)."""
    band = probing_build(lambda probes: schur_apply(sys, probes), d, sys.ngamma, batched=True,
                         device=sys.device)
    return BandPreconditioner(band, ranks=ranks, device=sys.device), band


__all__ = ["INTERFACE_LABEL", "BlocktriOperator", "CgStats", "SchurSystem", "SubdomainBlock", "cg_solve",
           "gmres_solve", "partition_numbering", "probing_preconditioner", "recover_interiors", "schur_apply",
           "schur_rhs", "solve_interface", "solve_schur"]
