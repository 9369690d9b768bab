"""Row-sharded dichotomy solve across GPUs (one process per GPU, NCCL).

The reference runs Algorithm 2 on *virtual* ranks inside one process
(``harness.py:147-216``): every rank sweeps its own range, the per-range
interface pairs (base, carry) are all-gathered in ceil(log2 p) dissemination
rounds, every rank solves the reduced system and recovers its range.  Here
the ranks are real processes, one B200 each:

* plan: each rank factors only its ranges (its block rows of the matrix) and
  emits four reduced-system contributions per range; one NCCL all-gather of
  those (4 M^2 doubles per range; the paper's step 1.2) lets every rank
  assemble the reduced system and its partition-tree inverse rows;
* solve: phase A (local fused sweeps) -> NCCL all-gather of one carry block
  per rank (the coupling into the next rank's first interface) -> phase B
  (interface RHS of the own ranges; partial series sums R_node f~ over the own
  ranges for the tree nodes whose segment crosses a rank boundary) -> NCCL
  all-gather of those partials, summed in rank order (deterministic) ->
  phase C (tree levels for the nodes this rank needs, local recovery).  This
  is the paper's "sum of a series over distributed data": M K (1 + #crossing
  nodes) doubles per rank per solve instead of the reference harness's
  all-gather of every range's (base, carry) pair.

On NVSwitch a single all-gather replaces the dissemination rounds; the stage
law (ceil(log2 p) logical stages) is reported by :func:`stage_count`.
The local compute is the C ABI of include/blocktri_b200.h; a ``backend``
object can replace it (the CPU gloo tests plug in a numpy restatement to
exercise this orchestration without a GPU).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native
from . import errors as _err

BIG = 1 << 62


def stage_count(p: int) -> int:
    """Logical dissemination stages of the interface exchange (ref harness.py:153, 280-283)."""
    return 0 if p <= 1 else math.ceil(math.log2(p))


class NativeBackend:
    """Local compute through the sm_100a library (CUDA tensors)."""

    def __init__(self, device):
        import torch

        self.torch = torch
        self.device = device
        self.lib = _native.load()
        self.comm_device = f"cuda:{device}"

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    @staticmethod
    def _p(t):
        return ctypes.c_void_p(t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data)

    def create(self, diag, lower, upper, n, m, ranks, split, rank, world):
        torch = self.torch
        flags = 0
        if isinstance(diag, torch.Tensor):
            flags = _native.BTD_MATRIX_ON_DEVICE
            arrs = [a.to(device=f"cuda:{self.device}", dtype=torch.float64).contiguous() for a in (diag, lower, upper)]
        else:
            arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (diag, lower, upper)]
        h = ctypes.c_void_p()
        info = (ctypes.c_int64 * 2)(-1, -1)
        with torch.cuda.device(self.device):
            st = self.lib.btd_plan_create_shard(self._p(arrs[0]), self._p(arrs[1]), self._p(arrs[2]), n, m, ranks,
                                                split, rank, world, self.device, flags, self._stream(),
                                                ctypes.byref(h), info)
        return h, st, int(info[0]), int(info[1])

    def info(self, h):
        pi = _native.PlanInfo()
        _native.check(self.lib.btd_plan_query(h, ctypes.byref(pi)))
        return pi

    def contrib(self, h):
        torch = self.torch
        nel = ctypes.c_int64()
        _native.check(self.lib.btd_shard_contrib(h, None, ctypes.byref(nel), None))
        buf = torch.empty(nel.value, dtype=torch.float64, device=f"cuda:{self.device}")
        with torch.cuda.device(self.device):
            _native.check(self.lib.btd_shard_contrib(h, self._p(buf), ctypes.byref(nel), self._stream()))
        return buf

    def finish(self, h, contrib_all):
        row = ctypes.c_int64(-1)
        with self.torch.cuda.device(self.device):
            st = self.lib.btd_shard_finish(h, self._p(contrib_all), self._stream(), ctypes.byref(row))
        return st, row.value

    def empty(self, nel):
        return self.torch.empty(nel, dtype=self.torch.float64, device=f"cuda:{self.device}")

    def prepare(self, f, out):
        """f as a contiguous float64 tensor on this device (converted if needed);
        ``out`` must already be one of f's shape -- the C side has no sizes."""
        t = self.torch
        dev = t.device("cuda", self.device)
        if not isinstance(f, t.Tensor):
            f = t.as_tensor(np.asarray(f, dtype=np.float64))
        f = f.to(device=dev, dtype=t.float64).contiguous()
        if out is None:
            return f, t.empty_like(f)
        if (not isinstance(out, t.Tensor) or out.device != dev or out.dtype != t.float64
                or not out.is_contiguous() or tuple(out.shape) != tuple(f.shape)):
            raise _err.DimensionMismatch(f"out must be a contiguous float64 tensor of shape {tuple(f.shape)} on {dev}")
        return f, out

    def exchange_size(self, h, k):
        nc, npart = ctypes.c_int64(), ctypes.c_int64()
        _native.check(self.lib.btd_shard_exchange_size(h, k, ctypes.byref(nc), ctypes.byref(npart)))
        return nc.value, npart.value

    def solve_a(self, h, f_local, x_local, k, carry):
        with self.torch.cuda.device(self.device):
            _native.check(self.lib.btd_shard_solve_a(h, self._p(f_local), self._p(x_local), k, self._p(carry),
                                                     self._stream()))

    def solve_b(self, h, carry_all, partial, k):
        with self.torch.cuda.device(self.device):
            _native.check(self.lib.btd_shard_solve_b(h, self._p(carry_all), self._p(partial), k, self._stream()))

    def solve_c(self, h, partial_all, f_local, x_local, k):
        with self.torch.cuda.device(self.device):
            _native.check(self.lib.btd_shard_solve_c(h, self._p(partial_all), self._p(f_local), self._p(x_local), k,
                                                     self._stream()))

    def copy_columns(self, host, c0, kc, dev, to_device, stream):
        """host (rows, m, K) pinned CPU tensor columns [c0, c0+kc) <-> dense device chunk."""
        rows = int(host.shape[0]) * int(host.shape[1])
        _native.check(self.lib.btd_copy_columns(self._p(host), rows, int(host.shape[2]), c0, kc, self._p(dev),
                                                1 if to_device else 0, ctypes.c_void_p(stream.cuda_stream)))

    def destroy(self, h):
        self.lib.btd_plan_destroy(h)


class ShardedPlan:
    """One rank's share of a row-sharded plan (mirrors ref DichotomyPlan +
    the per-rank state of ref harness.DichotomyRankProgram)."""

    def __init__(self, diag, lower, upper, ranks, *, split=1, group=None, device=None, backend=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        n, m = int(diag.shape[0]), int(diag.shape[1])
        if ranks < 1 or ranks > n:
            raise _err.InvalidRankCount(f"ranks={ranks} outside [1, N={n}]")
        if backend is None:
            import torch

            backend = NativeBackend(torch.cuda.current_device() if device is None else device)
        self.be = backend
        self.n, self.m, self.ranks, self.split = n, m, int(ranks), int(split)
        h, st, row, rng = backend.create(diag, lower, upper, n, m, self.ranks, self.split, self.rank, self.world)
        # every rank raises the same error: the first failing range wins (ref loop order)
        try:
            self._raise_consistently(st, row, rng)
        except _err.BlocktriError:
            if st == 0:
                backend.destroy(h)
            raise
        self.h = h
        local = backend.contrib(h)
        allc = backend.empty(local.numel() * self.world)
        dist.all_gather_into_tensor(allc, local, group=group)
        st, row = backend.finish(h, allc)
        if st:
            msg = _native.last_error() if isinstance(backend, NativeBackend) else "singular reduced system"
            backend.destroy(h)  # no plan object will own the handle
            self.h = None
            if st == _native.BTD_ERR_SINGULAR_PIVOT:
                raise _err.SingularPivot(row, msg)
            _native.check(st, row)
        info = backend.info(h)
        self.row_lo, self.row_hi = int(info.row_lo), int(info.row_hi)
        self.nranges, self.L = int(info.nranges), int(info.L)
        self.range_lo, self.range_hi = int(info.range_lo), int(info.range_hi)

    def _raise_consistently(self, st, row, rng):
        import torch

        code = torch.tensor([st, row, rng if st else BIG], dtype=torch.int64, device=self.be.comm_device)
        allc = torch.empty(3 * self.world, dtype=torch.int64, device=self.be.comm_device)
        self.dist.all_gather_into_tensor(allc, code, group=self.group)
        c = allc.view(self.world, 3).cpu().numpy()
        bad = [r for r in range(self.world) if c[r, 0] != 0]
        if not bad:
            return
        first = min(bad, key=lambda r: (c[r, 0] != _native.BTD_ERR_SINGULAR_PIVOT, c[r, 2]))
        code0, row0 = int(c[first, 0]), int(c[first, 1])
        if code0 == _native.BTD_ERR_SINGULAR_PIVOT:
            raise _err.SingularPivot(row0, f"block row {row0}: singular pivot (range {int(c[first, 2])})")
        if code0 == _native.BTD_ERR_INVALID_RANKS:
            raise _err.InvalidRankCount("invalid rank count")
        raise _err.DeviceError(f"shard plan build failed on rank {first} with status {code0}")

    def _gather(self, out, inp, label, trace, slot_bytes, cap_bytes):
        """One all-gather; with a trace, log its logical dissemination stages and
        its measured duration (CUDA events on the current stream, else wall clock)."""
        if trace is None:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
            return
        from .trace import allgather_schedule

        cuda = getattr(inp, "is_cuda", False)
        if cuda:
            import torch

            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        else:
            import time

            t0 = time.perf_counter()
        self.dist.all_gather_into_tensor(out, inp, group=self.group)
        if cuda:
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
        else:
            ms = (time.perf_counter() - t0) * 1e3
        allgather_schedule(trace, self.world, slot_bytes, cap_bytes, trace.stages)
        trace.timings.append((label, ms))

    def solve(self, f_local, out=None, trace=None):
        """f_local: (row_hi - row_lo, m, K) rows of this shard -> x_local
        (written into ``out`` when given; may alias f_local).  ``trace``: an
        :class:`~.trace.ExecutionTrace` (nranks = world) that receives the logical
        stages and measured times of the two exchanges."""
        rows = self.row_hi - self.row_lo
        if len(f_local.shape) != 3 or tuple(int(v) for v in f_local.shape[:2]) != (rows, self.m):
            raise _err.DimensionMismatch(
                f"shard rhs must be ({rows}, {self.m}, k) (rows {self.row_lo}..{self.row_hi}), "
                f"got {tuple(f_local.shape)}")
        k = int(f_local.shape[2])
        if k < 1:
            raise _err.empty_rhs("right-hand-side batch with zero columns")
        prep = getattr(self.be, "prepare", None)
        if prep is not None:
            f_local, x_local = prep(f_local, out)
        else:
            x_local = f_local.new_empty(f_local.shape) if out is None else out
        nc, npart = self.be.exchange_size(self.h, k)
        cap = (self.m * self.m + self.m) * 8 * k  # ref harness.py:166-180 message cap
        carry = self.be.empty(nc)
        self.be.solve_a(self.h, f_local, x_local, k, carry)
        carry_all = self.be.empty(nc * self.world)
        self._gather(carry_all, carry, "carry", trace, nc * 8, cap)
        part = self.be.empty(max(npart, 1))
        self.be.solve_b(self.h, carry_all, part, k)
        part_all = self.be.empty(max(npart, 1) * self.world)
        if npart:
            self._gather(part_all, part[:npart], "partial", trace, npart * 8, cap)
        self.be.solve_c(self.h, part_all, f_local, x_local, k)
        return x_local

    def solve_host(self, f_host, x_host, chunks=None):
        """Host-buffer solve of this shard (the reference's numpy-in / numpy-out
        contract, per rank): K columns in ``chunks`` column chunks through an
        H2D stream -> the solve (current stream, with its two all-gathers) -> a
        D2H stream, so chunk c+1's copy-in and chunk c-1's copy-out overlap chunk
        c's solve (the sharded counterpart of ``btd_plan_solve_host``).  f_host /
        x_host: pinned CPU tensors (row_hi - row_lo, m, K); returns x_host."""
        torch = self.be.torch
        shape = (self.row_hi - self.row_lo, self.m)
        for nm, t in (("f_host", f_host), ("x_host", x_host)):
            if (not isinstance(t, torch.Tensor) or t.device.type != "cpu" or t.dtype != torch.float64
                    or not t.is_contiguous() or t.dim() != 3 or tuple(t.shape[:2]) != shape):
                raise _err.DimensionMismatch(f"{nm} must be a contiguous float64 CPU tensor ({shape[0]}, {shape[1]}, k)")
        if tuple(x_host.shape) != tuple(f_host.shape):
            raise _err.DimensionMismatch("x_host must have f_host's shape")
        rows, m, k = (int(v) for v in f_host.shape)
        if chunks is None:  # as btd_plan_solve_host: >= 256-byte rows (64 columns from K = 256), <= 8
            chunks = max(1, min(8, k // (64 if k >= 256 else 32)))
        nch = max(1, min(int(chunks), k))
        while k % nch or ((k // nch) % 2 and nch > 1):
            nch -= 1
        kc = k // nch
        dev = torch.device("cuda", self.be.device)
        comp = torch.cuda.current_stream(dev)
        if not hasattr(self, "_hstreams"):
            self._hstreams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        s_in, s_out = self._hstreams
        nbuf = min(nch, 3)
        bufs = [torch.empty((rows, m, kc), dtype=torch.float64, device=dev) for _ in range(nbuf)]
        ev_in = [torch.cuda.Event() for _ in range(nch)]
        ev_sol = [torch.cuda.Event() for _ in range(nch)]
        ev_out = [torch.cuda.Event() for _ in range(nch)]
        s_in.wait_stream(comp)
        for c in range(nch):
            b = bufs[c % nbuf]
            if c >= nbuf:
                s_in.wait_event(ev_out[c - nbuf])  # buffer free again
            self.be.copy_columns(f_host, c * kc, kc, b, True, s_in)
            ev_in[c].record(s_in)
            comp.wait_event(ev_in[c])
            self.solve(b, out=b)
            ev_sol[c].record(comp)
            s_out.wait_event(ev_sol[c])
            self.be.copy_columns(x_host, c * kc, kc, b, False, s_out)
            ev_out[c].record(s_out)
        comp.wait_stream(s_out)
        s_out.synchronize()
        return x_host

    def collectives_per_solve(self, k=1):
        """1 (carry) or 2 (carry + crossing-node partial sums) all-gathers per solve."""
        return 1 + (self.be.exchange_size(self.h, k)[1] > 0)

    def close(self):
        if getattr(self, "h", None) is not None:
            self.be.destroy(self.h)
            self.h = None
