"""Install the B200 path into the reference package (drop-in by attribute).

Every consumer of the path reaches it through module attributes, so replacing
those attributes routes them all to the GPU with the reference code unchanged:

* ``blocktri.dichotomy.plan_build`` / ``plan_solve`` -- used by
  ``schur.BlocktriOperator`` (ref schur.py:176,186), ``bands.BandSolver``
  (bands.py:164,172), ``acoustic.PmlOperator`` (acoustic.py:392,405) and
  ``cli.cmd_solve`` / ``cmd_bench`` (cli.py:193,204,344);
* ``blocktri.harness.harness_solve`` -- ``cli.cmd_solve`` with ``ranks >= 2``
  and ``cmd_bench`` (cli.py:199-201,344-346).  The reference version reads the
  plan's host internals (``padded/ranges/reduced/tree/inverse_rows``,
  harness.py:186-230) that a GPU plan keeps in HBM; the installed one solves
  with :func:`plan_solve` and returns the trace the reference's message
  protocol would log (``trace.reference_protocol_trace``: same stages, records
  and bytes as harness.py:147-216; pinned by tests/test_trace.py);
* ``blocktri.io.write_plan`` / ``read_plan`` -- ``cli solve --plan-cache``
  (cli.py:183-196): GPU plans are written as GPU plan images in the DPLN
  container (io.py here), reference DPLN v1 files are validated and rebuilt
  on the GPU.  Reference (CPU) plans passed in still go to the originals.

The package's exception classes are rebound to ``blocktri.errors`` so
``except blocktri.errors.X`` keeps catching (ref errors.py).

    import paper_1108_4181_b200.install as inst
    inst.install()          # or inst.install(split=8) for the 2nd-level split
    ...
    inst.uninstall()
"""

from __future__ import annotations

import importlib

import numpy as np

from . import dichotomy as _dich
from . import errors as _err
from . import io as _io
from . import trace as _trace

_saved = {}

_PATCHES = (("dichotomy", "plan_build"), ("dichotomy", "plan_solve"), ("harness", "harness_solve"),
            ("io", "write_plan"), ("io", "read_plan"))


def install(split: int = 1, device=None, package: str = "blocktri"):
    mods = {m: importlib.import_module(f"{package}.{m}") for m in ("dichotomy", "harness", "io")}
    ref_err = importlib.import_module(f"{package}.errors")
    _err.rebind(ref_err)
    if not _saved:
        for m, attr in _PATCHES:
            _saved[(m, attr)] = (mods[m], getattr(mods[m], attr))
    orig = {key: fn for key, (_mod, fn) in _saved.items()}
    ref_trace_cls = mods["harness"].ExecutionTrace

    def plan_build(p_matrix, ranks):
        return _dich.plan_build(p_matrix, ranks, split=split, device=device)

    def harness_solve(plan, f):
        if not isinstance(plan, _dich.DevicePlan):
            return orig[("harness", "harness_solve")](plan, f)
        data = np.asarray(f, dtype=np.float64)
        x = _dich.plan_solve(plan, data)
        nrhs = data.shape[2] if data.ndim == 3 else 1
        tr = ref_trace_cls(plan.ranks)
        tr.records.extend(_trace.reference_protocol_trace(plan.ranks, plan.m, nrhs).records)
        return np.ascontiguousarray(x), tr

    def write_plan(path, plan):
        if isinstance(plan, _dich.DevicePlan):
            return _io.write_plan(path, plan)
        return orig[("io", "write_plan")](path, plan)

    def read_plan(path, matrix):
        return _io.read_plan(path, matrix, device=device, split=split)

    plan_build.__doc__ = _dich.plan_build.__doc__
    harness_solve.__doc__ = "GPU plan_solve + the reference protocol's logical trace (ref harness.py:219-233)."
    write_plan.__doc__ = _io.write_plan.__doc__
    read_plan.__doc__ = _io.read_plan.__doc__
    new = {("dichotomy", "plan_build"): plan_build, ("dichotomy", "plan_solve"): _dich.plan_solve,
           ("harness", "harness_solve"): harness_solve, ("io", "write_plan"): write_plan,
           ("io", "read_plan"): read_plan}
    for (m, attr), fn in new.items():
        setattr(mods[m], attr, fn)
    return mods["dichotomy"]


def uninstall():
    for (_m, attr), (mod, fn) in list(_saved.items()):
        setattr(mod, attr, fn)
    _saved.clear()
    _err.restore()
