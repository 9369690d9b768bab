"""Install the B200 path into the reference package (drop-in by attribute).

Every consumer of the path reaches it through the module attributes
``blocktri.dichotomy.plan_build`` / ``plan_solve`` (ref schur.py:176,186,
bands.py:164,172, acoustic.py:392,405, cli.py:193,204,344), so replacing
those two attributes routes them all to the GPU.  The package's exception
classes are rebound to ``blocktri.errors`` so ``except blocktri.errors.X``
keeps catching (ref errors.py).

    import paper_1108_4181_b200.install as inst
    inst.install()          # or inst.install(split=8) for the 2nd-level split
    ...
    inst.uninstall()
"""

from __future__ import annotations

import importlib

from . import dichotomy as _dich
from . import errors as _err

_saved = {}


def install(split: int = 1, device=None, package: str = "blocktri"):
    ref_dich = importlib.import_module(f"{package}.dichotomy")
    ref_err = importlib.import_module(f"{package}.errors")
    _err.rebind(ref_err)
    if "plan_build" not in _saved:
        _saved["plan_build"] = ref_dich.plan_build
        _saved["plan_solve"] = ref_dich.plan_solve
        _saved["module"] = ref_dich

    def plan_build(p_matrix, ranks):
        return _dich.plan_build(p_matrix, ranks, split=split, device=device)

    plan_build.__doc__ = _dich.plan_build.__doc__
    ref_dich.plan_build = plan_build
    ref_dich.plan_solve = _dich.plan_solve
    return ref_dich


def uninstall():
    mod = _saved.pop("module", None)
    if mod is not None:
        mod.plan_build = _saved.pop("plan_build")
        mod.plan_solve = _saved.pop("plan_solve")
    _err.restore()
