"""B200-native many-RHS block-tridiagonal dichotomy solver (arXiv 1108.4181).

Drop-in for the reference's ``blocktri.dichotomy.plan_build`` /
``plan_solve`` path, executed by hand-written sm_100a kernels behind the C ABI
in ``include/blocktri_b200.h``.  See DESIGN.md.
"""

from . import errors
from .core import BlockTriMatrix, BlockVector
from .dichotomy import DevicePlan, pinned_array, pinned_empty, plan_build, plan_build_arrays, plan_solve

__version__ = "0.1.0"

__all__ = [
    "BlockTriMatrix", "BlockVector", "DevicePlan", "errors", "pinned_array", "pinned_empty", "plan_build",
    "plan_build_arrays", "plan_solve",
]
