"""Diagnostic: max rel error of the GPU path vs the reference goldens, all cases, both modes."""
import os, sys
sys.path[:0] = ["tests", "oracle", "."]
import numpy as np
import blocktri_oracle as O
from golden_cases import case_inputs, load
from paper_1108_4181_b200 import BlockTriMatrix, plan_build, plan_solve
META, NPZ = load()
for mode in ("0", "1"):
    os.environ["BTD_FORCE_MODE"] = mode
    for name in sorted(k for k in META["cases"] if k != "thomas"):
        c = META["cases"][name]
        d, lo, up, f = case_inputs(c)
        try:
            plan = plan_build(BlockTriMatrix(d, lo, up), c["ranks"])
            x = plan_solve(plan, f)
            ref = NPZ["python"][f"{name}.x"]
            print(f"mode{mode} {name:10s} n={c['n']} m={c['m']} k={c['k']} P={c['ranks']} L={plan.L} err={O.max_rel_err(x, ref):.2e} res={O.rel_residual(d, lo, up, x, f):.2e}")
        except Exception as e:
            print(f"mode{mode} {name:10s} EXC {type(e).__name__}: {e}")
