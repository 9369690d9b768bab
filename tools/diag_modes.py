"""Diagnostic: GPU vs oracle across block orders / modes / rank counts."""
import os, sys
sys.path[:0] = ["tests", "oracle", "."]
import numpy as np
import blocktri_oracle as O
from paper_1108_4181_b200 import BlockTriMatrix, configs, plan_build, plan_solve
cases = [(7, 320, 8, 3, "1"), (7, 320, 8, 1, "1"), (9, 320, 8, 3, "1"), (7, 72, 8, 3, "1"), (7, 128, 8, 3, "1"),
         (7, 128, 8, 3, "0"), (7, 264, 8, 3, "1"), (12, 320, 8, 3, "1"), (7, 256, 8, 3, "1"), (7, 512, 8, 3, "1"),
         (7, 96, 8, 3, "1"), (7, 192, 8, 3, "1")]
for n, m, k, P, mode in cases:
    os.environ["BTD_FORCE_MODE"] = mode
    d, lo, up, f = configs.dominant_numpy(n, m, k, seed=1)
    x = plan_solve(plan_build(BlockTriMatrix(d, lo, up), P), f)
    ref = O.plan_solve(O.plan_build(d, lo, up, P), f)
    print(f"n={n} m={m} P={P} mode={mode} err={O.max_rel_err(x, ref):.2e} res={O.rel_residual(d, lo, up, x, f):.2e}")
