import os, sys
sys.path[:0] = ["tests", "oracle", "."]
import numpy as np
import blocktri_oracle as O
from paper_1108_4181_b200 import BlockTriMatrix, configs, plan_build, plan_solve
for n, m, k, P, mode in [(7, 256, 8, 3, "0"), (7, 256, 8, 3, "1"), (7, 256, 64, 3, "1"), (7, 256, 64, 3, "0"),
                         (7, 256, 8, 1, "0"), (2, 256, 8, 1, "1"), (2, 256, 8, 1, "0"), (3, 256, 8, 1, "0"),
                         (3, 256, 2, 1, "1"), (1, 256, 2, 1, "0"), (3, 200, 2, 1, "0"), (3, 232, 2, 1, "0")]:
    os.environ["BTD_FORCE_MODE"] = mode
    d, lo, up, f = configs.dominant_numpy(n, m, k, seed=1)
    x = plan_solve(plan_build(BlockTriMatrix(d, lo, up), P), f)
    ref = O.plan_solve(O.plan_build(d, lo, up, P), f)
    print(f"n={n} m={m} k={k} P={P} mode={mode} err={O.max_rel_err(x, ref):.2e} res={O.rel_residual(d, lo, up, x, f):.2e}")
