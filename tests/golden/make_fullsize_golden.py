"""Reference-written goldens at the FULL BASELINE.json sizes (c1, c2, c3, c4).

Run in the build container (where /root/reference exists):

    python tests/golden/make_fullsize_golden.py c1 c2 ...   # one process per config

It runs the unmodified reference package (built into oracle/_ref by
oracle/build_ref.sh with the reference's own setup.py) through its public
``blocktri.core.BlockTriMatrix`` / ``dichotomy.plan_build`` / ``plan_solve`` on
the numpy-stream inputs of each config (``configs.generate_columns``: the exact
arrays ``configs.generate(name)`` draws, F restricted to a few columns; columns
are independent in the algorithm), and stores

* X_ref at the sampled block rows of ``fullsize_cases.sample_rows`` (all rows
  for c3) for those columns,
* per-column checksums over ALL rows (sum, sum of |x|, max |x|),
* the reference's own relative residual (``cli.py:211-214`` definition),
* input sha256s and the backend / ranks / timings used.

Backends: ``python`` (numpy ``@``) for the M = 256 / 2048 configs, whose
compiled Cython loops (``_kernels.pyx:97-108``, strided inner products) take
hours there; ``compiled`` for M = 16 / 64.  The two backends agree to ~1e-15
(SURVEY.md 8c).  Output: tests/golden/fullsize_<name>.npz and .json.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(HERE))

import fullsize_cases as FC  # noqa: E402


def _sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(a.tobytes())
    return h.hexdigest()


def run(name):
    case = FC.CASES[name]
    os.environ["BLOCKTRI_BACKEND"] = case["backend"]
    import subprocess

    subprocess.run([str(REPO / "oracle" / "build_ref.sh")], check=True)
    sys.path.insert(0, str(REPO / "oracle" / "_ref"))
    import numpy as np

    from blocktri import backend as bk
    from blocktri import core, dichotomy

    from paper_1108_4181_b200 import configs

    assert bk.backend_name() == case["backend"], bk.backend_name()
    t0 = time.time()
    diag, lower, upper, f = configs.generate_columns(name, case["cols"])
    t_gen = time.time() - t0
    sha = _sha(diag, lower, upper, f)
    P = core.BlockTriMatrix(diag, lower, upper)
    del diag, lower, upper
    t0 = time.time()
    plan = dichotomy.plan_build(P, case["ranks"])
    t_build = time.time() - t0
    t0 = time.time()
    x = dichotomy.plan_solve(plan, f)
    t_solve = time.time() - t0
    del plan
    r = P.apply(x) - f  # ref core.py:118-127
    res = float(np.abs(r).max() / np.abs(f).max())
    del r
    rows = FC.sample_rows(name)
    np.savez_compressed(HERE / f"fullsize_{name}.npz", x_rows=np.ascontiguousarray(x[rows]), rows=rows,
                        **FC.checksums(x))
    meta = dict(name=name, cols=list(case["cols"]), ranks=case["ranks"], backend=case["backend"],
                sha_inputs=sha, ref_rel_residual=res, t_generate_s=t_gen, t_build_s=t_build,
                t_solve_s=t_solve, reference="/root/reference/pkg (blocktri 0.1.0) via oracle/_ref",
                generator="tests/golden/make_fullsize_golden.py", cpus=os.cpu_count())
    (HERE / f"fullsize_{name}.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(json.dumps(meta))


if __name__ == "__main__":
    for nm in sys.argv[1:] or sorted(FC.CASES):
        run(nm)
