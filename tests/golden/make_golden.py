"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch dir under /tmp, builds the Cython
kernels there (``setup.py build_ext --inplace``; the reference's own build
recipe, nothing copied into this repo), then runs the reference's public
``blocktri.dichotomy.plan_build`` / ``plan_solve`` and
``blocktri.core.thomas_factor`` / ``thomas_solve`` on seeded inputs under both
kernel backends (``BLOCKTRI_BACKEND=compiled`` and ``python``).  Inputs are
regenerated from seeds by ``paper_1108_4181_b200.configs`` in the tests; only
their sha256 is stored here, plus the reference outputs.

Output: tests/golden/golden_<backend>.npz and tests/golden/cases.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
SCRATCH = Path("/tmp/blocktri_ref_golden")

# (name, kind, n, m, k, ranks, seed, form)   form: "3d" (n,m,k) or "2d" (n,m)
CASES = [
    ("c0", "dominant", 512, 8, 32, 4, 0, "3d"),
    ("p1", "dominant", 32, 3, 5, 1, 11, "3d"),
    ("p2", "dominant", 33, 4, 3, 2, 12, "3d"),
    ("p3_nodiv", "dominant", 37, 3, 4, 5, 13, "3d"),
    ("p8", "dominant", 64, 4, 10, 8, 14, "3d"),
    ("pN", "dominant", 16, 2, 2, 16, 15, "3d"),
    ("allpad", "dominant", 5, 2, 3, 4, 16, "3d"),      # last range entirely padding
    ("lenone", "dominant", 10, 3, 2, 9, 17, "3d"),     # L=2 / L=1 mixtures
    ("m1", "dominant", 40, 1, 3, 6, 18, "3d"),
    ("k1", "dominant", 48, 5, 1, 4, 19, "3d"),
    ("vec2d", "dominant", 30, 4, 0, 3, 20, "2d"),
    ("n1", "dominant", 1, 4, 3, 1, 21, "3d"),
    ("m8p7", "dominant", 100, 8, 16, 7, 22, "3d"),
    ("m16p12", "dominant", 300, 16, 6, 12, 23, "3d"),
    ("m64", "dominant", 96, 64, 6, 6, 24, "3d"),
    ("strip16", "strip", 64, 16, 4, 4, 25, "3d"),
    ("strip64", "strip", 40, 64, 8, 5, 26, "3d"),
]

# (name, n, m, ranks, singular_row)  -- a zero diag block at global row
# `singular_row` with zero couplings around it => singular sweep pivot.
ERROR_CASES = [
    ("sing_r7", 24, 3, 3, 7),
    ("sing_r0_range2", 24, 3, 3, 17),
    ("sing_iface", 24, 3, 3, 8),     # singular block sitting on an interface row
]


def _sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(a.tobytes())
    return h.hexdigest()


def _inputs(kind, n, m, k, seed):
    sys.path.insert(0, str(REPO))
    from paper_1108_4181_b200 import configs

    if kind == "dominant":
        return configs.dominant_numpy(n, m, k, seed)
    return configs.strip_numpy(n, m, k, 0.01, seed)


def singular_inputs(n, m, row, seed=5):
    import numpy as np

    sys.path.insert(0, str(REPO))
    from paper_1108_4181_b200 import configs

    diag, lower, upper, _ = configs.dominant_numpy(n, m, 0, seed)
    diag[row] = 0.0
    if row > 0:
        upper[row - 1] = 0.0
        lower[row - 1] = 0.0
    if row < n - 1:
        lower[row] = 0.0
        upper[row] = 0.0
    return diag, lower, upper


def build_reference():
    so = list((SCRATCH / "src" / "blocktri").glob("_kernels*.so"))
    if so:
        return
    if SCRATCH.exists():
        shutil.rmtree(SCRATCH)
    shutil.copytree("/root/reference/pkg", SCRATCH)
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                   check=True, capture_output=True)


def run_backend(backend):
    """Child process: import the reference under one backend, emit outputs."""
    import numpy as np

    os.environ["BLOCKTRI_BACKEND"] = backend
    sys.path.insert(0, str(SCRATCH / "src"))
    from blocktri import backend as bk
    from blocktri import core, dichotomy, errors

    assert bk.backend_name() == backend, bk.backend_name()
    out = {}
    meta = {}
    for (name, kind, n, m, k, ranks, seed, form) in CASES:
        diag, lower, upper, f = _inputs(kind, n, m, max(k, 1), seed)
        if form == "2d":
            f = np.ascontiguousarray(f[:, :, 0])
        P = core.BlockTriMatrix(diag, lower, upper)
        plan = dichotomy.plan_build(P, ranks)
        x = dichotomy.plan_solve(plan, f)
        out[f"{name}.x"] = x
        out[f"{name}.xt_rdiag"] = plan.reduced.matrix.diag
        meta[name] = dict(kind=kind, n=n, m=m, k=k, ranks=ranks, seed=seed, form=form,
                          sha_inputs=_sha(diag, lower, upper, f), L=plan.L, npad=plan.npad,
                          depth=plan.tree.depth, tree=[list(t) for t in plan.tree.nodes],
                          fingerprint=P.fingerprint())
    # Thomas level (kernel seam) pins on one case
    diag, lower, upper, f = _inputs("dominant", 20, 5, 3, 31)
    dlu, dpiv, sup = bk.thomas_factor(diag, lower, upper)
    out["thomas.dlu"], out["thomas.dpiv"], out["thomas.supper"] = dlu, dpiv, sup
    out["thomas.x"] = bk.thomas_solve(dlu, dpiv, sup, lower, f)
    meta["thomas"] = dict(n=20, m=5, k=3, seed=31, sha_inputs=_sha(diag, lower, upper, f))
    errs = {}
    for (name, n, m, ranks, row) in ERROR_CASES:
        d, lo, up = singular_inputs(n, m, row)
        try:
            dichotomy.plan_build(core.BlockTriMatrix(d, lo, up), ranks)
            errs[name] = dict(error=None)
        except errors.BlocktriError as exc:
            errs[name] = dict(error=type(exc).__name__, row=getattr(exc, "row", None),
                              n=n, m=m, ranks=ranks, singular_row=row)
    for ranks in (0, 25):
        d, lo, up, _ = _inputs("dominant", 24, 2, 1, 3)
        try:
            dichotomy.plan_build(core.BlockTriMatrix(d, lo, up), ranks)
            errs[f"ranks{ranks}"] = dict(error=None)
        except errors.BlocktriError as exc:
            errs[f"ranks{ranks}"] = dict(error=type(exc).__name__, n=24, m=2, ranks=ranks)
    d, lo, up, _ = _inputs("dominant", 24, 2, 1, 3)
    plan = dichotomy.plan_build(core.BlockTriMatrix(d, lo, up), 3)
    try:
        dichotomy.plan_solve(plan, np.zeros((23, 2, 1)))
        errs["dim"] = dict(error=None)
    except errors.BlocktriError as exc:
        errs["dim"] = dict(error=type(exc).__name__)
    np.savez_compressed(HERE / f"golden_{backend}.npz", **out)
    return meta, errs


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        meta, errs = run_backend(sys.argv[2])
        print(json.dumps(dict(meta=meta, errors=errs)))
        return
    build_reference()
    results = {}
    for backend in ("compiled", "python"):
        res = subprocess.run([sys.executable, __file__, "--child", backend], check=True,
                             capture_output=True, text=True)
        results[backend] = json.loads(res.stdout.strip().splitlines()[-1])
    assert results["compiled"]["meta"] == results["python"]["meta"]
    assert results["compiled"]["errors"] == results["python"]["errors"]
    cases = dict(cases=results["python"]["meta"], errors=results["python"]["errors"],
                 generator="tests/golden/make_golden.py",
                 reference="/root/reference/pkg (blocktri 0.1.0)")
    (HERE / "cases.json").write_text(json.dumps(cases, indent=1, sort_keys=True))
    print("wrote", sorted(p.name for p in HERE.glob("golden_*.npz")))


if __name__ == "__main__":
    main()
