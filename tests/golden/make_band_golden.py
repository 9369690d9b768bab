"""Golden vectors for the band route from the REFERENCE
package itself (blocktri.bands: BandMatrix, probing_build, band_as_blocktrid,
BandSolver, BandPreconditioner).  Same scratch build as make_golden.py.

    python tests/golden/make_band_golden.py

Inputs are regenerated from seeds by tests/golden/band_cases.py; only the
reference outputs are stored (tests/golden/band_golden.npz).
"""
from __future__ import annotations

import subprocess
import sys
import warnings

from make_golden import HERE, SCRATCH, build_reference


def child():
    import numpy as np

    sys.path.insert(0, str(SCRATCH / "src"))
    sys.path.insert(0, str(HERE))
    from band_cases import CASES, dense_band, rhs
    from blocktri import bands

    out = {}
    for name, n, d, m, seed, spd in CASES:
        a = dense_band(n, d, seed, spd)
        b = bands.BandMatrix.from_dense(a, d)
        out[f"{name}.bands"] = b.bands
        out[f"{name}.sym"] = b.symmetrized().bands
        mat, nn = bands.band_as_blocktrid(b, m)
        out[f"{name}.diag"], out[f"{name}.lower"], out[f"{name}.upper"] = mat.diag, mat.lower, mat.upper
        out[f"{name}.probe"] = bands.probing_build(lambda v: a @ v, d, n).bands
        r = rhs(n, seed)
        if spd:
            out[f"{name}.solve"] = bands.BandSolver(b.symmetrized()).solve(r)
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            pc = bands.BandPreconditioner(b)
        out[f"{name}.precond"] = pc.apply(r)
        out[f"{name}.fallback"] = np.array(pc.fallback)
    np.savez_compressed(HERE / "band_golden.npz", **out)
    print("cases", len(CASES))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
    else:
        build_reference()
        res = subprocess.run([sys.executable, __file__, "--child"], check=True, capture_output=True, text=True)
        print(res.stdout.strip())
