"""Goldens for the generic Schur API from the REFERENCE
package itself: blocktri.schur SchurSystem / solve_schur / probing_preconditioner
on the systems of tests/golden/schur_cases.py.

    python tests/golden/make_schur_golden.py
"""
from __future__ import annotations

import json
import subprocess
import sys
import warnings

from make_golden import HERE, REPO


def child():
    import numpy as np

    sys.path.insert(0, str(REPO / "oracle" / "_ref"))
    sys.path.insert(0, str(HERE))
    from blocktri import core, schur
    from schur_cases import CASES, build

    arrays, meta = {}, {}
    for name, nx, heights, ranks, seed, symm in CASES:
        interiors, cpl, cplt, a_gamma, f = build(nx, heights, seed, symm)
        blocks = [schur.SubdomainBlock(i, schur.BlocktriOperator(core.BlockTriMatrix(*interiors[i]), ranks),
                                       cpl[i], cplt[i], symmetric=symm) for i in range(len(heights))]
        sys_ = schur.SchurSystem(blocks, a_gamma)
        x, st = schur.solve_schur(sys_, f, tol=1e-10)
        arrays[f"{name}.x"] = x
        arrays[f"{name}.rhs"] = schur.schur_rhs(sys_, f)
        arrays[f"{name}.S_e0"] = schur.schur_apply(sys_, np.eye(sys_.ngamma)[0])
        m = dict(iterations=st.iterations, relative_residual=st.relative_residual, converged=st.converged,
                 history=[float(h) for h in st.history])
        # probing preconditioner on every case; on the unsymmetric (PML-like) one it drives the
        # preconditioned scipy GMRES the reference uses there (schur.py:349-358)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            pc, band = schur.probing_preconditioner(sys_, 2, ranks=2)
        arrays[f"{name}.band"] = band.bands
        xp, stp = schur.solve_schur(sys_, f, tol=1e-10, precond=pc.apply)
        arrays[f"{name}.xp"] = xp
        m.update(precond_iterations=stp.iterations, precond_fallback=bool(pc.fallback),
                 precond_converged=bool(stp.converged), precond_relative_residual=stp.relative_residual,
                 precond_history=[float(h) for h in stp.history])
        meta[name] = m
    np.savez_compressed(HERE / "schur_golden.npz", **arrays)
    (HERE / "schur_golden.json").write_text(json.dumps(meta, indent=1))
    print(json.dumps(meta))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
    else:
        subprocess.run([str(REPO / "oracle" / "build_ref.sh")], check=True)
        res = subprocess.run([sys.executable, __file__, "--child"], check=True, capture_output=True, text=True)
        print(res.stdout.strip())
