"""Row f1, generic Schur API on the GPU, against the reference's own
solve_schur / schur_rhs / schur_apply / probing_preconditioner outputs
(tests/golden/schur_golden.*, written by tests/golden/make_schur_golden.py)."""
import json
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from schur_cases import CASES, build  # noqa: E402

from paper_1108_4181_b200 import BlockTriMatrix, schur  # noqa: E402

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(__file__), "golden")
G = np.load(os.path.join(HERE, "schur_golden.npz"))
META = json.load(open(os.path.join(HERE, "schur_golden.json")))


def _system(name):
    _n, nx, heights, ranks, seed, symm = next(c for c in CASES if c[0] == name)
    interiors, cpl, cplt, a_gamma, f = build(nx, heights, seed, symm)
    blocks = [schur.SubdomainBlock(i, schur.BlocktriOperator(BlockTriMatrix(*interiors[i]), ranks), cpl[i], cplt[i],
                                   symmetric=symm) for i in range(len(heights))]
    return schur.SchurSystem(blocks, a_gamma), f


def _rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("name", [c[0] for c in CASES])
def test_schur_pieces_match_reference(name):
    sys_, f = _system(name)
    assert _rel(schur.schur_rhs(sys_, f), G[f"{name}.rhs"]) <= 1e-12
    assert _rel(schur.schur_apply(sys_, np.eye(sys_.ngamma)[0]), G[f"{name}.S_e0"]) <= 1e-12


@pytest.mark.parametrize("name", [c[0] for c in CASES])
def test_solve_schur_matches_reference(name):
    import torch

    sys_, f = _system(name)
    x, st = schur.solve_schur(sys_, f, tol=1e-10)
    assert st.converged and abs(st.iterations - META[name]["iterations"]) <= 1
    assert _rel(x, G[f"{name}.x"]) <= 1e-8
    # residual of the full saddle system (device apply_full)
    assert np.abs(sys_.apply_full(x) - f).max() / np.abs(f).max() <= 1e-8
    xt, _ = schur.solve_schur(sys_, torch.from_numpy(f).cuda(), tol=1e-10)  # device in -> device out
    assert xt.is_cuda and _rel(xt.cpu().numpy(), x) <= 1e-12


@pytest.mark.parametrize("name", [c[0] for c in CASES])
def test_probing_preconditioner_matches_reference(name):
    """Symmetric cases: preconditioned CG; the unsymmetric case: the preconditioned
    restarted GMRES with scipy's stopping semantics (true residual <= tol ||b||,
    ref schur.py:349-358) -- same convergence flag, iterations and pr_norm history."""
    sys_, f = _system(name)
    meta = META[name]
    pc, band = schur.probing_preconditioner(sys_, 2, ranks=2)
    assert pc.fallback == meta["precond_fallback"] and band.symmetric
    assert np.abs(band.bands - G[f"{name}.band"]).max() <= 1e-12 * np.abs(G[f"{name}.band"]).max()
    xp, stp = schur.solve_schur(sys_, f, tol=1e-10, precond=pc)
    assert stp.converged == meta["precond_converged"] and abs(stp.iterations - meta["precond_iterations"]) <= 1
    assert _rel(xp, G[f"{name}.xp"]) <= 1e-8
    assert stp.relative_residual <= 1e-10
    h, hr = np.asarray(stp.history), np.asarray(meta["precond_history"])
    n = min(len(h), len(hr))
    assert np.allclose(h[:n], hr[:n], rtol=1e-5, atol=1e-13)


def test_blocktri_operator_apply_and_unpadded():
    from paper_1108_4181_b200 import configs

    d, lo, up, _ = configs.dominant_numpy(9, 5, 1, seed=4)
    op = schur.BlocktriOperator(BlockTriMatrix(d, lo, up), ranks=3, unpadded=43)
    x = np.random.default_rng(0).standard_normal(43)
    full = np.zeros(45)
    full[:43] = x
    y_ref = BlockTriMatrix(d, lo, up).apply(full.reshape(9, 5)).reshape(-1)[:43]
    assert np.abs(op.apply(x) - y_ref).max() <= 1e-13
    X = np.random.default_rng(1).standard_normal((43, 3))
    sol = op.solve(X)
    assert sol.shape == (43, 3)


def test_cg_breakdown_and_zero_rhs():
    import torch

    from paper_1108_4181_b200 import errors

    x, st = schur.cg_solve(lambda v: v, np.zeros(5))
    assert st.iterations == 0 and st.converged and not np.any(x)
    with pytest.raises(errors.Breakdown):
        schur.cg_solve(lambda v: -v, torch.ones(4, dtype=torch.float64, device="cuda"))
