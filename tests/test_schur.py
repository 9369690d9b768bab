"""Config-3 Schur-complement assembly (north-star subsystem 4), CPU checks."""
import numpy as np
import scipy.sparse.linalg as spl

import blocktri_oracle as O
from paper_1108_4181_b200 import schur


def _dense_schur(nx, nz, nsub):
    A = schur.grid_operator(nx, nz).toarray()
    z = schur.interface_rows(nz, nsub)
    G = np.concatenate([np.arange(s * nx, (s + 1) * nx) for s in z])
    I = np.setdiff1d(np.arange(nx * nz), G)
    return A[np.ix_(G, G)] - A[np.ix_(G, I)] @ np.linalg.solve(A[np.ix_(I, I)], A[np.ix_(I, G)])


def _assemble(d, lo, up):
    N, m = d.shape[0], d.shape[1]
    S = np.zeros((N * m, N * m))
    for s in range(N):
        S[s * m:(s + 1) * m, s * m:(s + 1) * m] = d[s]
        if s + 1 < N:
            S[s * m:(s + 1) * m, (s + 1) * m:(s + 2) * m] = -up[s]
            S[(s + 1) * m:(s + 2) * m, s * m:(s + 1) * m] = -lo[s]
    return S


def test_schur_blocks_equal_brute_force_schur_complement():
    for nx, nz, nsub in [(16, 64, 8), (12, 50, 5), (9, 33, 4)]:
        d, lo, up = schur.schur_blocks_numpy(nx, nz, nsub)
        Sd = _dense_schur(nx, nz, nsub)
        assert np.abs(_assemble(d, lo, up) - Sd).max() <= 1e-13 * np.abs(Sd).max()
        assert np.abs(Sd - Sd.T).max() <= 1e-13  # symmetric, as the DD theory says


def test_dd_interface_solve_matches_monolithic():
    nx, nz, nsub = 16, 96, 8
    d, lo, up = schur.schur_blocks_numpy(nx, nz, nsub)
    f = np.random.default_rng(0).standard_normal((nx * nz, 3))
    x = spl.spsolve(schur.grid_operator(nx, nz).tocsc(), f)
    fg = schur.interface_rhs_from_grid(f, nx, nz, nsub)
    xs = O.plan_solve(O.plan_build(d, lo, up, 3), fg)
    z = schur.interface_rows(nz, nsub)
    assert np.abs(xs - x.reshape(nz, nx, -1)[z]).max() <= 1e-12 * np.abs(x).max()


def test_config3_layout():
    z = schur.interface_rows(8192, 64)
    assert len(z) == 63 and z[0] == 128 and z[-1] == 8064
    gaps = np.diff(np.concatenate([[-1], z, [8192]])) - 1
    assert set(gaps.tolist()) == {127, 128}
    c = schur.layered_velocity(8192, 16, 0)
    assert c.min() >= 1500 and c.max() <= 4500 and len(np.unique(c)) == 16
