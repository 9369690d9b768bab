"""Schur-complement domain decomposition of config 3 (north-star subsystem 4).

Operator: the 5-point finite-difference -Delta u + (sigma/c^2) u on an
nx (x) by nz (z) grid with Dirichlet edges, scaled by h^2; block row z of
the natural ordering is ``C_z = tridiag(-1, 4 + sigma h^2 / c_z^2, -1)``
(M = nx), couplings ``A = B = I`` -- the reference's ``_blocktri_strip``
layout (models.py:48-57) with a z-dependent shift.  The grid is split in z by
``nsub - 1`` interface rows into ``nsub`` subdomains; the interface Schur
complement (Eq. 14, ref schur.py:313-319 ``schur_apply``)

    S = A_GG - sum_i A_iG^T A_ii^{-1} A_iG

is block tridiagonal over the interface rows: subdomain i touches only the
interface rows above and below it, through -I couplings, so it contributes
the four corner blocks of A_ii^{-1}.  All blocks of a subdomain share the
DST-I eigenbasis Q of T2 = tridiag(-1, 2, -1) (C_z = (2 + s_z) I + T2), so

    S.diag[s]  = Q diag(2 + s_{z_s} + lam_k - g_last^(s)(k) - g_first^(s+1)(k)) Q
    S.upper[s] = S.lower[s] = Q diag(g_corner^(s+1)(k)) Q

with g the corner entries of the inverse of the scalar tridiagonal chain of
mode k in each subdomain (continued-fraction sweeps, vectorised over modes
and subdomains).  This is the reference's separable route
(separable.py:50-229) for forming S; solving S x = f
(K right-hand sides) is the dichotomy path itself (plan_build/plan_solve).

Full-size config 3: nx = 2048, nz = 8192, h = 5 m, sigma = 50 1/s, 16
horizontal layers with c ~ U(1500, 4500) m/s (seeded), 64 subdomains
-> S has N = 63 block rows of M = 2048.  Interface rows sit at
z_s = round(s * nz / nsub) (8192/64: every 128th row), leaving 127 or 128
interior rows per subdomain.
"""

from __future__ import annotations

import math

import numpy as np


def layered_velocity(nz, layers=16, seed=0, lo=1500.0, hi=4500.0):
    """c(z): `layers` equal horizontal layers with seeded U(lo, hi) velocities."""
    rng = np.random.default_rng(seed)
    cl = rng.uniform(lo, hi, size=layers)
    idx = np.minimum((np.arange(nz) * layers) // nz, layers - 1)
    return cl[idx]


def shifts(nz, h=5.0, sigma=50.0, layers=16, seed=0):
    """sigma h^2 / c(z)^2 per grid row z."""
    c = layered_velocity(nz, layers, seed)
    return sigma * h * h / (c * c)


def interface_rows(nz, nsub):
    return np.array([int(round(s * nz / nsub)) for s in range(1, nsub)], dtype=np.int64)


def dst_basis(m, xp=np):
    """Orthonormal DST-I matrix Q (symmetric, Q Q = I) and eigenvalues of T2."""
    k = xp.arange(1, m + 1, dtype=xp.float64)
    Q = math.sqrt(2.0 / (m + 1)) * xp.sin(xp.outer(k, k) * math.pi / (m + 1))
    lam = 2.0 - 2.0 * xp.cos(k * math.pi / (m + 1))
    return Q, lam


def _corner_entries(diag_modes, xp=np):
    """Corners of the inverse of tridiag(-1, d_j, -1), j = 0..n-1, per mode.

    diag_modes: (n, M).  Returns (g_first, g_last, g_corner) = (T^{-1})_{00},
    (T^{-1})_{n-1,n-1}, (T^{-1})_{0,n-1}, each (M,), via continued fractions
    r_j = d_j - 1/r_{j-1} (forward) and s_j = d_j - 1/s_{j+1} (backward);
    (T^{-1})_{0,n-1} = prod_j 1/r_j (off-diagonals -1 make all signs +)."""
    n = diag_modes.shape[0]
    r = diag_modes[0].copy()
    logc = -xp.log(r)
    for j in range(1, n):
        r = diag_modes[j] - 1.0 / r
        logc = logc - xp.log(r)
    g_last = 1.0 / r
    s = diag_modes[n - 1].copy()
    for j in range(n - 2, -1, -1):
        s = diag_modes[j] - 1.0 / s
    g_first = 1.0 / s
    return g_first, g_last, xp.exp(logc)


def schur_spectra(nx, nz, nsub, h=5.0, sigma=50.0, layers=16, seed=0, xp=np):
    """Per-mode diagonals of the S blocks: returns (Q, dS (N, M), uS (N-1, M), shift)."""
    sh = shifts(nz, h, sigma, layers, seed)
    z_if = interface_rows(nz, nsub)
    Q, lam = dst_basis(nx, xp)
    sh_x = xp.asarray(sh)
    bounds = np.concatenate([[-1], z_if, [nz]])
    gf, gl, gc = [], [], []
    for i in range(nsub):
        a, b = bounds[i] + 1, bounds[i + 1]  # interior rows a..b-1 of subdomain i
        dm = (2.0 + sh_x[a:b])[:, None] + lam[None, :]
        f_, l_, c_ = _corner_entries(dm, xp)
        gf.append(f_)
        gl.append(l_)
        gc.append(c_)
    N = nsub - 1
    dS = xp.stack([2.0 + sh_x[z_if[s]] + lam - gl[s] - gf[s + 1] for s in range(N)])
    uS = xp.stack([gc[s + 1] for s in range(N - 1)]) if N > 1 else xp.zeros((0, nx))
    return Q, dS, uS, sh


def schur_blocks_numpy(nx, nz, nsub, **kw):
    """Explicit S = (diag, lower, upper) as numpy arrays (small grids / tests)."""
    Q, dS, uS, _ = schur_spectra(nx, nz, nsub, **kw)
    diag = np.stack([(Q * d[None, :]) @ Q for d in dS])
    up = np.stack([(Q * u[None, :]) @ Q for u in uS]) if len(uS) else np.zeros((0, nx, nx))
    return diag, up.copy(), up


def schur_blocks_torch(nx, nz, nsub, device="cuda", **kw):
    """Explicit S on the GPU: spectra in fp64, then Q diag Q per block (3 GEMMs of
    M^3 per block row; preprocessing, timed separately from the S solve)."""
    import torch

    Q, dS, uS, _ = schur_spectra(nx, nz, nsub, **kw)
    Qt = torch.from_numpy(Q).to(device)
    dSt = torch.from_numpy(np.ascontiguousarray(dS)).to(device)
    uSt = torch.from_numpy(np.ascontiguousarray(uS)).to(device)
    diag = torch.empty((nsub - 1, nx, nx), dtype=torch.float64, device=device)
    up = torch.empty((max(nsub - 2, 0), nx, nx), dtype=torch.float64, device=device)
    for s in range(nsub - 1):
        torch.matmul(Qt * dSt[s][None, :], Qt, out=diag[s])
    for s in range(nsub - 2):
        torch.matmul(Qt * uSt[s][None, :], Qt, out=up[s])
    return diag, up, up  # S is symmetric: lower[s] = upper[s]^T = upper[s]


def grid_operator(nx, nz, h=5.0, sigma=50.0, layers=16, seed=0):
    """Monolithic sparse operator in natural (z-major) ordering, for oracle checks."""
    import scipy.sparse as sp

    sh = shifts(nz, h, sigma, layers, seed)
    tx = sp.diags([-np.ones(nx - 1), np.zeros(nx), -np.ones(nx - 1)], [-1, 0, 1])
    tz = sp.diags([-np.ones(nz - 1), np.zeros(nz), -np.ones(nz - 1)], [-1, 0, 1])
    main = sp.kron(sp.diags(4.0 + sh), sp.identity(nx))
    return (main + sp.kron(sp.identity(nz), tx) + sp.kron(tz, sp.identity(nx))).tocsr()


def interface_rhs_from_grid(fgrid, nx, nz, nsub, **kw):
    """Condensed interface RHS f_G - sum A_iG^T A_ii^{-1} f_i (ref schur.py:322-328),
    by dense sparse-LU per subdomain -- test-scale helper (small grids only)."""
    import scipy.sparse.linalg as spl

    A = grid_operator(nx, nz, **kw)
    z_if = interface_rows(nz, nsub)
    bounds = np.concatenate([[-1], z_if, [nz]])
    fg = fgrid.reshape(nz, nx, -1)
    out = fg[z_if].copy()
    for i in range(nsub):
        a, b = bounds[i] + 1, bounds[i + 1]
        rows = np.arange(a * nx, b * nx)
        Aii = A[rows][:, rows].tocsc()
        w = spl.splu(Aii).solve(fg[a:b].reshape((b - a) * nx, -1))
        w = w.reshape(b - a, nx, -1)
        if i >= 1:  # interface above: A_iG = -I at the first row -> out[s-1] += w[first]
            out[i - 1] += w[0]
        if i < nsub - 1:
            out[i] += w[-1]
    return out
