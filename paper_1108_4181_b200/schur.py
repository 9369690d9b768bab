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


class HelmholtzDD:
    """Full Schur-complement DD solve of the config-3 operator on the GPU
    (ref schur.py:322-372 solve_schur = schur_rhs ->
    solve_interface -> recover_interiors).

    * Interiors: subdomain i (z rows a_i..b_i-1) in the reference's
      block-per-x-column orientation (acoustic.py:231-243): nx block rows of
      order n_i <= Mi with C = tridiag(-1, 4 + s_z, -1) over z and A = B = I.
      ``groups`` plans each stack nsub/groups subdomains (zero couplings between
      them; shorter subdomains padded to order Mi by a decoupled tridiag(-1, 4, -1)
      chain with zero right-hand sides, so every coupling block stays I -- a
      scalar-coupled plan, two-product forward sweep) -- every A_ii^{-1} of a
      group is ONE dichotomy solve.
    * Interface: the explicit S (schur_blocks_torch) solved by its own plan.
    * solve(f): f (nz, nx, K) on the device -> x (nz, nx, K).
    """

    def __init__(self, nx, nz, nsub, *, h=5.0, sigma=50.0, layers=16, seed=0, groups=1, ranks_int=None,
                 split_int=1, ranks_s=None, device="cuda"):
        import torch

        from .dichotomy import plan_build_arrays

        self.torch = torch
        self.nx, self.nz, self.nsub, self.groups = nx, nz, nsub, groups
        if nsub % groups:
            raise ValueError("nsub must be a multiple of groups")
        self.device = device
        self.sh = torch.from_numpy(shifts(nz, h, sigma, layers, seed)).to(device)
        self.z_if = interface_rows(nz, nsub)
        b = np.concatenate([[-1], self.z_if, [nz]])
        self.sub = [(int(b[i] + 1), int(b[i + 1])) for i in range(nsub)]
        self.Mi = max(e - a for a, e in self.sub)
        Mi = self.Mi
        per = nsub // groups
        self.plans = []
        for gidx in range(groups):
            subs = self.sub[gidx * per:(gidx + 1) * per]
            n = per * nx
            diag = torch.zeros((per, Mi, Mi), dtype=torch.float64, device=device)
            eye = torch.zeros((per, Mi, Mi), dtype=torch.float64, device=device)
            for j, (a, e) in enumerate(subs):
                ni = e - a
                d = torch.diag(4.0 + self.sh[a:e]) - torch.diag(torch.ones(ni - 1, dtype=torch.float64,
                                                                             device=device), 1) \
                    - torch.diag(torch.ones(ni - 1, dtype=torch.float64, device=device), -1)
                diag[j, :ni, :ni] = d
                diag[j, ni:, ni:] = 4.0 * torch.eye(Mi - ni, dtype=torch.float64, device=device)
                eye[j] = torch.eye(Mi, dtype=torch.float64, device=device)
            D = diag.repeat_interleave(nx, dim=0).contiguous()
            cpl = eye.repeat_interleave(nx, dim=0)[: n - 1].clone()
            cpl[nx - 1::nx] = 0.0  # no coupling across subdomain boundaries
            P = ranks_int or max(1, min(n, 9 * per))
            self.plans.append(plan_build_arrays(D, cpl, cpl, P, split=split_int, device=device))
            del D, cpl
        d, lo, up = schur_blocks_torch(nx, nz, nsub, device=device, h=h, sigma=sigma, layers=layers, seed=seed)
        self.plan_s = plan_build_arrays(d, lo, up, ranks_s or min(9, nsub - 1), device=device)
        del d, lo, up
        torch.cuda.empty_cache()

    def _stack(self, f, gidx):
        """grid rows of the group's subdomains -> (per*nx, Mi, K) interior blocks."""
        torch = self.torch
        per = self.nsub // self.groups
        K = f.shape[2]
        out = torch.empty((per * self.nx, self.Mi, K), dtype=torch.float64, device=f.device)
        for j, (a, e) in enumerate(self.sub[gidx * per:(gidx + 1) * per]):
            out[j * self.nx:(j + 1) * self.nx, : e - a] = f[a:e].permute(1, 0, 2)
            if e - a < self.Mi:  # padding rows of shorter subdomains: zero right-hand side (no full zero fill)
                out[j * self.nx:(j + 1) * self.nx, e - a:] = 0.0
        return out

    def solve(self, f):
        """x = A^{-1} f by Schur-complement DD (f, x: (nz, nx, K) CUDA tensors)."""
        from .dichotomy import plan_solve

        torch = self.torch
        nx, per = self.nx, self.nsub // self.groups
        K = f.shape[2]
        # 1. interior solves g_i = A_ii^{-1} f_i   (ref schur.py:322-328)
        fg = f[torch.as_tensor(self.z_if, device=f.device)].clone()  # (N, nx, K) interface RHS
        stacked = [self._stack(f, gidx) for gidx in range(self.groups)]
        for gidx in range(self.groups):
            g = plan_solve(self.plans[gidx], stacked[gidx])
            for j in range(per):
                i = gidx * per + j
                a, e = self.sub[i]
                gi = g[j * nx:(j + 1) * nx]  # (nx, Mi, K)
                if i >= 1:              # interface above: -A_G,i A_ii^{-1} f_i = + first row
                    fg[i - 1] += gi[:, 0]
                if i < self.nsub - 1:   # interface below: + last interior row
                    fg[i] += gi[:, e - a - 1]
            del g
        # 2. interface solve S x_G = f~_G (the dichotomy S-solve)
        xg = plan_solve(self.plan_s, fg.contiguous())
        # 3. recovery x_i = A_ii^{-1} (f_i - A_iG x_G)   (ref schur.py:331-335)
        x = torch.empty_like(f)
        x[torch.as_tensor(self.z_if, device=f.device)] = xg
        for gidx in range(self.groups):
            h_ = stacked[gidx]
            for j in range(per):
                i = gidx * per + j
                a, e = self.sub[i]
                if i >= 1:
                    h_[j * nx:(j + 1) * nx, 0] += xg[i - 1]
                if i < self.nsub - 1:
                    h_[j * nx:(j + 1) * nx, e - a - 1] += xg[i]
            xi = plan_solve(self.plans[gidx], h_)
            for j in range(per):
                a, e = self.sub[gidx * per + j]
                x[a:e] = xi[j * nx:(j + 1) * nx, : e - a].permute(1, 0, 2)
        return x

    def residual(self, x, f):
        """max|A x - f| / max|f| on the grid (5-point operator)."""
        r = (4.0 + self.sh)[:, None, None] * x - f
        r[1:] -= x[:-1]
        r[:-1] -= x[1:]
        r[:, 1:] -= x[:, :-1]
        r[:, :-1] -= x[:, 1:]
        return float(r.abs().max() / f.abs().max())


# The reference's generic matrix-free Schur API (ref schur.py:29-378), device-resident.
from .schur_system import (INTERFACE_LABEL, BlocktriOperator, CgStats, SchurSystem, SubdomainBlock,  # noqa: E402
                           cg_solve, gmres_solve, partition_numbering, probing_preconditioner,
                           recover_interiors, schur_apply, schur_rhs, solve_interface, solve_schur)
