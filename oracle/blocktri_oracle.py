"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain-numpy restatement of the reference's many-RHS dichotomy path
(``/root/reference/pkg/src/blocktri``), used by ``tests/``, by
``__graft_entry__.smoke()`` and by ``bench.py``'s CPU-baseline leg as the
*checker*.  The product path (``paper_1108_4181_b200``) never imports this
module; it fails loudly when its CUDA library is missing instead.

Parity pin: every function here is checked against golden vectors produced by
running the reference package itself (``tests/golden/make_golden.py``,
fixtures ``tests/golden/*.npz``) in ``tests/test_oracle_golden.py``.

Conventions (ref ``core.py:1-10``): row i of the operator reads
``-lower[i-1] x_{i-1} + diag[i] x_i - upper[i] x_{i+1} = f_i``; interfaces sit
at ``K_q = q*L`` with ``L = ceil(N/P)`` and the closure ``x_N = 0``
(ref ``dichotomy.py:11, 318-338``).
"""

from __future__ import annotations

import numpy as np

from paper_1108_4181_b200 import errors as _err

RCOND = 1e-13  # ref _kernels_py.py:14 / _kernels.pyx:17


# --------------------------------------------------------------------------
# Block kernels (ref _kernels_py.py:19-105, _kernels.pyx:35-194)
# --------------------------------------------------------------------------

def lu_factor(block):
    """Partial-pivot LU, LAPACK-style swap list; the pivot test is
    ``|pivot| <= RCOND * ||block||_inf`` (ref _kernels_py.py:19-44)."""
    work = np.array(block, dtype=np.float64, order="C", copy=True)
    m = work.shape[0]
    swaps = np.zeros(m, dtype=np.int64)
    tol = RCOND * (np.abs(work).sum(axis=1).max() if m else 0.0)
    for col in range(m):
        cand = np.abs(work[col:, col])
        p = col + int(np.argmax(cand))
        if abs(work[p, col]) <= tol:
            raise _err.SingularBlock(f"column {col}: pivot {abs(work[p, col]):.3e} <= {tol:.3e}")
        swaps[col] = p
        if p != col:
            work[[col, p]] = work[[p, col]]
        if col + 1 < m:
            work[col + 1:, col] /= work[col, col]
            work[col + 1:, col + 1:] -= np.outer(work[col + 1:, col], work[col, col + 1:])
    return work, swaps


def lu_solve(lu, swaps, rhs):
    """Apply the swap list, unit-lower forward and upper backward
    substitution (ref _kernels_py.py:47-58)."""
    x = np.array(rhs, dtype=np.float64, copy=True)
    m = lu.shape[0]
    for col in range(m):
        if swaps[col] != col:
            x[[col, swaps[col]]] = x[[swaps[col], col]]
    for r in range(1, m):
        x[r] -= lu[r, :r] @ x[:r]
    for r in range(m - 1, -1, -1):
        if r + 1 < m:
            x[r] -= lu[r, r + 1:] @ x[r + 1:]
        x[r] /= lu[r, r]
    return x


def thomas_factor(diag, lower, upper):
    """Block forward elimination D_0 = C_0, D_i = C_i - A_i S_{i-1},
    S_i = D_i^{-1} B_i; SingularPivot carries the local row
    (ref _kernels_py.py:61-88)."""
    n, m = diag.shape[0], diag.shape[1]
    dlu = np.empty((n, m, m))
    dpiv = np.empty((n, m), dtype=np.int64)
    supper = np.empty((max(n - 1, 0), m, m))
    pivot_block = diag[0]
    for i in range(n):
        try:
            dlu[i], dpiv[i] = lu_factor(pivot_block)
        except _err.SingularBlock as exc:
            raise _err.SingularPivot(i, f"block row {i}: {exc}") from exc
        if i + 1 < n:
            supper[i] = lu_solve(dlu[i], dpiv[i], upper[i])
            pivot_block = diag[i + 1] - lower[i] @ supper[i]
    return dlu, dpiv, supper


def thomas_solve(dlu, dpiv, supper, lower, f):
    """Forward x_i = D_i^{-1}(f_i + A_i x_{i-1}), backward x_i += S_i x_{i+1}
    (ref _kernels_py.py:91-105)."""
    f = np.asarray(f, dtype=np.float64)
    n = dlu.shape[0]
    x = np.empty_like(f)
    x[0] = lu_solve(dlu[0], dpiv[0], f[0])
    for i in range(1, n):
        x[i] = lu_solve(dlu[i], dpiv[i], f[i] + lower[i - 1] @ x[i - 1])
    for i in range(n - 2, -1, -1):
        x[i] += supper[i] @ x[i + 1]
    return x


# --------------------------------------------------------------------------
# Dichotomy (Algorithm 1 + 2), ref dichotomy.py:28-390
# --------------------------------------------------------------------------

def partition_tree(count):
    """BFS list of (lo, hi, k, level) with split k = lo + (hi-lo+1)//2
    (ref dichotomy.py:28-57)."""
    if count < 1:
        raise _err.InvalidRankCount(f"partition tree needs count >= 1, got {count}")
    out, frontier, level = [], [(0, count - 1)], 0
    while frontier:
        nxt = []
        for lo, hi in frontier:
            k = lo + (hi - lo + 1) // 2
            out.append((lo, hi, k, level))
            if k > lo:
                nxt.append((lo, k - 1))
            if k < hi:
                nxt.append((k + 1, hi))
        frontier, level = nxt, level + 1
    return out


def tree_depth(count):
    return (count - 1).bit_length()


class OraclePlan:
    """Everything Algorithm 2 step 1 produces (ref dichotomy.py:99-131)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


def _padded(diag, lower, upper, npad):
    """Identity rows with zero couplings up to npad (ref dichotomy.py:307-315)."""
    n, m = diag.shape[0], diag.shape[1]
    if npad == n:
        return diag, lower, upper
    extra = npad - n
    d = np.concatenate([diag, np.broadcast_to(np.eye(m), (extra, m, m))])
    z = np.zeros((extra, m, m))
    return d, np.concatenate([lower, z]), np.concatenate([upper, z])


def _range_factors(d, lo_, up_, lo, hi):
    """U, V, interior Thomas factors of range [lo, hi] (ref dichotomy.py:172-193)."""
    m = d.shape[1]
    L = hi - lo
    U = np.zeros((L + 1, m, m))
    V = np.zeros((L + 1, m, m))
    U[0] = np.eye(m)
    V[L] = np.eye(m)
    fact = None
    if L >= 2:
        # interior rows lo+1 .. hi-1 (submatrix, ref core.py:129-135)
        sd, sl, su = d[lo + 1:hi], lo_[lo + 1:hi - 1], up_[lo + 1:hi - 1]
        fact = thomas_factor(sd, sl, su) + (sl,)
        e0 = np.zeros((L - 1, m, m))
        e0[0] = lo_[lo]
        U[1:L] = thomas_solve(fact[0], fact[1], fact[2], sl, e0)
        eL = np.zeros((L - 1, m, m))
        if hi - 1 < d.shape[0] - 1:
            eL[L - 2] = up_[hi - 1]
        V[1:L] = thomas_solve(fact[0], fact[1], fact[2], sl, eL)
    return U, V, fact


def _reduced_blocks(d, lo_, up_, L, P, Us, Vs):
    """Eq. 7 three-point interface system (ref dichotomy.py:212-236)."""
    m = d.shape[1]
    npad = d.shape[0]
    rd = np.empty((P, m, m))
    rl = np.empty((max(P - 1, 0), m, m))
    ru = np.empty((max(P - 1, 0), m, m))
    for q in range(P):
        K = q * L
        blk = d[K].copy()
        if q >= 1:
            blk -= lo_[K - 1] @ Vs[q - 1][L - 1]
            rl[q - 1] = lo_[K - 1] @ Us[q - 1][L - 1]
        if K < npad - 1:
            blk -= up_[K] @ Us[q][1]
            if q <= P - 2:
                ru[q] = up_[K] @ Vs[q][1]
        rd[q] = blk
    return rd, rl, ru


def _inverse_rows(rd, rl, ru, lo, hi, k):
    """Block row (k-lo) of (R[lo..hi])^{-1} by transposed sweeps with unit RHS
    (ref dichotomy.py:134-146)."""
    m = rd.shape[1]
    sd = rd[lo:hi + 1].transpose(0, 2, 1)
    sl = ru[lo:hi].transpose(0, 2, 1)  # transpose swaps the couplings (ref core.py:137-143)
    su = rl[lo:hi].transpose(0, 2, 1)
    dlu, dpiv, sup = thomas_factor(np.ascontiguousarray(sd), np.ascontiguousarray(sl),
                                   np.ascontiguousarray(su))
    rhs = np.zeros((hi - lo + 1, m, m))
    rhs[k - lo] = np.eye(m)
    y = thomas_solve(dlu, dpiv, sup, np.ascontiguousarray(sl), rhs)
    return np.ascontiguousarray(y.transpose(2, 0, 1).reshape(m, (hi - lo + 1) * m))


def plan_build(diag, lower, upper, ranks):
    """Algorithm 2 step 1 (ref dichotomy.py:318-338)."""
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    n, m = diag.shape[0], diag.shape[1]
    lower = np.ascontiguousarray(lower, dtype=np.float64).reshape(max(n - 1, 0), m, m)
    upper = np.ascontiguousarray(upper, dtype=np.float64).reshape(max(n - 1, 0), m, m)
    if ranks < 1 or ranks > n:
        raise _err.InvalidRankCount(f"ranks={ranks} outside [1, N={n}]")
    L = -(-n // ranks)
    npad = L * ranks
    d, lo_, up_ = _padded(diag, lower, upper, npad)
    Us, Vs, facts = [], [], []
    for q in range(ranks):
        U, V, f = _range_factors(d, lo_, up_, q * L, (q + 1) * L)
        Us.append(U)
        Vs.append(V)
        facts.append(f)
    rd, rl, ru = _reduced_blocks(d, lo_, up_, L, ranks, Us, Vs)
    tree = partition_tree(ranks)
    inv_rows = [_inverse_rows(rd, rl, ru, lo, hi, k) for (lo, hi, k, _lvl) in tree]
    return OraclePlan(n=n, m=m, ranks=ranks, L=L, npad=npad, diag=d, lower=lo_, upper=up_,
                      U=Us, V=Vs, facts=facts, rdiag=rd, rlower=rl, rupper=ru,
                      tree=tree, inverse_rows=inv_rows)


def _reduced_solve(plan, ftilde):
    """Algorithm 1 on the interface system (ref dichotomy.py:279-295)."""
    fmod = np.array(ftilde, copy=True)
    xt = np.empty_like(fmod)
    for (lo, hi, k, _lvl), rows in zip(plan.tree, plan.inverse_rows):
        seg = fmod[lo:hi + 1].reshape((hi - lo + 1) * plan.m, -1)
        xt[k] = (rows @ seg).reshape(fmod.shape[1:])
        if k - 1 >= lo:
            fmod[k - 1] += plan.rupper[k - 1] @ xt[k]
        if k + 1 <= hi:
            fmod[k + 1] += plan.rlower[k] @ xt[k]
    return xt


def plan_solve(plan, f):
    """Algorithm 2 step 2 for (n,m) or (n,m,k) right-hand sides
    (ref dichotomy.py:358-390): particular solutions W per range,
    interface RHS (ref 239-276), reduced solve, superposition recovery
    (ref 345-355)."""
    f = np.asarray(f, dtype=np.float64)
    if f.shape[0] != plan.n or f.shape[1] != plan.m:
        raise _err.DimensionMismatch(f"rhs layout {f.shape[:2]} does not match plan ({plan.n}, {plan.m})")
    squeeze = f.ndim == 2
    fk = f[:, :, None] if squeeze else f
    L, P = plan.L, plan.ranks
    fp = np.zeros((plan.npad,) + fk.shape[1:])
    fp[:plan.n] = fk
    Ws = []
    for q in range(P):
        w = np.zeros((L + 1,) + fk.shape[1:])
        if L >= 2:
            dlu, dpiv, sup, sl = plan.facts[q]
            w[1:L] = thomas_solve(dlu, dpiv, sup, sl, fp[q * L + 1:(q + 1) * L])
        Ws.append(w)
    ft = np.empty((P,) + fk.shape[1:])
    for q in range(P):
        K = q * L
        ft[q] = fp[K]
        if K < plan.npad - 1:
            ft[q] += plan.upper[K] @ Ws[q][1]
        if q >= 1:
            ft[q] += plan.lower[K - 1] @ Ws[q - 1][L - 1]
    xt = _reduced_solve(plan, ft)
    x = np.empty_like(fp)
    for q in range(P):
        K = q * L
        x[K] = xt[q]
        if L >= 2:
            nxt = xt[q + 1] if q + 1 < P else np.zeros_like(xt[0])
            x[K + 1:K + L] = (np.einsum("lij,jc->lic", plan.U[q][1:L], xt[q])
                              + np.einsum("lij,jc->lic", plan.V[q][1:L], nxt) + Ws[q][1:L])
    x = np.ascontiguousarray(x[:plan.n])
    return x[:, :, 0] if squeeze else x


# --------------------------------------------------------------------------
# Parity metrics (ref test_core.py:154,208; cli.py:211-214)
# --------------------------------------------------------------------------

def apply(diag, lower, upper, x):
    """y = C x - A x_{i-1} - B x_{i+1} (ref core.py:118-127)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.einsum("nij,nj...->ni...", diag, x)
    if diag.shape[0] > 1:
        y[1:] -= np.einsum("nij,nj...->ni...", lower, x[:-1])
        y[:-1] -= np.einsum("nij,nj...->ni...", upper, x[1:])
    return y


def max_rel_err(x, ref):
    den = np.abs(ref).max()
    return float(np.abs(np.asarray(x) - ref).max() / (den if den > 0 else 1.0))


def rel_residual(diag, lower, upper, x, f):
    den = np.abs(f).max()
    return float(np.abs(apply(diag, lower, upper, x) - f).max() / (den if den > 0 else 1.0))
