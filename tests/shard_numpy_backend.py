"""TEST INFRASTRUCTURE: numpy restatement of the native shard phases
(btd_plan_create_shard / btd_shard_finish / btd_shard_solve_a / _b) so the
ShardedPlan orchestration and its gloo collectives can run on CPU.

Same formulation as the CUDA path (paper_1108_4181_b200/csrc/btd_api.cu):
forward y_j = Dinv_j f + AD_j y_{j-1}, base_q = f_lo + sum Tb_j y_j,
carry_q = A_hi y_last; four reduced contributions per range; reduced system
solved densely here (the tree is covered by the GPU tests)."""
import types

import numpy as np
import torch

from paper_1108_4181_b200 import errors

RCOND = 1e-13


def _inv_checked(d, m):
    tol = RCOND * np.abs(d[:m, :m]).sum(axis=1).max()
    # same pivot test as the reference LU (first max, |pivot| <= tol)
    w = d.copy()
    for k in range(m):
        p = k + int(np.argmax(np.abs(w[k:, k])))
        if abs(w[p, k]) <= tol:
            return None
        w[[k, p]] = w[[p, k]]
        w[k + 1:] -= np.outer(w[k + 1:, k] / w[k, k], w[k])
    return np.linalg.inv(d)


class NumpyShardBackend:
    comm_device = "cpu"

    def create(self, diag, lower, upper, n, m, ranks, split, rank, world):
        h = types.SimpleNamespace()
        nr = min(n, ranks * split)
        if nr % world:
            return h, 7, -1, -1
        L = -(-n // nr)
        nrl = nr // world
        q0 = rank * nrl
        R0 = q0 * L
        nl = nrl * L
        nloc = max(0, min(nl, n - R0))
        C = np.tile(np.eye(m), (nl, 1, 1))
        Lw = np.zeros((nl, m, m))
        Uw = np.zeros((nl, m, m))
        c = max(0, min(nl, n - R0))
        C[:c] = diag[R0:R0 + c]
        c1 = max(0, min(nl, n - 1 - R0))
        Lw[:c1] = lower[R0:R0 + c1]
        Uw[:c1] = upper[R0:R0 + c1]
        h.__dict__.update(n=n, m=m, nr=nr, L=L, nrl=nrl, q0=q0, R0=R0, nl=nl, nloc=nloc, world=world)
        h.fac, h.contrib = [], np.zeros((nrl, 4, m, m))
        for ql in range(nrl):
            lo = ql * L
            F = dict(Dinv=[], AD=[], S=[], G=[], Tb=[])
            for j in range(L - 1):
                g = lo + 1 + j
                D = C[g] - (Lw[g - 1] @ F["S"][j - 1] if j else 0)
                Di = _inv_checked(D, m)
                if Di is None:
                    return h, 2, j, q0 + ql
                F["Dinv"].append(Di)
                F["S"].append(Di @ Uw[g])
                F["AD"].append(Di @ Lw[g - 1])
                F["G"].append(F["AD"][j] if j == 0 else F["AD"][j] @ F["G"][j - 1])
                F["Tb"].append(Uw[lo] if j == 0 else F["Tb"][j - 1] @ F["S"][j - 1])
            Fc = Lw[lo + L - 1]
            if L >= 2:
                BU = sum(F["Tb"][j] @ F["G"][j] for j in range(L - 1))
                h.contrib[ql] = [C[lo] - BU, Fc @ F["S"][-1], Fc @ F["G"][-1], F["Tb"][-1] @ F["S"][-1]]
            else:
                h.contrib[ql] = [C[lo], np.zeros((m, m)), Fc, Uw[lo]]
            F["Fc"] = Fc
            F["nint"] = max(0, min(L - 1, n - (q0 + ql) * L - 1))
            h.fac.append(F)
        return h, 0, -1, -1

    def info(self, h):
        return types.SimpleNamespace(row_lo=h.R0, row_hi=h.R0 + h.nloc, nranges=h.nr, L=h.L,
                                     range_lo=h.q0, range_hi=h.q0 + h.nrl)

    def contrib(self, h):
        return torch.from_numpy(h.contrib.reshape(-1).copy())

    def empty(self, nel):
        return torch.empty(nel, dtype=torch.float64)

    def finish(self, h, contrib_all):
        m, nr = h.m, h.nr
        c = contrib_all.numpy().reshape(nr, 4, m, m)
        R = np.zeros((nr * m, nr * m))
        for q in range(nr):
            R[q * m:(q + 1) * m, q * m:(q + 1) * m] = c[q, 0] - (c[q - 1, 1] if q else 0)
            if q:
                R[q * m:(q + 1) * m, (q - 1) * m:q * m] = -c[q - 1, 2]
            if q + 1 < nr:
                R[q * m:(q + 1) * m, (q + 1) * m:(q + 2) * m] = -c[q, 3]
        h.R = R
        return 0, -1

    def exchange_size(self, h, k):
        # carry block; "partials" = this rank's f~ slices embedded in a global array
        return h.m * k, h.nr * h.m * k

    def solve_a(self, h, f_local, x_local, k, carry):
        f, x = f_local.numpy(), x_local.numpy()
        h.base = np.zeros((h.nrl, h.m, k))
        h.carries = np.zeros((h.nrl, h.m, k))
        for ql, F in enumerate(h.fac):
            lo = ql * h.L
            base = f[lo].copy() if lo < h.nloc else np.zeros((h.m, k))
            y = None
            for j in range(F["nint"]):
                y = F["Dinv"][j] @ f[lo + 1 + j] + (F["AD"][j] @ y if j else 0)
                x[lo + 1 + j] = y
                base += F["Tb"][j] @ y
            h.base[ql] = base
            if F["nint"] == h.L - 1 and h.L >= 2 and h.q0 + ql + 1 < h.nr and (h.q0 + ql + 1) * h.L <= h.n:
                h.carries[ql] = F["Fc"] @ x[lo + h.L - 1]
        carry.copy_(torch.from_numpy(h.carries[-1].reshape(-1).copy()))

    def solve_b(self, h, carry_all, partial, k):
        ca = carry_all.numpy().reshape(h.world, h.m, k)
        ft = h.base.copy()
        ft[1:] += h.carries[:-1]
        if h.q0 > 0:
            ft[0] += ca[h.q0 // h.nrl - 1]
        glob = np.zeros((h.nr, h.m, k))
        glob[h.q0:h.q0 + h.nrl] = ft
        partial.copy_(torch.from_numpy(glob.reshape(-1)))

    def solve_c(self, h, partial_all, f_local, x_local, k):
        x = x_local.numpy()
        parts = partial_all.numpy().reshape(h.world, h.nr, h.m, k)
        ft = parts[0].copy()
        for r in range(1, h.world):
            ft += parts[r]
        xt = np.linalg.solve(h.R, ft.reshape(h.nr * h.m, k)).reshape(h.nr, h.m, k)
        xt = np.concatenate([xt, np.zeros((1, h.m, k))])
        for ql, F in enumerate(h.fac):
            q = h.q0 + ql
            lo = ql * h.L
            if lo < h.nloc:
                x[lo] = xt[q]
            nxt = xt[q + 1]
            for j in range(F["nint"] - 1, -1, -1):
                xj = x[lo + 1 + j] + F["G"][j] @ xt[q] + F["S"][j] @ nxt
                x[lo + 1 + j] = xj
                nxt = xj

    def destroy(self, h):
        pass
