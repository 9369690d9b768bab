"""Seeded Schur-DD systems for the generic Schur API goldens (shared by
make_schur_golden.py and the tests): a 5-point grid operator split in z into
subdomains by single interface rows; interiors are block tridiagonal over z
(blocks of order nx: C = tridiag(-1, 4 + s_z, -1), A = B = I)."""
import numpy as np
import scipy.sparse as sp

# (name, nx, heights, ranks, seed, symmetric)
CASES = [
    ("sym3", 16, (6, 7, 5), 2, 1, True),
    ("sym4", 12, (5, 5, 6, 4), 2, 2, True),
    ("unsym3", 10, (4, 6, 5), 2, 3, False),
]


def build(nx, heights, seed, symmetric):
    rng = np.random.default_rng(seed)
    nsub = len(heights)
    nz = sum(heights) + nsub - 1
    shift = rng.uniform(0.05, 0.5, nz)
    T = lambda s: (np.diag(np.full(nx, 4.0 + s)) - np.eye(nx, k=1) - np.eye(nx, k=-1))  # noqa: E731
    interiors, couplings, z = [], [], 0
    ngamma = (nsub - 1) * nx
    for i, h in enumerate(heights):
        diag = np.stack([T(shift[z + j]) for j in range(h)])
        eye = np.stack([np.eye(nx)] * (h - 1)) if h > 1 else np.zeros((0, nx, nx))
        interiors.append((diag, eye.copy(), eye.copy()))
        c = sp.lil_matrix((h * nx, ngamma))
        if i >= 1:  # interface above (index i-1) touches the first interior row
            for x in range(nx):
                c[x, (i - 1) * nx + x] = -1.0
        if i < nsub - 1:  # interface below (index i) touches the last interior row
            for x in range(nx):
                c[(h - 1) * nx + x, i * nx + x] = -1.0
        couplings.append(c.tocsr())
        z += h
        if i < nsub - 1:
            z += 1
    zi = np.cumsum(heights)[:-1] + np.arange(nsub - 1)
    a_gamma = sp.block_diag([sp.csr_matrix(T(shift[z_])) for z_ in zi]).tocsr()
    couplings_t = [None if symmetric else (1.1 * c.T).tocsr() for c in couplings]
    total = sum(h * nx for h in heights) + ngamma
    f = rng.standard_normal(total)
    return interiors, couplings, couplings_t, a_gamma, f
