"""Seeded synthetic inputs for the BASELINE.json configurations.

Draw order and distributions follow BASELINE.json ``configs`` and SURVEY.md
section 8(d): ``numpy.random.default_rng(seed)`` drawing A (``lower``, N-1
blocks), then B (``upper``), then C (``diag``), then F.  Config 1 is the
reference's ``models._blocktri_strip`` operator (``models.py:48-57``);
config 3's operator is the explicit Schur complement built in
:mod:`paper_1108_4181_b200.schur`.

Large configs can also be drawn on the GPU (``device=...``) with a seeded
torch generator; those arrays differ from the numpy stream, so parity at full
size is checked through residuals, and the exact-array parity cases use the
numpy stream at sizes the oracle finishes in seconds.
"""

from __future__ import annotations

import numpy as np

CONFIGS = {
    # name: (N, M, K, P)   P = ranks used for the reference-equivalent plan
    "c0": dict(n=512, m=8, k=32, ranks=4, kind="dominant"),
    "c1": dict(n=4096, m=256, k=256, ranks=32, kind="strip", shift=0.01),
    "c2": dict(n=16384, m=64, k=1024, ranks=64, kind="dominant"),
    "c3": dict(n=63, m=2048, k=128, ranks=8, kind="schur", nx=2048, nz=8192, nsub=64),
    "c4": dict(n=1 << 20, m=16, k=64, ranks=8, kind="dominant"),
}


def dominant_numpy(n, m, k, seed=0):
    """Config 0/2/4 family: A, B ~ U(-1,1)/(4M); C = I + U(-1,1)/(4M); F ~ N(0,1)."""
    rng = np.random.default_rng(seed)
    s = 1.0 / (4 * m)
    lower = rng.uniform(-1.0, 1.0, size=(n - 1, m, m)) * s
    upper = rng.uniform(-1.0, 1.0, size=(n - 1, m, m)) * s
    diag = rng.uniform(-1.0, 1.0, size=(n, m, m)) * s
    diag += np.eye(m)
    f = rng.standard_normal(size=(n, m, k)) if k else None
    return diag, lower, upper, f


def strip_numpy(n, m, k, shift=0.01, seed=0):
    """Config 1: C = tridiag(-1, 4+shift, -1), A = B = I (ref models.py:48-57);
    F ~ N(0,1) from default_rng(seed)."""
    col = np.diag(np.full(m, 4.0 + shift)) - np.diag(np.ones(m - 1), 1) - np.diag(np.ones(m - 1), -1)
    diag = np.broadcast_to(col, (n, m, m)).copy()
    eye = np.broadcast_to(np.eye(m), (n - 1, m, m)).copy()
    rng = np.random.default_rng(seed)
    f = rng.standard_normal(size=(n, m, k)) if k else None
    return diag, eye, eye.copy(), f


def dominant_torch(n, m, k, seed=0, device="cuda"):
    """Same distributions as :func:`dominant_numpy`, drawn on the device
    (Philox stream; not bit-identical to numpy)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    s = 1.0 / (4 * m)
    kw = dict(dtype=torch.float64, device=device, generator=g)
    lower = (torch.rand((n - 1, m, m), **kw) * 2 - 1) * s
    upper = (torch.rand((n - 1, m, m), **kw) * 2 - 1) * s
    diag = (torch.rand((n, m, m), **kw) * 2 - 1) * s
    diag += torch.eye(m, dtype=torch.float64, device=device)
    f = torch.randn((n, m, k), **kw) if k else None
    return diag, lower, upper, f


def strip_torch(n, m, k, shift=0.01, seed=0, device="cuda"):
    import torch

    col = (torch.diag(torch.full((m,), 4.0 + shift, dtype=torch.float64))
           - torch.diag(torch.ones(m - 1, dtype=torch.float64), 1)
           - torch.diag(torch.ones(m - 1, dtype=torch.float64), -1)).to(device)
    diag = col.expand(n, m, m).contiguous()
    eye = torch.eye(m, dtype=torch.float64, device=device).expand(n - 1, m, m).contiguous()
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    f = torch.randn((n, m, k), dtype=torch.float64, device=device, generator=g) if k else None
    return diag, eye, eye.clone(), f


def _normal_rows(rng, n, m, k, cols, chunk_rows):
    """Columns ``cols`` of ``rng.standard_normal((n, m, k))`` drawn in row chunks:
    Generator draws are sequential, so chunked draws give the identical stream."""
    cols = np.asarray(cols, dtype=np.int64)
    out = np.empty((n, m, len(cols)))
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        out[r0:r1] = rng.standard_normal(size=(r1 - r0, m, k))[:, :, cols]
    return out


def generate_columns(name, cols, *, seed=0, chunk_rows=None):
    """Numpy-stream inputs of config ``name`` with F restricted to columns ``cols``.

    (diag, lower, upper, F[:, :, cols]) are bit-identical to ``generate(name)``
    (same generator, same draw order), without holding the full F: this is how
    the full-size parity tests and the reference-written full-size goldens
    (tests/golden/make_fullsize_golden.py) get identical inputs at BASELINE sizes."""
    cfg = dict(CONFIGS[name])
    n, m, k = cfg["n"], cfg["m"], cfg["k"]
    if chunk_rows is None:
        chunk_rows = max(1, (1 << 24) // (m * k))
    if cfg["kind"] == "dominant":
        rng = np.random.default_rng(seed)
        s = 1.0 / (4 * m)
        lower = rng.uniform(-1.0, 1.0, size=(n - 1, m, m)) * s
        upper = rng.uniform(-1.0, 1.0, size=(n - 1, m, m)) * s
        diag = rng.uniform(-1.0, 1.0, size=(n, m, m)) * s
        diag += np.eye(m)
        return diag, lower, upper, _normal_rows(rng, n, m, k, cols, chunk_rows)
    if cfg["kind"] == "strip":
        diag, lower, upper, _ = strip_numpy(n, m, 0, cfg["shift"], seed)
        return diag, lower, upper, _normal_rows(np.random.default_rng(seed), n, m, k, cols, chunk_rows)
    d, lo, up, f = generate(name, seed=seed)
    return d, lo, up, np.ascontiguousarray(f[:, :, np.asarray(cols)])


def generate(name, *, device=None, seed=0, n=None, k=None):
    """Inputs of config ``name`` (optionally with N or K overridden)."""
    cfg = dict(CONFIGS[name])
    n = cfg["n"] if n is None else n
    k = cfg["k"] if k is None else k
    m = cfg["m"]
    if cfg["kind"] == "dominant":
        return (dominant_numpy(n, m, k, seed) if device is None
                else dominant_torch(n, m, k, seed, device))
    if cfg["kind"] == "strip":
        return (strip_numpy(n, m, k, cfg["shift"], seed) if device is None
                else strip_torch(n, m, k, cfg["shift"], seed, device))
    if cfg["kind"] == "schur":
        from . import schur

        if device is None:
            d, lo, up = schur.schur_blocks_numpy(cfg["nx"], cfg["nz"], cfg["nsub"], seed=seed)
            f = np.random.default_rng(seed).standard_normal((d.shape[0], m, k)) if k else None
            return d, lo, up, f
        import torch

        d, lo, up = schur.schur_blocks_torch(cfg["nx"], cfg["nz"], cfg["nsub"], device=device, seed=seed)
        f = None
        if k:
            g = torch.Generator(device=device)
            g.manual_seed(seed)
            f = torch.randn((d.shape[0], m, k), dtype=torch.float64, device=device, generator=g)
        return d, lo, up, f
    raise ValueError(f"unknown config kind {cfg['kind']}")
