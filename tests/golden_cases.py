"""Loads the reference-generated golden fixtures (see tests/golden/make_golden.py)."""
import hashlib
import json
import os

import numpy as np

from paper_1108_4181_b200 import configs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load():
    with open(os.path.join(GOLDEN, "cases.json")) as fh:
        meta = json.load(fh)
    npz = {b: dict(np.load(os.path.join(GOLDEN, f"golden_{b}.npz"))) for b in ("compiled", "python")}
    return meta, npz


def sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def case_inputs(c):
    k = max(c["k"], 1)
    if c["kind"] == "dominant":
        diag, lower, upper, f = configs.dominant_numpy(c["n"], c["m"], k, c["seed"])
    else:
        diag, lower, upper, f = configs.strip_numpy(c["n"], c["m"], k, 0.01, c["seed"])
    if c["form"] == "2d":
        f = np.ascontiguousarray(f[:, :, 0])
    return diag, lower, upper, f


def singular_inputs(n, m, row, seed=5):
    diag, lower, upper, _ = configs.dominant_numpy(n, m, 0, seed)
    diag[row] = 0.0
    if row > 0:
        upper[row - 1] = 0.0
        lower[row - 1] = 0.0
    if row < n - 1:
        lower[row] = 0.0
        upper[row] = 0.0
    return diag, lower, upper
