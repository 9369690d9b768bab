"""PARITY CHECKER -- TEST / BENCH-REPORT INFRASTRUCTURE ONLY.

Compares a GPU solution of a BASELINE.json config, solved on the numpy-stream
inputs (``configs.generate`` / ``generate_columns``: the arrays the reference
itself was run on), with

* the reference-written full-size goldens (tests/golden/fullsize_<name>.npz,
  made by tests/golden/make_fullsize_golden.py from the unmodified reference):
  X at sampled block rows (all rows for c3) and per-column checksums over all
  rows;
* the C oracle (oracle/liboracle.so, pinned to the reference goldens by
  tests/test_coracle.py) run live on the same inputs, all rows, a column subset.

Metrics follow the reference tests: max|X - X_ref| / max|X_ref| (test_core.py:
154,208).  Used by tests/test_gpu_fullsize.py and by bench.py's parity report
(after the timed region).  Never imported by paper_1108_4181_b200/.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(ROOT, "tests", "golden")
for _p in (HERE, GOLDEN):
    if _p not in sys.path:
        sys.path.insert(0, _p)

import fullsize_cases as FC  # noqa: E402


def golden(name):
    p = os.path.join(GOLDEN, f"fullsize_{name}.npz")
    if not os.path.exists(p):
        return None, None
    with open(os.path.join(GOLDEN, f"fullsize_{name}.json")) as fh:
        meta = json.load(fh)
    return dict(np.load(p)), meta


def compare_golden(name, x_cols):
    """x_cols: (N, M, len(cols)) host array of the GPU solution at the golden's
    columns.  Returns a dict of errors (None when no golden exists)."""
    g, meta = golden(name)
    if g is None:
        return None
    rows = g["rows"]
    ref = g["x_rows"]
    scale = float(g["col_max"].max())
    err_rows = float(np.abs(x_cols[rows] - ref).max() / scale)
    cs = FC.checksums(x_cols)
    err_sum = float((np.abs(cs["col_sum"] - g["col_sum"]) / g["col_abs_sum"]).max())
    err_abs = float((np.abs(cs["col_abs_sum"] - g["col_abs_sum"]) / g["col_abs_sum"]).max())
    err_max = float((np.abs(cs["col_max"] - g["col_max"]) / g["col_max"]).max())
    return {"max_rel_err_sampled_rows": err_rows, "rows_compared": int(len(rows)),
            "checksum_rel_err": max(err_sum, err_abs, err_max), "cols": meta["cols"],
            "ref_backend": meta["backend"], "ref_ranks": meta["ranks"],
            "ref_rel_residual": meta["ref_rel_residual"], "sha_inputs": meta["sha_inputs"]}


def oracle_columns(diag, lower, upper, f_cols, ranks):
    """C-oracle solution (all rows) of the column subset f_cols."""
    import coracle

    plan = coracle.CPlan(diag, lower, upper, ranks)
    try:
        return plan.solve(f_cols)
    finally:
        del plan


def max_rel_err(x, ref):
    return float(np.abs(x - ref).max() / np.abs(ref).max())


def sha_inputs(diag, lower, upper, f_cols):
    import hashlib

    h = hashlib.sha256()
    for a in (diag, lower, upper, f_cols):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
