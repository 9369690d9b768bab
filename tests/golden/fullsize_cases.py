"""Full-size parity cases shared by make_fullsize_golden.py (writer, runs the
reference) and tests/test_gpu_fullsize.py (reader, runs the GPU and the C oracle).

Columns: a few columns of each config's seeded F (SURVEY.md 7 hard part 7 and
BASELINE.md 2 allow column subsets: columns are independent).  Rows: a fixed
sample of block rows (both ends, interior spread) -- all rows of c3's 63."""

from __future__ import annotations

import numpy as np

CASES = {
    # ranks = the reference's P for its own run (any valid P gives the same
    # solution to ~1e-14)
    "c1": dict(cols=(0, 128, 255), ranks=32, backend="python"),
    "c2": dict(cols=(0, 511, 1023), ranks=64, backend="compiled"),
    "c3": dict(cols=(0, 127), ranks=8, backend="python"),
    "c4": dict(cols=(0, 32, 63), ranks=8, backend="compiled"),
}

N = {"c1": 4096, "c2": 16384, "c3": 63, "c4": 1 << 20}


def sample_rows(name, count=192):
    n = N[name]
    if n <= count:
        return np.arange(n, dtype=np.int64)
    rows = np.concatenate([np.arange(4), np.arange(n - 4, n),
                           np.linspace(0, n - 1, count).astype(np.int64)])
    return np.unique(rows)


def checksums(x):
    """Per-column size-independent summaries over all block rows."""
    return dict(col_sum=x.sum(axis=(0, 1)), col_abs_sum=np.abs(x).sum(axis=(0, 1)),
                col_max=np.abs(x).max(axis=(0, 1)))
