"""Full BASELINE.json sizes (c1-c4).

``test_full_size_parity``: parity on IDENTICAL inputs at full size -- the
numpy-stream arrays of ``configs.generate(name)`` that the unmodified reference
was run on (tests/golden/make_fullsize_golden.py) -- solved on the GPU with the
bench's plan parameters and all K columns, then compared with
  * the reference-written golden: X at sampled block rows (all 63 rows for
    c3) and per-column checksums over all rows, max rel err <= 1e-9;
  * the C oracle run live on the same inputs (all rows, the golden's columns),
    max rel err <= 1e-9 (c1, c2, c4; c3's M = 2048 CPU plan takes minutes, its
    golden holds every row);
  * the relative residual max|P X - F| / max|F| <= 1e-10 over all columns
    (ref cli.py:211-214).

``test_full_size_properties``: size-independent properties on the bench's
device-generated inputs: residual, linearity, column independence, bitwise
run-to-run determinism.
"""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def _residual(torch, diag, lower, upper, X, F):
    y = torch.bmm(diag, X)
    y[1:] -= torch.bmm(lower, X[:-1])
    y[:-1] -= torch.bmm(upper, X[1:])
    return ((y - F).abs().max() / F.abs().max()).item()


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_full_size_parity(name):
    import torch

    import bench
    import parity
    from paper_1108_4181_b200 import configs, plan_build_arrays, plan_solve

    g, meta = parity.golden(name)
    assert g is not None, f"missing tests/golden/fullsize_{name}.npz"
    cols = meta["cols"]
    torch.cuda.set_device(0)
    diag, lower, upper, F = configs.generate(name)
    f_cols = np.ascontiguousarray(F[:, :, cols])
    if configs.CONFIGS[name]["kind"] != "schur":  # S is formed with BLAS: equal to rounding only
        assert parity.sha_inputs(diag, lower, upper, f_cols) == meta["sha_inputs"]
    dd, dl, du = (torch.from_numpy(a).cuda() for a in (diag, lower, upper))
    Fd = torch.from_numpy(F).cuda()
    del F
    ranks, split = bench.plan_params(name, 1)
    plan = plan_build_arrays(dd, dl, du, ranks, split=split)
    X = plan_solve(plan, Fd)
    assert _residual(torch, dd, dl, du, X, Fd) <= 1e-10
    x_cols = X[:, :, cols].cpu().numpy()
    del X, Fd, dd, dl, du, plan
    torch.cuda.empty_cache()
    rep = parity.compare_golden(name, x_cols)
    assert rep["max_rel_err_sampled_rows"] <= 1e-9, rep
    assert rep["checksum_rel_err"] <= 1e-9, rep
    if name != "c3":
        ref = parity.oracle_columns(diag, lower, upper, f_cols, configs.CONFIGS[name]["ranks"])
        assert parity.max_rel_err(x_cols, ref) <= 1e-9


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_full_size_properties(name):
    import torch

    import bench
    from paper_1108_4181_b200 import configs, plan_build_arrays, plan_solve

    torch.cuda.set_device(0)
    ranks, split = bench.plan_params(name, 1)
    diag, lower, upper, F = configs.generate(name, device="cuda")
    plan = plan_build_arrays(diag, lower, upper, ranks, split=split)
    X = plan_solve(plan, F)
    assert torch.isfinite(X).all()
    assert _residual(torch, diag, lower, upper, X, F) <= 1e-10
    del diag, lower, upper
    torch.cuda.empty_cache()
    # determinism (no atomics anywhere on the path)
    assert torch.equal(plan_solve(plan, F), X)
    # linearity with a second right-hand side (columns reversed)
    G = F.flip(2).contiguous()
    XG = plan_solve(plan, G)
    XC = plan_solve(plan, 2.0 * F - 3.0 * G)
    ref = 2.0 * X - 3.0 * XG
    assert ((XC - ref).abs().max() / ref.abs().max()).item() <= 1e-12
    del G, XG, XC, ref
    # column independence: the first half of the columns alone
    k2 = F.shape[2] // 2
    Xh = plan_solve(plan, F[:, :, :k2].contiguous())
    assert ((Xh - X[:, :, :k2]).abs().max() / X.abs().max()).item() <= 1e-13
    del F, X, Xh
    torch.cuda.empty_cache()
