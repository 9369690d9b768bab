"""GPU: plan images (btd_plan_export / btd_plan_import) behind the DPLN container
(ref io.py:125-203 write_plan/read_plan) and the CLI plan cache (ref cli.py:183-196).

An imported plan must solve bitwise like the plan it was exported from (same
factors, same kernels); reference-written DPLN v1 files bind to their matrix and
give the reference's answer."""
import json
import os

import numpy as np
import pytest

import blocktri_oracle as O
from paper_1108_4181_b200 import BlockTriMatrix, cli, configs, plan_build, plan_solve
from paper_1108_4181_b200 import io as bio

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("n,m,k,ranks,split,mode", [
    (37, 3, 4, 5, 1, "0"),      # padding, small blocks (fused tree)
    (300, 16, 6, 12, 2, "0"),   # second-level split
    (96, 64, 6, 6, 1, "0"),     # chain kernels
    (64, 24, 5, 4, 1, "1"),     # GEMM-per-step sweep mode
    (1, 4, 3, 1, 1, "0"),       # single row
])
def test_roundtrip_bitwise(tmp_path, monkeypatch, n, m, k, ranks, split, mode):
    monkeypatch.setenv("BTD_FORCE_MODE", mode)
    d, lo, up, f = configs.dominant_numpy(n, m, k, seed=n + m)
    P = BlockTriMatrix(d, lo, up)
    plan = plan_build(P, ranks, split=split)
    x = plan_solve(plan, f)
    path = tmp_path / "p.dpln"
    bio.write_plan(path, plan)
    monkeypatch.setenv("BTD_FORCE_MODE", "0" if mode == "1" else "1")  # the image's mode wins
    q = bio.read_plan(path, P)
    assert (q.L, q.npad, q.mode, q.split, q.nranges) == (plan.L, plan.npad, plan.mode, plan.split, plan.nranges)
    assert q.matches(P)
    assert np.array_equal(plan_solve(q, f), x)
    ref = O.plan_solve(O.plan_build(d, lo, up, ranks), f)
    assert O.max_rel_err(x, ref) <= 1e-9


def test_reference_written_plan_file():
    matrix = bio.read_matrix(os.path.join(GOLDEN, "ref_plan_p3.btr"))
    plan = bio.read_plan(os.path.join(GOLDEN, "ref_plan_p3.dpln"), matrix)
    assert plan.ranks == 5 and plan.L == 8 and plan.npad == 40
    f = np.random.default_rng(1).standard_normal((37, 3, 4))
    x = plan_solve(plan, f)
    ref = O.plan_solve(O.plan_build(matrix.diag, matrix.lower, matrix.upper, 5), f)
    assert O.max_rel_err(x, ref) <= 1e-9


def test_corrupt_image_rejected(tmp_path):
    d, lo, up, _ = configs.dominant_numpy(20, 4, 1, seed=2)
    P = BlockTriMatrix(d, lo, up)
    path = tmp_path / "p.dpln"
    bio.write_plan(path, plan_build(P, 3))
    raw = bytearray(path.read_bytes())
    fplen = int.from_bytes(raw[52:60], "little")
    img = 60 + fplen + 16
    bad = bytearray(raw)
    bad[img:img + 8] = b"NOTAPLAN"  # image magic
    path.write_bytes(bytes(bad))
    with pytest.raises(bio.FileFormatError):
        bio.read_plan(path, P)
    path.write_bytes(bytes(raw[:-16]))  # truncated image
    with pytest.raises(bio.FileFormatError):
        bio.read_plan(path, P)


def test_cli_plan_cache(tmp_path):
    d, lo, up, f = configs.dominant_numpy(64, 8, 2, seed=8)
    bio.write_matrix(tmp_path / "a.btr", BlockTriMatrix(d, lo, up))
    rhs = []
    for i in range(2):
        bio.write_vector(tmp_path / f"f{i}.bvc", f[:, :, i])
        rhs += ["--rhs", str(tmp_path / f"f{i}.bvc")]
    cache = str(tmp_path / "plan.dpln")
    reports, sols = [], []
    for run, ranks in enumerate([4, 4, 2]):
        out = tmp_path / f"out{run}"
        args = ["solve", "--matrix", str(tmp_path / "a.btr"), *rhs, "--ranks", str(ranks), "--out", str(out),
                "--plan-cache", cache]
        assert cli.main(args) == cli.EXIT_OK
        reports.append(json.loads((out / "solve_report.json").read_text())["results"])
        sols.append(bio.read_vector(out / "solution_000.bvc").data)
    assert [r["plan_cache_hit"] for r in reports] == [False, True, False]  # ranks change -> rebuild
    assert np.array_equal(sols[0], sols[1])
    assert bio.read_plan(cache, BlockTriMatrix(d, lo, up)).ranks == 2
