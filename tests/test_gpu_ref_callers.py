"""The reference's own callers of the path, UNCHANGED, driven through
install() on the B200: ``schur`` (SchurSystem / solve_schur / probing
preconditioner -> BlocktriOperator, ref schur.py:168-195,365-378),
``bands.BandSolver`` (bands.py:157-173), ``cli.cmd_solve`` with ranks >= 2 and
a plan cache (cli.py:171-232: harness.harness_solve + io.write_plan/read_plan)
and ``cli.cmd_bench`` (cli.py:336-360).  Each result is compared with the same
call on the uninstalled reference (its CPU path) on identical inputs.

The reference package comes from oracle/_ref (oracle/build_ref.sh; it travels
to the GPU box with the snapshot)."""
import json
import os
import struct
import sys
import warnings

import numpy as np
import pytest

import refpkg

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))


@pytest.fixture(scope="module")
def ref():
    if not refpkg.available():
        pytest.skip("reference package not built (oracle/build_ref.sh)")
    import torch

    torch.cuda.set_device(0)
    return refpkg.import_blocktri()


def _rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max())


def _installed(fn, **kw):
    from paper_1108_4181_b200 import install

    install.install(**kw)
    try:
        return fn()
    finally:
        install.uninstall()


def test_schur_pipeline_unchanged(ref):
    from blocktri import core, schur
    from schur_cases import CASES, build

    for name, nx, heights, ranks, seed, symm in CASES:
        def run():
            interiors, cpl, cplt, a_gamma, f = build(nx, heights, seed, symm)
            blocks = [schur.SubdomainBlock(i, schur.BlocktriOperator(core.BlockTriMatrix(*interiors[i]), ranks),
                                           cpl[i], cplt[i], symmetric=symm) for i in range(len(heights))]
            sys_ = schur.SchurSystem(blocks, a_gamma)
            out = {"plan_types": {type(b.op.plan).__name__ for b in blocks}}
            if symm:
                x, st = schur.solve_schur(sys_, f, tol=1e-10)
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    pc, band = schur.probing_preconditioner(sys_, 2, ranks=2)
                xp, stp = schur.solve_schur(sys_, f, tol=1e-10, precond=pc.apply)
                out.update(x=x, it=st.iterations, band=band.bands, xp=xp, itp=stp.iterations)
            out["rhs"] = schur.schur_rhs(sys_, f)
            out["S_e0"] = schur.schur_apply(sys_, np.eye(sys_.ngamma)[0])
            return out

        cpu = run()
        gpu = _installed(run)
        assert cpu["plan_types"] == {"DichotomyPlan"} and gpu["plan_types"] == {"DevicePlan"}
        assert _rel(gpu["rhs"], cpu["rhs"]) <= 1e-12, name
        assert _rel(gpu["S_e0"], cpu["S_e0"]) <= 1e-12, name
        if symm:
            assert _rel(gpu["x"], cpu["x"]) <= 1e-8, name
            assert abs(gpu["it"] - cpu["it"]) <= 1, name
            assert _rel(gpu["band"], cpu["band"]) <= 1e-12, name
            assert _rel(gpu["xp"], cpu["xp"]) <= 1e-8, name


def test_band_solver_unchanged(ref):
    from blocktri import bands
    from band_cases import CASES, dense_band, rhs

    from paper_1108_4181_b200.dichotomy import DevicePlan

    for name, n, d, m, seed, spd in CASES:
        a = dense_band(n, d, seed, spd)
        r = rhs(n, seed)

        def run():
            bm = bands.BandMatrix.from_dense(a, d, symmetric=spd)
            s = bands.BandSolver(bm)
            return s.solve(r), type(s.plan)

        x_cpu, _ = run()
        x_gpu, cls = _installed(run)
        assert cls is DevicePlan
        assert _rel(x_gpu, x_cpu) <= 1e-9, name
        assert _rel(a @ x_gpu, r) <= 1e-10, name


def _write_inputs(ref, tmp, n=48, m=6, k=3, seed=3):
    from blocktri import core
    from blocktri import io as rio

    from paper_1108_4181_b200 import configs

    d_, lo, up, f = configs.dominant_numpy(n, m, k, seed)
    rio.write_matrix(str(tmp / "A.btr"), core.BlockTriMatrix(d_, lo, up))
    paths = []
    for i in range(k):
        p = str(tmp / f"f{i}.bvc")
        rio.write_vector(p, core.BlockVector(np.ascontiguousarray(f[:, :, i])))
        paths.append(p)
    return d_, lo, up, f, paths


@pytest.mark.parametrize("ranks", [1, 4])
def test_cli_solve_with_plan_cache_unchanged(ref, tmp_path, ranks):
    from blocktri import cli

    from paper_1108_4181_b200 import io as bio

    _d, _lo, _up, f, paths = _write_inputs(ref, tmp_path)

    def run(tag):
        out = tmp_path / tag
        cfg = cli.load_config("solve", None, {"matrix": str(tmp_path / "A.btr"), "rhs": paths, "ranks": ranks,
                                              "out": str(out), "plan_cache": str(tmp_path / f"{tag}.dpln"),
                                              "tol": 1e-10})
        first = cli.cmd_solve(cfg)
        second = cli.cmd_solve(cfg)  # reuses the cache (read_plan)
        xs = [np.fromfile(p, dtype="<f8", offset=20) for p in first["solutions"]]
        with open(tmp_path / f"{tag}.dpln", "rb") as fh:
            fh.read(4)
            (version,) = struct.unpack("<Q", fh.read(8))
        return first, second, xs, version

    c1, c2, xc, vc = run("cpu")
    g1, g2, xg, vg = _installed(lambda: run("gpu"))
    assert vc == 1 and vg == bio.GPU_PLAN_VERSION
    assert g1["stages"] == c1["stages"] and g2["stages"] == c2["stages"]
    assert g1["residual"] <= 1e-12 and g2["residual"] <= 1e-12
    for a, b in zip(xg, xc):
        assert _rel(a, b) <= 1e-12
    rep = json.loads((tmp_path / "gpu" / "solve_report.json").read_text())
    assert rep["results"]["ranks"] == ranks


def test_cli_bench_unchanged(ref, tmp_path):
    from blocktri import cli

    def run(tag):
        cfg = cli.load_config("bench", None, {"out": str(tmp_path / tag), "p_list": [2, 4, 8], "n": 64, "m": 4})
        cli.cmd_bench(cfg)
        return (tmp_path / tag / "bench.csv").read_text()

    assert _installed(lambda: run("gpu")) == run("cpu")
