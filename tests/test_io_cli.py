"""Row f2: BTR1/BVC1 containers (byte-compatible with the reference layout)
and the GPU ``solve`` command's config handling / exit codes."""
import json
import os
import struct

import numpy as np
import pytest

from paper_1108_4181_b200 import BlockTriMatrix, BlockVector, cli, configs
from paper_1108_4181_b200 import io as bio


def test_btr1_bvc1_roundtrip_and_layout(tmp_path):
    d, lo, up, f = configs.dominant_numpy(7, 3, 1, seed=4)
    P = BlockTriMatrix(d, lo, up)
    p = tmp_path / "a.btr"
    bio.write_matrix(p, P)
    raw = p.read_bytes()
    assert raw[:4] == b"BTR1" and struct.unpack("<QQ", raw[4:20]) == (7, 3)
    assert len(raw) == 20 + 8 * (7 + 2 * 6) * 9
    Q = bio.read_matrix(p)
    assert Q.fingerprint() == P.fingerprint()
    v = tmp_path / "f.bvc"
    bio.write_vector(v, BlockVector(f[:, :, 0]))
    assert np.array_equal(bio.read_vector(v).data, f[:, :, 0])


def test_format_errors(tmp_path):
    p = tmp_path / "bad.btr"
    p.write_bytes(b"XXXX" + b"\0" * 16)
    with pytest.raises(bio.FileFormatError):
        bio.read_matrix(p)
    p.write_bytes(b"BVC1" + struct.pack("<QQ", 4, 2) + b"\0" * 8)
    with pytest.raises(bio.FileFormatError):
        bio.read_vector(p)


def test_config_validation_and_report_reuse(tmp_path):
    with pytest.raises(cli.ConfigError):
        cli.load_config(None, {"bogus": 1})
    with pytest.raises(cli.ConfigError):
        cli.load_config(None, {"ranks": "4"})
    rep = tmp_path / "r.json"
    rep.write_text(json.dumps({"command": "solve", "config": {"ranks": 3, "tol": 1e-6}}))
    cfg = cli.load_config(str(rep), {"out": "x"})
    assert cfg["ranks"] == 3 and cfg["tol"] == 1e-6 and cfg["out"] == "x" and cfg["split"] == 1
    assert cli.main(["solve", "--ranks", "2"]) == cli.EXIT_CONFIG          # no matrix/rhs
    assert cli.main(["solve", "--matrix", str(tmp_path / "nope.btr"), "--rhs", "x.bvc"]) == cli.EXIT_IO


@pytest.mark.gpu
def test_cli_solve_end_to_end(tmp_path):
    d, lo, up, f = configs.dominant_numpy(64, 4, 3, seed=8)
    bio.write_matrix(tmp_path / "a.btr", BlockTriMatrix(d, lo, up))
    rhs = []
    for i in range(3):
        bio.write_vector(tmp_path / f"f{i}.bvc", f[:, :, i])
        rhs += ["--rhs", str(tmp_path / f"f{i}.bvc")]
    out = tmp_path / "out"
    rc = cli.main(["solve", "--matrix", str(tmp_path / "a.btr"), *rhs, "--ranks", "4", "--out", str(out)])
    assert rc == cli.EXIT_OK
    rep = json.loads((out / "solve_report.json").read_text())
    assert rep["results"]["residual"] <= 1e-12 and rep["results"]["stages"] == 2
    x0 = bio.read_vector(out / "solution_000.bvc").data
    import blocktri_oracle as O
    ref = O.plan_solve(O.plan_build(d, lo, up, 4), f)
    assert O.max_rel_err(x0, ref[:, :, 0]) <= 1e-9


# ---- DPLN plan containers (ref io.py:125-203) ------------------------------------
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
REF_BTR = os.path.join(GOLDEN, "ref_plan_p3.btr")
REF_DPLN = os.path.join(GOLDEN, "ref_plan_p3.dpln")  # written by the reference (make_ref_plan.py)


def test_reference_dpln_header_and_binding(monkeypatch):
    from paper_1108_4181_b200 import dichotomy

    matrix = bio.read_matrix(REF_BTR)
    calls = []
    monkeypatch.setattr(dichotomy, "plan_build", lambda m, ranks, **kw: calls.append((m.n, m.m, ranks)) or "plan")
    assert bio.read_plan(REF_DPLN, matrix) == "plan"  # payload length matched the reference's file
    assert calls == [(37, 3, 5)]
    raw = open(REF_DPLN, "rb").read()
    n, m, ranks, L, npad = struct.unpack("<QQQQQ", raw[12:52])
    assert (n, m, ranks, L, npad) == (37, 3, 5, 8, 40)
    assert len(raw) - 60 - struct.unpack("<Q", raw[52:60])[0] == bio._ref_plan_payload_bytes(n, m, ranks, L)


def test_dpln_rejections(tmp_path, monkeypatch):
    from paper_1108_4181_b200 import dichotomy

    monkeypatch.setattr(dichotomy, "plan_build", lambda *a, **k: "plan")
    matrix = bio.read_matrix(REF_BTR)
    raw = open(REF_DPLN, "rb").read()
    p = tmp_path / "x.dpln"
    for bad, what in [(b"XPLN" + raw[4:], "magic"), (raw[:4] + struct.pack("<Q", 7) + raw[12:], "version"),
                      (raw[:-8], "truncated"), (raw + b"\0", "trailing")]:
        p.write_bytes(bad)
        with pytest.raises(bio.FileFormatError):
            bio.read_plan(p, matrix)
    d, lo, up, _ = configs.dominant_numpy(37, 3, 1, seed=99)  # another matrix
    with pytest.raises(bio.FileFormatError, match="does not belong"):
        bio.read_plan(REF_DPLN, BlockTriMatrix(d, lo, up))
