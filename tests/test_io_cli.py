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
