"""Row f4: execution traces and the cost model, pinned to traces and model
values the REFERENCE harness produced (tests/golden/trace_golden.json, written
by tests/golden/make_trace_golden.py)."""
import json
import os

import pytest

from paper_1108_4181_b200 import errors
from paper_1108_4181_b200.trace import (CostModelParams, ExecutionTrace, allgather_schedule, audit_trace,
                                        predict_preprocess_comm, predict_solve_comm, reference_protocol_trace)

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "trace_golden.json")))


@pytest.mark.parametrize("case", G["cases"], ids=[f"p{c['ranks']}m{c['m']}k{c['k']}" for c in G["cases"]])
def test_reference_protocol_schedule_reproduces_reference_trace(case):
    tr = reference_protocol_trace(case["ranks"], case["m"], case["k"])
    assert [list(r) for r in tr.records] == case["records"]
    assert tr.to_csv() == case["csv"]
    assert tr.per_rank_stages() == case["per_rank_stages"]
    if "audit" in case:
        got = audit_trace(tr, CostModelParams(1e-6, 1e-9, case["m"], case["ranks"]), nrhs=case["k"])
        for key, val in case["audit"].items():
            assert got[key] == pytest.approx(val, rel=1e-15, abs=0), key


@pytest.mark.parametrize("mdl", G["models"], ids=lambda d: f"m{d['m']}p{d['p']}")
def test_cost_model_values(mdl):
    prm = CostModelParams(mdl["alpha"], mdl["beta"], mdl["m"], mdl["p"])
    assert predict_preprocess_comm(prm) == pytest.approx(mdl["pre"], rel=1e-15)
    assert predict_solve_comm(prm) == pytest.approx(mdl["solve"], rel=1e-15)


def test_errors_and_chunking(tmp_path):
    with pytest.raises(errors.InvalidRankCount):
        predict_solve_comm(CostModelParams(1, 1, 4, 1))
    with pytest.raises(ValueError):
        CostModelParams(-1, 0, 4, 2)
    tr = ExecutionTrace(4)
    allgather_schedule(tr, 4, slot_bytes=1000, cap_bytes=300)  # slot above the cap: split into pieces
    assert tr.max_message_bytes() == 300 and tr.total_bytes() == 4 * 3 * 1000
    with pytest.raises(errors.StageViolation):
        audit_trace(tr, CostModelParams(0, 0, 4, 4), collectives=2)
    p = tmp_path / "t.csv"
    tr.to_csv(str(p))
    assert p.read_text().splitlines()[0] == "stage,sender,receiver,bytes"
