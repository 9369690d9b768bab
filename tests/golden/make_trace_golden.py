"""Golden traces for row f4 from the REFERENCE harness itself (blocktri.harness:
harness_solve -> ExecutionTrace, audit_trace, predict_* cost model).

    python tests/golden/make_trace_golden.py

Output: tests/golden/trace_golden.json (records + audit per case, model values).
"""
from __future__ import annotations

import json
import subprocess
import sys

from make_golden import HERE, SCRATCH, _inputs, build_reference

CASES = [(64, 3, 2, 4, 1), (40, 4, 3, 5, 2), (96, 2, 1, 8, 3), (30, 5, 4, 3, 4), (17, 8, 2, 16, 5), (12, 3, 1, 1, 6)]
PARAMS = [(1e-6, 1e-9, 16, 8), (2e-6, 5e-10, 64, 64), (0.0, 1e-9, 3, 2), (5e-6, 0.0, 256, 3)]


def child():
    sys.path.insert(0, str(SCRATCH / "src"))
    from blocktri import core, dichotomy, harness

    out = {"cases": [], "models": []}
    for n, m, k, ranks, seed in CASES:
        d, lo, up, f = _inputs("dominant", n, m, k, seed)
        plan = dichotomy.plan_build(core.BlockTriMatrix(d, lo, up), ranks)
        _x, tr = harness.harness_solve(plan, f)
        entry = dict(n=n, m=m, k=k, ranks=ranks, records=[list(r) for r in tr.records], csv=tr.to_csv(),
                     per_rank_stages=tr.per_rank_stages())
        if ranks >= 2:
            entry["audit"] = harness.audit_trace(tr, harness.CostModelParams(1e-6, 1e-9, m, ranks), nrhs=k)
        out["cases"].append(entry)
    for a, b, m, p in PARAMS:
        prm = harness.CostModelParams(a, b, m, p)
        out["models"].append(dict(alpha=a, beta=b, m=m, p=p, pre=harness.predict_preprocess_comm(prm),
                                  solve=harness.predict_solve_comm(prm)))
    (HERE / "trace_golden.json").write_text(json.dumps(out, indent=1))
    print("cases", len(out["cases"]))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
    else:
        build_reference()
        res = subprocess.run([sys.executable, __file__, "--child"], check=True, capture_output=True, text=True)
        print(res.stdout.strip())
