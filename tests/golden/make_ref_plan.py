"""Generate a reference-written DPLN v1 plan file (plus its BTR1 matrix) by running
the REFERENCE package's own ``blocktri.io.write_matrix`` / ``write_plan``.

Run in the build container (where /root/reference exists), after or instead of
make_golden.py (same scratch build under /tmp):

    python tests/golden/make_ref_plan.py

Output: tests/golden/ref_plan_p3.btr, tests/golden/ref_plan_p3.dpln -- used by
tests/test_io_cli.py to pin this package's DPLN reader (header, fingerprint
binding, payload length) against a file the reference itself wrote.
"""
from __future__ import annotations

import subprocess
import sys

from make_golden import HERE, SCRATCH, _inputs, build_reference

CASE = ("dominant", 37, 3, 1, 5, 13)  # kind, n, m, k, ranks, seed (golden case p3_nodiv's matrix)


def child():
    sys.path.insert(0, str(SCRATCH / "src"))
    from blocktri import core, dichotomy, io

    kind, n, m, k, ranks, seed = CASE
    diag, lower, upper, _ = _inputs(kind, n, m, k, seed)
    P = core.BlockTriMatrix(diag, lower, upper)
    io.write_matrix(str(HERE / "ref_plan_p3.btr"), P)
    io.write_plan(str(HERE / "ref_plan_p3.dpln"), dichotomy.plan_build(P, ranks))
    print("fingerprint", P.fingerprint())


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
    else:
        build_reference()
        out = subprocess.run([sys.executable, __file__, "--child"], check=True, capture_output=True, text=True)
        print(out.stdout.strip())
