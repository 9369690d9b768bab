"""Multi-process (world_size 2, gloo, CPU) checks of the row-sharded solve
orchestration: partition, contribution all-gather, (base, carry) exchange
layout, error propagation.  Local compute = numpy restatement of the native
shard phases (tests/shard_numpy_backend.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1108_4181_b200 import configs
from paper_1108_4181_b200.distributed import ShardedPlan, stage_count


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    for p_ in (here, os.path.join(os.path.dirname(here), "oracle"), os.path.dirname(here)):
        sys.path.insert(0, p_)
    import torch

    from golden_cases import singular_inputs
    from shard_numpy_backend import NumpyShardBackend

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m, k, ranks, split = case["n"], case["m"], case["k"], case["ranks"], case["split"]
        if case.get("singular_row") is not None:
            d, lo, up = singular_inputs(n, m, case["singular_row"])
            f = np.zeros((n, m, k))
        else:
            d, lo, up, f = configs.dominant_numpy(n, m, k, seed=case["seed"])
        try:
            plan = ShardedPlan(d, lo, up, ranks, split=split, backend=NumpyShardBackend())
        except Exception as exc:  # noqa: BLE001
            q.put((rank, "error", type(exc).__name__, getattr(exc, "row", None)))
            return
        from paper_1108_4181_b200.trace import ExecutionTrace

        tr = ExecutionTrace(world)
        xl = plan.solve(torch.from_numpy(np.ascontiguousarray(f[plan.row_lo:plan.row_hi])), trace=tr)
        q.put((rank, "ok", plan.row_lo, plan.row_hi, xl.numpy(), tr.records, tr.timings,
               plan.collectives_per_solve(k)))
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("case", [
    dict(n=96, m=3, k=4, ranks=4, split=1, seed=1),
    dict(n=101, m=4, k=3, ranks=2, split=3, seed=2),     # padding, split second level
    dict(n=10, m=2, k=2, ranks=8, split=1, seed=3),      # L = 2, fully padded tail range
])
def test_world2_matches_oracle(case):
    import blocktri_oracle as O

    res = _run(case)
    assert all(r[1] == "ok" for r in res), res
    x = np.concatenate([r[4] for r in res])
    assert res[0][2] == 0 and res[-1][3] == case["n"]
    d, lo, up, f = configs.dominant_numpy(case["n"], case["m"], case["k"], seed=case["seed"])
    ref = O.plan_solve(O.plan_build(d, lo, up, case["ranks"]), f)
    assert O.max_rel_err(x, ref) <= 1e-9
    assert O.rel_residual(d, lo, up, x, f) <= 1e-10


def test_world2_singular_pivot_raised_on_every_rank():
    # singular block in the second rank's rows; every rank must raise the same error
    res = _run(dict(n=24, m=3, k=1, ranks=4, split=1, seed=0, singular_row=19))
    assert [r[1] for r in res] == ["error", "error"]
    assert {r[2] for r in res} == {"SingularPivot"}
    assert res[0][3] == res[1][3]


def test_stage_law():
    assert [stage_count(p) for p in (1, 2, 3, 4, 6, 8, 64, 256)] == [0, 1, 2, 2, 3, 3, 6, 8]


@pytest.mark.parametrize("world", [2, 4])
def test_solve_trace_stage_law_and_volume(world):
    """Row f4: the sharded solve's logical trace has collectives*ceil(log2 W) stages,
    every rank logs the same schedule, each all-gather moves W(W-1) slots."""
    from paper_1108_4181_b200.trace import CostModelParams, ExecutionTrace, audit_trace

    case = dict(n=200, m=3, k=2, ranks=8, split=2, seed=7)
    res = _run(case, world=world)
    assert all(r[1] == "ok" for r in res), res
    recs, ncoll = res[0][5], res[0][7]
    assert all(r[5] == recs for r in res) and all(r[7] == ncoll for r in res)
    assert all(len(r[6]) == ncoll for r in res)  # one timing per real collective
    tr = ExecutionTrace(world)
    tr.records = [tuple(x) for x in recs]
    assert tr.stages == ncoll * stage_count(world)
    m, k = case["m"], case["k"]
    carry_total = world * (world - 1) * m * k * 8
    assert tr.total_bytes() >= carry_total
    rep = audit_trace(tr, CostModelParams(1e-6, 1e-9, m, world), nrhs=k, collectives=ncoll)
    assert rep["stages"] == tr.stages and rep["max_message_bytes"] <= (m * m + m) * 8 * k
    x = np.concatenate([r[4] for r in res])
    import blocktri_oracle as O

    d, lo, up, f = configs.dominant_numpy(case["n"], m, k, seed=case["seed"])
    assert O.max_rel_err(x, O.plan_solve(O.plan_build(d, lo, up, case["ranks"]), f)) <= 1e-9
