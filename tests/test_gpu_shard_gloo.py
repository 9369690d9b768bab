"""ShardedPlan end to end through torch.distributed with the NATIVE shard API:
world 2 and 4 processes share the one GPU, collectives over gloo (host), so no
kernel waits on another rank's kernel.  Checks the device solve and the pipelined
host-buffer solve of every rank against the CPU oracle (the NCCL flavour of the
same code is bench.py's multi-GPU path)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


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
    import torch.distributed as dist

    from paper_1108_4181_b200 import configs
    from paper_1108_4181_b200.distributed import ShardedPlan

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m, k, ranks, split = case
        d, lo, up, f = configs.dominant_numpy(n, m, k, seed=n + m + world)
        plan = ShardedPlan(torch.from_numpy(d).cuda(), torch.from_numpy(lo).cuda(), torch.from_numpy(up).cuda(),
                           ranks, split=split)
        fl = torch.from_numpy(np.ascontiguousarray(f[plan.row_lo:plan.row_hi]))
        x_dev = plan.solve(fl.cuda()).cpu().numpy()
        xh = torch.zeros_like(fl).pin_memory()
        plan.solve_host(fl.pin_memory(), xh, chunks=2)
        q.put((rank, plan.row_lo, plan.row_hi, x_dev, xh.numpy()))
        plan.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, (256, 16, 8, 8, 2)), (2, (96, 64, 6, 4, 1)), (4, (203, 8, 6, 4, 3)),
                                        (2, (40, 256, 4, 4, 1))])
def test_sharded_plan_two_processes_one_gpu(world, case):
    import torch.multiprocessing as mp

    import blocktri_oracle as O
    from paper_1108_4181_b200 import configs

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, m, k, ranks, split = case
    d, lo, up, f = configs.dominant_numpy(n, m, k, seed=n + m + world)
    x = np.concatenate([r[3] for r in res])
    xh = np.concatenate([r[4] for r in res])
    assert [r[1] for r in res] == sorted(r[1] for r in res) and res[-1][2] == n
    ref = O.plan_solve(O.plan_build(d, lo, up, ranks), f)
    for y in (x, xh):
        assert O.max_rel_err(y, ref) <= 1e-9
        assert O.rel_residual(d, lo, up, y, f) <= 1e-10
