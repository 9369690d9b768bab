"""Small end-to-end exercise of every solve path (compute-sanitizer is closed on this pool;
this is the bounds-checked-by-parity substitute):
stream sweeps + fused tree (M=16), chain sweeps (M=64), mode 1 with split-K row steps and
the side-stream fork (M=128 forced), host pipeline, and a world-2 emulated shard solve
(fused shard-tree kernels).  Sizes are tiny; exits non-zero on a parity failure."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import blocktri_oracle as O  # noqa: E402
from paper_1108_4181_b200 import BlockTriMatrix, configs, plan_build, plan_solve  # noqa: E402


def check(x, d, lo, up, f, ranks):
    ref = O.plan_solve(O.plan_build(d, lo, up, ranks), f)
    err = O.max_rel_err(x, ref)
    assert err <= 1e-9, err


for n, m, k, ranks, split, mode in [(96, 16, 64, 4, 6, "0"), (40, 64, 24, 4, 1, "0"), (47, 128, 64, 16, 1, "1")]:
    os.environ["BTD_FORCE_MODE"] = mode
    d, lo, up, f = configs.dominant_numpy(n, m, k, seed=n)
    plan = plan_build(BlockTriMatrix(d, lo, up), ranks, split=split)
    os.environ.pop("BTD_FORCE_MODE")
    check(plan_solve(plan, torch.from_numpy(f).cuda()).cpu().numpy(), d, lo, up, f, ranks)
    check(plan_solve(plan, f), d, lo, up, f, ranks)  # host pipeline
    print("ok", n, m, k, ranks, split, mode, flush=True)

from test_gpu_shard import _emulate  # noqa: E402

d, lo, up, f = configs.dominant_numpy(200, 16, 20, seed=5)
res = _emulate(d, lo, up, f, 8, 2, 2)
assert res[0] == "ok"
check(res[1], d, lo, up, f, 8)
print("ok shard world 2", flush=True)
