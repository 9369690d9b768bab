"""Solves of one plan issued on different CUDA streams without host
synchronisation in between: the plan's shared scratch is ordered on the device
(event wait), so every result is correct and the host never blocks on the
earlier stream (include/blocktri_b200.h, btd_plan_solve threading note)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m,k,ranks", [(300, 16, 64, 12), (64, 128, 32, 8)])
def test_interleaved_streams(n, m, k, ranks):
    import coracle
    import torch

    from paper_1108_4181_b200 import BlockTriMatrix, configs, plan_build, plan_solve

    torch.cuda.set_device(0)
    d, lo, up, f = configs.dominant_numpy(n, m, 4 * k, seed=n + m)
    plan = plan_build(BlockTriMatrix(d, lo, up), ranks)
    ref = coracle.CPlan(d, lo, up, ranks).solve(f)
    fs = [torch.from_numpy(np.ascontiguousarray(f[:, :, i * k:(i + 1) * k])).cuda() for i in range(4)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = []
    for rep in range(3):
        for i, fi in enumerate(fs):
            s = streams[(i + rep) % 2]
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                outs.append((i, plan_solve(plan, fi)))
    torch.cuda.synchronize()
    for i, x in outs:
        xi = x.cpu().numpy()
        r = ref[:, :, i * k:(i + 1) * k]
        assert np.abs(xi - r).max() <= 1e-9 * np.abs(r).max()
