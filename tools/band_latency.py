"""K=1 band-solve latency (preconditioner apply inside CG)."""
import sys, time
import numpy as np
import torch
from paper_1108_4181_b200 import bands

for n, d, split in [(129024, 16, None), (129024, 16, 1), (129024, 8, None), (16384, 4, None)]:
    rng = np.random.default_rng(0)
    bd = np.zeros((2 * d + 1, n))
    for off in range(1, d + 1):
        v = rng.uniform(-1, 1, n - off)
        bd[d + off, : n - off] = v
        bd[d - off, off:] = v
    bd[d] = np.abs(bd).sum(axis=0) + 1.0
    b = bands.BandMatrix(n, d, bd, symmetric=True)
    t0 = time.perf_counter()
    s = bands.BandSolver(b, split=split)
    build = time.perf_counter() - t0
    r = rng.standard_normal(n)
    rt = torch.from_numpy(r).cuda()
    for _ in range(5):
        s.solve(rt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        x = s.solve(rt)
    e1.record(); torch.cuda.synchronize()
    dev_us = e0.elapsed_time(e1) / 200 * 1e3
    t0 = time.perf_counter()
    for _ in range(50):
        x = s.solve(r)
    host_us = (time.perf_counter() - t0) / 50 * 1e6
    res = np.abs(b.matvec(s.solve(r)) - r).max() / np.abs(r).max()
    print(f"n={n} d={d} ranks={s.ranks} split={s.split} L={s.plan.L} build={build:.2f}s "
          f"device-tensor solve {dev_us:.1f} us, numpy solve {host_us:.1f} us, rel res {res:.1e}")
