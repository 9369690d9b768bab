"""K=1 band-solve latency vs second-level split (chain length)."""
import numpy as np
import torch
from paper_1108_4181_b200 import bands

n, d = 129024, 16
rng = np.random.default_rng(0)
bd = np.zeros((2 * d + 1, n))
for off in range(1, d + 1):
    v = rng.uniform(-1, 1, n - off)
    bd[d + off, : n - off] = v
    bd[d - off, off:] = v
bd[d] = np.abs(bd).sum(axis=0) + 1.0
b = bands.BandMatrix(n, d, bd, symmetric=True)
r = torch.from_numpy(rng.standard_normal(n)).cuda()
for split in (63, 126, 252, 504, 1008):
    s = bands.BandSolver(b, split=split)
    for _ in range(5):
        s.solve(r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        s.solve(r)
    e1.record(); torch.cuda.synchronize()
    print(f"split={split} L={s.plan.L} K=1 solve {e0.elapsed_time(e1) / 200 * 1e3:.1f} us")
    for k in (2, 16):
        rk = torch.from_numpy(rng.standard_normal((n, k))).cuda()
        for _ in range(3):
            s.solve(rk)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(50):
            s.solve(rk)
        e1.record(); torch.cuda.synchronize()
        print(f"   K={k}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
