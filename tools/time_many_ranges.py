import time, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
from paper_1108_4181_b200 import BlockTriMatrix, configs, plan_build, plan_solve
import coracle
for n, split in [(140000, 17000), (40000, 5000)]:
    d, lo, up, f = configs.dominant_numpy(n, 2, 3, seed=1)
    t0 = time.time(); plan = plan_build(BlockTriMatrix(d, lo, up), 4, split=split); t1 = time.time()
    x = plan_solve(plan, f); t2 = time.time()
    ref = coracle.CPlan(d, lo, up, 4).solve(f); t3 = time.time()
    print(n, split, plan.nranges, 'build %.1f solve %.1f oracle %.1f' % (t1 - t0, t2 - t1, t3 - t2), flush=True)
