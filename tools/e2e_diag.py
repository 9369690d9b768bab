"""Per-call timing of the public numpy path (plan_solve(plan, numpy)) -- pinning and
pool behaviour of the host staging.  Usage: python tools/e2e_diag.py c4 [calls]"""
import ctypes
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1108_4181_b200 as btd  # noqa: E402
from paper_1108_4181_b200 import _native, configs, dichotomy  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 6
torch.cuda.set_device(0)
d, lo, up, F = configs.generate(name)
ranks, split = bench.plan_params(name, 1)
plan = btd.plan_build_arrays(torch.from_numpy(d).cuda(), torch.from_numpy(lo).cuda(), torch.from_numpy(up).cuda(),
                             ranks, split=split)
del d, lo, up
if len(sys.argv) > 3 and sys.argv[3] == "pinned":  # input in cudaHostAlloc memory instead of registered numpy
    F = btd.pinned_array(F)
lib = _native.load()
for i in range(calls):
    t0 = time.perf_counter()
    x = btd.plan_solve(plan, F)
    t1 = time.perf_counter()
    was = ctypes.c_int(0)
    lib.btd_host_pin(ctypes.c_void_p(F.ctypes.data), 8, ctypes.byref(was))
    print(f"{name} call {i}: {1e3 * (t1 - t0):8.1f} ms  ({F.shape[2] / (t1 - t0):8.1f} RHS/s)  F pinned={was.value} "
          f"pool={ {k: len(v) for k, v in dichotomy._pool.items()} }", flush=True)
# raw library call on the same buffers (no Python staging)
X = np.empty_like(F)
for i in range(2):
    t0 = time.perf_counter()
    _native.check(lib.btd_plan_solve_host(plan.handle, ctypes.c_void_p(F.ctypes.data), ctypes.c_void_p(x.ctypes.data),
                                          F.shape[2], None))
    print(f"{name} raw btd_plan_solve_host (pinned F, pinned X): {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
# per-chunk timeline of one more raw call (BTD_HOST_TRACE is read once per process)
