"""Plan build of one config (for an ncu launch list of the preprocessing kernels).
Usage: python tools/build_profile.py c1"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1108_4181_b200 import configs, plan_build_arrays  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
torch.cuda.set_device(0)
d, lo, up, _ = configs.generate(name, device="cuda", k=0)
ranks, split = bench.plan_params(name, 1)
torch.cuda.synchronize()
t0 = time.perf_counter()
plan = plan_build_arrays(d, lo, up, ranks, split=split)
torch.cuda.synchronize()
print(f"{name} plan_build {time.perf_counter() - t0:.3f} s", flush=True)
