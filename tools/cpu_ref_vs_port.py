"""The CPU baseline is a C port of the reference algorithm (oracle/blocktri_oracle.c, all host
threads); this relates it to the reference package itself (its compiled Cython backend and its
numpy backend), built from /root/reference in a scratch dir, on the same bounded samples.
Run in the build container (the reference cannot travel to the GPU box)."""
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden")]
import make_golden  # noqa: E402  (builds the reference into /tmp/blocktri_ref_golden)
from paper_1108_4181_b200 import configs  # noqa: E402
import coracle  # noqa: E402

SAMPLES = {"c0": (512, 8, 32, 4), "c1": (256, 256, 256, 8), "c2": (512, 64, 1024, 8), "c4": (65536, 16, 64, 16)}


def time_ref(backend, d, lo, up, f, P):
    code = f"""
import sys, time, numpy as np
sys.path.insert(0, {str(make_golden.SCRATCH / 'src')!r})
from blocktri import core, dichotomy
d, lo, up, f = (np.load(p) for p in {[f'/tmp/_cs_{n}.npy' for n in 'dluf']!r})
A = core.BlockTriMatrix(d, lo, up)
plan = dichotomy.plan_build(A, {P})
best = 1e9
for _ in range(2):
    t0 = time.perf_counter(); dichotomy.plan_solve(plan, f); best = min(best, time.perf_counter() - t0)
print(best)
"""
    for n, a in zip("dluf", (d, lo, up, f)):
        np.save(f"/tmp/_cs_{n}.npy", a)
    env = dict(os.environ, BLOCKTRI_BACKEND=backend, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True)
    return float(out.stdout.strip().splitlines()[-1])


if __name__ == "__main__":
    make_golden.build_reference()
    for name in sys.argv[1:] or list(SAMPLES):
        n, m, k, P = SAMPLES[name]
        cfg = configs.CONFIGS[name]
        if cfg["kind"] == "strip":
            d, lo, up, f = configs.strip_numpy(n, m, k, cfg["shift"], 0)
        else:
            d, lo, up, f = configs.dominant_numpy(n, m, k, 0)
        cp = coracle.CPlan(d, lo, up, P)
        cp.solve(f)
        t0 = time.perf_counter(); cp.solve(f); tport = time.perf_counter() - t0
        tc = time_ref("compiled", d, lo, up, f, P)
        tp = time_ref("python", d, lo, up, f, P)
        print(f"{name} sample N={n} M={m} K={k} P={P}: C port {coracle.threads()} threads {tport:.3f} s | "
              f"reference Cython (1 thread) {tc:.3f} s | reference numpy (1 BLAS thread) {tp:.3f} s | "
              f"port speed-up vs Cython {tc / tport:.1f}x", flush=True)
