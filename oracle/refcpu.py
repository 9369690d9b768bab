"""REFERENCE CPU ARM -- BASELINE INFRASTRUCTURE ONLY.

Times the unmodified reference package (oracle/_ref, built from
/root/reference/pkg by oracle/build_ref.sh with its own setup.py) -- its public
``blocktri.dichotomy.plan_build`` / ``plan_solve`` (dichotomy.py:318-390) --
on a bounded sample of a BASELINE.json config, on the host cores.  The
reference's kernels are single-threaded (``_kernels.pyx`` has no nogil/prange),
so "all the host threads it can use" = W worker processes, each holding the
same plan (built once, untimed) and solving its own slice of the K columns
(columns are independent in the algorithm).  A step is one solve of all K
columns of the sample; its time is the wall clock from dispatch to the last
worker's return.

Kernel backend per block order: the compiled Cython kernels for M <= 64; the
reference's numpy backend above (the Cython inner products are strided loops,
``_kernels.pyx:97-108``, ~10x slower there than numpy ``@``).

Used by bench.py's ``--impl reference`` and ``cpu_baseline`` legs only.
"""

from __future__ import annotations

import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.path.join(HERE, "_ref")

# (block rows, ranks) of the sample per config: the same operator family at
# full M and K over N_s block rows (solve cost is linear in N); c3: the S of the
# same 64-subdomain DD on a 512 x 2048 grid (M = 512), scaled by (512/2048)^2.
SAMPLE = {
    "c0": dict(ns=512, ranks=4),
    "c1": dict(ns=256, ranks=8),
    "c2": dict(ns=1024, ranks=8),
    "c3": dict(ns=63, ranks=8, mx=512),
    "c4": dict(ns=65536, ranks=8),
}


def available() -> bool:
    return os.path.isfile(os.path.join(REF, "blocktri", "dichotomy.py"))


def backend_for(m):
    return "compiled" if m <= 64 else "python"


def _inputs(name, cols):
    sys.path.insert(0, ROOT)
    import numpy as np

    from paper_1108_4181_b200 import configs

    cfg = configs.CONFIGS[name]
    s = SAMPLE[name]
    if cfg["kind"] == "strip":
        d, lo, up, f = configs.strip_numpy(s["ns"], cfg["m"], cfg["k"], cfg["shift"], 0)
    elif cfg["kind"] == "schur":
        from paper_1108_4181_b200 import schur

        d, lo, up = schur.schur_blocks_numpy(s["mx"], cfg["nz"] // 4, cfg["nsub"])
        f = np.random.default_rng(0).standard_normal((d.shape[0], s["mx"], cfg["k"]))
    else:
        d, lo, up, f = configs.dominant_numpy(s["ns"], cfg["m"], cfg["k"], 0)
    return d, lo, up, np.ascontiguousarray(f[:, :, cols[0]:cols[1]])


def _worker(name, c0, c1):
    """Child process (``python refcpu.py --worker name c0 c1``): build the plan,
    then one timed solve per ``go`` line on stdin; replies on stdout."""
    sys.path.insert(0, REF)
    from blocktri import backend, core, dichotomy

    d, lo, up, f = _inputs(name, (c0, c1))
    plan = dichotomy.plan_build(core.BlockTriMatrix(d, lo, up), SAMPLE[name]["ranks"])
    out = sys.stdout
    out.write(f"ready {backend.backend_name()}\n")
    out.flush()
    for line in sys.stdin:
        if line.strip() != "go":
            break
        t0 = time.perf_counter()
        dichotomy.plan_solve(plan, f)
        out.write(f"done {time.perf_counter() - t0}\n")
        out.flush()


class RefSample:
    """W reference processes over column slices of config ``name``'s sample."""

    def __init__(self, name, workers=None):
        import subprocess

        sys.path.insert(0, ROOT)
        from paper_1108_4181_b200 import configs

        if not available():
            raise RuntimeError("oracle/_ref missing (run oracle/build_ref.sh where /root/reference exists)")
        cfg = configs.CONFIGS[name]
        self.name, self.cfg = name, cfg
        k = cfg["k"]
        w = min(workers or os.cpu_count() or 1, k)
        bounds = [(i * k // w, (i + 1) * k // w) for i in range(w)]
        self.m = SAMPLE[name].get("mx", cfg["m"])
        env = {"BLOCKTRI_BACKEND": backend_for(self.m), "OPENBLAS_NUM_THREADS": "1", "OMP_NUM_THREADS": "1",
               "MKL_NUM_THREADS": "1"}
        penv = dict(os.environ, **env)
        self.procs = [subprocess.Popen([sys.executable, os.path.abspath(__file__), "--worker", name, str(b[0]),
                                        str(b[1])], stdin=subprocess.PIPE, stdout=subprocess.PIPE, env=penv,
                                       text=True, bufsize=1) for b in bounds]
        self.backend = None
        for p in self.procs:
            line = p.stdout.readline().split()
            if not line or line[0] != "ready":
                self.close()
                raise RuntimeError(f"reference worker failed to start ({name})")
            self.backend = line[1]
        self.workers = w
        s = SAMPLE[name]
        self.scale = (s["ns"] / cfg["n"]) if cfg["kind"] != "schur" else (self.m / cfg["m"]) ** 2
        self.sample = (f"unmodified reference blocktri 0.1.0 (oracle/_ref) plan_solve, {self.backend} kernels, "
                       f"{w} processes x 1 thread over column slices of K={k}; "
                       + (f"S of the same 64-subdomain DD on a {self.m} x 2048 grid (M = {self.m}, N = 63), "
                          f"RHS/s scaled by ({self.m}/{cfg['m']})^2 (solve flops ~ N M^2 K)"
                          if cfg["kind"] == "schur" else
                          f"N={s['ns']} of {cfg['n']} block rows, P={s['ranks']}, RHS/s scaled by N_s/N "
                          "(solve cost is linear in N)"))

    def step(self):
        """(RHS/s of the whole sample over all workers, wall seconds); the per-worker
        solve times of the step are kept in ``last_worker_s``."""
        t0 = time.perf_counter()
        for p in self.procs:
            p.stdin.write("go\n")
            p.stdin.flush()
        self.last_worker_s = []
        for p in self.procs:
            line = p.stdout.readline()
            if not line.startswith("done"):
                raise RuntimeError("reference worker died")
            self.last_worker_s.append(float(line.split()[1]))
        t = time.perf_counter() - t0
        return self.cfg["k"] / t * self.scale, t

    def one_core_value(self):
        """RHS/s of ONE reference process (its columns over its own solve time), i.e. the
        reference's single-threaded throughput on one core of this host."""
        k = self.cfg["k"]
        cols = [(i + 1) * k // self.workers - i * k // self.workers for i in range(self.workers)]
        return sum(c / t for c, t in zip(cols, self.last_worker_s)) / self.workers * self.scale

    def close(self):
        for p in getattr(self, "procs", []):
            try:
                p.stdin.write("stop\n")
                p.stdin.close()
            except (BrokenPipeError, OSError, ValueError):
                pass
        for p in getattr(self, "procs", []):
            try:
                p.wait(timeout=30)
            except Exception:
                p.kill()
        self.procs = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


if __name__ == "__main__" and len(sys.argv) == 5 and sys.argv[1] == "--worker":
    _worker(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
