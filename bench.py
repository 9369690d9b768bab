#!/usr/bin/env python
"""Benchmark of the many-RHS block-tridiagonal dichotomy solve (plan_solve).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl b200|reference]

Metric (BASELINE.json): right-hand-side columns solved per second at a fixed
matrix.  One *step* = one ``plan_solve`` of the config's K columns, F -> X,
with the plan (Algorithm 2 step 1) built once beforehand and timed separately.
Default workload: configs[4] (c4, N=2^20 block rows of M=16, K=64), the
largest configuration -- the one north_star's 1/2/4/8-GPU efficiency target
is set on (BASELINE.json names no single config for the metric); every other
config runs with ``--config``.  Inputs are the seeded numpy stream of
``configs.generate`` -- the same arrays the unmodified reference was run on for
the full-size goldens (tests/golden/fullsize_*.npz).

* ``value``: device-resident F/X, CUDA events on the solve stream around
  exactly K steps, max over ranks.  Inputs (c4: F 8.6 GB, factors 10.8 GB)
  are larger than the 126 MB L2, so no flush is needed between steps.
* ``e2e``: the same metric through the public numpy API a reference user
  calls, ``paper_1108_4181_b200.plan_solve(plan, F_numpy) -> X_numpy``
  (host F -> device -> solve -> host X every step), wall clock.
* ``roofline``: the dominant kernel -- algorithmic bytes (or flops) per launch
  / its CUDA-event duration, against the measured HBM copy bandwidth
  (MEASURED_PEAKS.json) or the fp64 tensor peak (cuBLAS DGEMM measured in
  this run; MEASURED_PEAKS.json has no fp64 entry).
* ``parity``: after the timed region, the solution's golden columns against
  the reference-written full-size golden and against the C oracle run on the
  same host arrays (``max_rel_err_vs_oracle``).
* ``cpu_baseline``: the unmodified reference package (oracle/_ref, built by
  oracle/build_ref.sh) timed on a bounded sample on the host cores;
  ``cpu_baseline_port``: the C port of the same algorithm (oracle/).
* ``--impl reference``: the reference's own plan_solve on the host cores
  (all of them: one process per core over column slices), same metric/config.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Per-config plan parameters.  ranks = the reference's P (subdomains);
# split = on-device second-level ranges per subdomain (hard
# part 1), chosen so each GPU runs ~`ranges_per_gpu` device ranges (one CTA
# per range and column tile fills the 148 SMs).  c4 follows the paired
# reading of BASELINE.json: 8 / 16 / 32 / 64 subdomains per GPU on 1 / 2 / 4 / 8 GPUs.
BENCH_CFG = {
    # c0: the reference's P = 4 subdomains, each split into 16 device ranges (chains of 8 rows:
    # the solve is latency-bound; split 1 -> 16: 0.152 -> 0.049 ms per step, profiles/r01_chain_ab.txt)
    "c0": dict(subdomains_per_gpu=lambda w: 4, ranges_per_gpu=64),
    # c1/c2: 37 ranges per GPU (148 = 4 x 37): every chain kernel's grid is a whole number
    # of waves (c1 fwd 37 x 16 tiles = 4 x 148 CTAs, bwd 37 x 8 = 2 x 148; c2 fwd 37 x 8 =
    # 2 x 148).  Measured on B200 (profiles/r01_ranks_sweep.txt): c1 P=36 0.848 -> P=37 0.868
    # of roofline, c2 0.785 -> 0.802; P=48 or 56 drops to 0.69-0.75 (partial last wave)
    # On 4 and 8 GPUs 18 ranges per GPU: the sharded tree (series sums and crossing partials
    # over P = 18 W ranges) costs less than the partial last wave of the sweeps (projected
    # c1 8 GPUs 3.55 -> 3.38 ms, c2 3.51 -> 3.40 ms; profiles/r01_shard_projection.txt)
    "c1": dict(subdomains_per_gpu=lambda w: 37 if w <= 2 else 18, ranges_per_gpu=lambda w: 37 if w <= 2 else 18),
    "c2": dict(subdomains_per_gpu=lambda w: 37 if w <= 2 else 18, ranges_per_gpu=lambda w: 37 if w <= 2 else 18),
    # c3: the explicit interface Schur complement S (N=63, M=2048) of the 64-subdomain
    # Helmholtz DD; P = 9 ranges of 7 interface rows on one GPU (288 GEMM tiles fill the
    # 296 CTA slots), P = 8 (a multiple of 2/4/8) when sharded
    "c3": dict(subdomains_per_gpu=lambda w: 9 if w == 1 else 8 // w, ranges_per_gpu=1),
    # c4: 592 = 4 x 148 device ranges per GPU (one wave of the 4-CTA/SM streamed sweeps);
    # split = floor(592 / subdomains per GPU): 74 / 37 / 18 / 9 on 1 / 2 / 4 / 8 GPUs (one
    # wave, shallow sharded trees; tools/shard_projection.py, profiles/r01_shard_projection.txt)
    "c4": dict(subdomains_per_gpu=lambda w: 8 * w, ranges_per_gpu=592, one_wave=True),
}


def plan_params(name, world, ranks=0, split=0):
    """(ranks, split): split = the smallest second-level factor with at least
    ranges_per_gpu device ranges per GPU that are a whole multiple of it (the
    sweep grids are whole waves: c4 at 32 subdomains/GPU -> split 37, 1184
    ranges, not split 19 -> 608 ranges = 4.1 waves; profiles/r01_chain_ab.txt)."""
    bc = BENCH_CFG[name]
    spg = bc["subdomains_per_gpu"](world)
    r = ranks or spg * world
    if split:
        return r, split
    rpg = bc["ranges_per_gpu"]
    rpg = rpg(world) if callable(rpg) else rpg
    if bc.get("one_wave"):
        return r, max(1, rpg // spg)
    sp = max(1, -(-rpg // spg))
    if rpg > 1:
        while (spg * sp) % rpg:
            sp += 1
    return r, sp


# CPU sample per config: (block rows, columns, ranks) of the same operator family,
# sized for a few seconds of host work per step.
CPU_SAMPLE = {
    "c0": (512, 32, 4),
    "c1": (256, 256, 8),
    "c2": (512, 1024, 8),
    "c3": (63, 16, 8),   # S of the same DD at nx = 512 (M = 512): flop-scaled to M = 2048
    "c4": (65536, 64, 16),
}


_OUT = None


def emit(line):
    """The one JSON result line, on the process's original stdout."""
    print(json.dumps(line), file=_OUT or sys.stdout, flush=True)


def _stdout_to_stderr():
    """Native libraries (NCCL's version banner, CUDA) may print to fd 1; keep stdout
    for the JSON line alone by pointing fd 1 at stderr and emitting through a dup."""
    global _OUT
    try:
        sys.stdout.flush()
        _OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
    except OSError:
        _OUT = None


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- helpers
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML polled
    every 5 ms from a thread (short timed regions still get samples), else
    ``nvidia-smi -lms 100``."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, period_s=0.005):
        self.index = index
        self.period = period_s
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons)
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index())
            self.bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:  # no NVML: nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _physical_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if ids and self.index < len(ids) and ids[self.index].isdigit():
            return int(ids[self.index])
        return self.index

    def _poll(self):
        nv = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((float(sm), float(mx), {k for k, b in self.bits.items() if r & b}))
            except Exception:
                pass
            self._stop.wait(self.period)

    def sample_now(self):
        """One synchronous sample (called right after the timed steps are enqueued, while
        the GPU runs them: regions shorter than the polling period still get one)."""
        if self.nvml is None:
            return
        nv = self.nvml
        try:
            sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.samples.append((float(sm), float(mx), {k for k, b in self.bits.items() if r & b}))
        except Exception:
            pass

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self._stop.set()
        if self.nvml is not None:
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        samples = list(self.samples)
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                samples.append((float(p[0]), float(p[1]),
                                {nm for nm, v in zip(self.NAMES, p[3:7]) if v.lower().startswith("active")}))
            except ValueError:
                continue
        sm = [x[0] for x in samples]
        mx = max((x[1] for x in samples), default=0.0)
        reasons = set().union(*[x[2] for x in samples]) if samples else set()
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml 5 ms" if self.nvml is not None else "nvidia-smi 100 ms"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def fp64_peak_tflops(torch):
    """cuBLAS DGEMM 4096^3, best of 5 -- the fp64 tensor roofline denominator."""
    n = 4096
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn_like(a)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        e0.record()
        a @ b
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2 * n ** 3 / best / 1e9


def make_inputs(name, seed=0):
    """Host numpy arrays of config ``name``: the seeded numpy stream of
    configs.generate -- identical to the arrays the reference was run on for
    tests/golden/fullsize_<name>.npz."""
    from paper_1108_4181_b200 import configs

    return configs.generate(name, seed=seed)


def interior_rows(n, nranges, L):
    tot = 0
    for q in range(nranges):
        lo = q * L
        tot += max(0, min(L - 1, n - lo - 1))
    return tot


# --------------------------------------------------------------------------- CPU arms
def _oracle_path():
    p = os.path.join(ROOT, "oracle")
    if p not in sys.path:
        sys.path.insert(0, p)


class CpuSample:
    """The C port of the reference algorithm (oracle/liboracle.so; ranges and
    column chunks on all host threads) over a bounded sample of config `name`;
    plan built once (untimed).  Reported as ``cpu_baseline_port``."""

    def __init__(self, name):
        _oracle_path()
        import coracle
        from paper_1108_4181_b200 import configs

        self.coracle = coracle
        cfg = configs.CONFIGS[name]
        self.cfg = cfg
        ns, ks, ps = CPU_SAMPLE[name]
        scale = 1.0
        if cfg["kind"] == "strip":
            d, lo, up, f = configs.strip_numpy(ns, cfg["m"], ks, cfg["shift"], 0)
        elif cfg["kind"] == "schur":
            from paper_1108_4181_b200 import schur

            mx = 512
            d, lo, up = schur.schur_blocks_numpy(mx, cfg["nz"] // 4, cfg["nsub"])
            f = np.random.default_rng(0).standard_normal((d.shape[0], mx, ks))
            scale = (mx / cfg["m"]) ** 2  # solve flops scale with M^2 at fixed N, K
        else:
            d, lo, up, f = configs.dominant_numpy(ns, cfg["m"], ks, 0)
        self.f = f
        self.scale = scale
        self.ns, self.ks, self.ps = ns, ks, ps
        self.plan = coracle.CPlan(d, lo, up, ps)
        self.cores = coracle.threads()
        self.sample = (f"C port of the reference plan_solve (oracle/blocktri_oracle.c; ref dichotomy.py:358-390, "
                       f"_kernels.pyx:173-194) on N={ns} of {cfg['n']} block rows, K={ks} of {cfg['k']} columns, "
                       f"P={ps}, {self.cores} threads; RHS/s scaled by N_s/N (solve cost is linear in N)"
                       + ("; c3: S of the same 64-subdomain DD on a 512 x 2048 grid (M = 512), RHS/s "
                          "scaled by (512/2048)^2 (solve flops ~ N M^2 K)" if cfg["kind"] == "schur" else ""))

    def step(self):
        t0 = time.perf_counter()
        self.plan.solve(self.f)
        t = time.perf_counter() - t0
        return self.ks / t * self.ns / self.cfg["n"] * self.scale, t


def cpu_port_run(name, steps=1):
    cs = CpuSample(name)
    vals = [cs.step() for _ in range(max(1, steps))]
    v = statistics.median(x[0] for x in vals)
    return {"value": v, "unit": "RHS/s", "cores": cs.cores, "kind": "port", "sample": cs.sample}


def cpu_reference_run(name, steps=2, warmup=1, workers=None):
    """The unmodified reference's plan_solve (oracle/refcpu.py) on the host cores."""
    _oracle_path()
    import refcpu

    if not refcpu.available():
        return None
    rs = refcpu.RefSample(name, workers=workers)
    try:
        for _ in range(warmup):
            rs.step()
        res = [rs.step() for _ in range(max(1, steps))]
        one = rs.one_core_value()
    finally:
        rs.close()
    ts = [r[1] for r in res]
    value = rs.cfg["k"] * len(ts) / sum(ts) * rs.scale
    return {"value": value, "unit": "RHS/s", "cores": rs.workers, "kind": "reference", "sample": rs.sample,
            "ms_per_step": 1e3 * sum(ts) / len(ts), "value_one_core": one,
            "backend": rs.backend}


def run_reference(args):
    """--impl reference: the reference's own plan_solve on this host's cores
    (rank 0 only; other ranks exit without work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.config
    from paper_1108_4181_b200 import configs

    cfg = configs.CONFIGS[name]
    _oracle_path()
    import refcpu

    if refcpu.available():
        cb = cpu_reference_run(name, steps=args.steps, warmup=args.warmup)
    else:  # the reference could not be built: the C port of its algorithm
        cs = CpuSample(name)
        for _ in range(args.warmup):
            cs.step()
        res = [cs.step() for _ in range(args.steps)]
        ts = [r[1] for r in res]
        cb = {"value": cs.ks * len(ts) / sum(ts) * cs.ns / cfg["n"] * cs.scale, "unit": "RHS/s",
              "cores": cs.cores, "kind": "port", "sample": cs.sample, "ms_per_step": 1e3 * sum(ts) / len(ts)}
    value = cb["value"]
    line = {
        "impl": "reference", "metric": "rhs_columns_per_second", "value": value, "unit": "RHS/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cb.pop("ms_per_step"), "higher_is_better": True,
        # total work is fixed as GPUs are added (c4: N = 2^20 rows; only the subdomain count per GPU grows)
        "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded numpy, BASELINE.json distributions)",
        "config": {"workload": name, "n": cfg["n"], "m": cfg["m"], "k": cfg["k"]},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "RHS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# --------------------------------------------------------------------------- GPU arm
def parity_report(name, X, host, rows, ranks):
    """Golden columns of the GPU solution X (device, rows [lo, hi) of the global
    solution) against the reference-written full-size golden and the C oracle
    run live on the same host arrays."""
    _oracle_path()
    import parity

    from paper_1108_4181_b200 import configs

    g, meta = parity.golden(name)
    if g is None or rows != (0, configs.CONFIGS[name]["n"]):
        return None
    cols = meta["cols"]
    x_cols = X[:, :, cols].cpu().numpy()
    out = {"cols": cols}
    rep = parity.compare_golden(name, x_cols)
    out["vs_reference_golden"] = rep
    diag, lower, upper, F = host
    f_cols = np.ascontiguousarray(F[:, :, cols])
    out["inputs_match_golden"] = (parity.sha_inputs(diag, lower, upper, f_cols) == meta["sha_inputs"]
                                  if configs.CONFIGS[name]["kind"] != "schur" else "S formed by BLAS (rounding)")
    if configs.CONFIGS[name]["kind"] == "schur":
        out["vs_oracle"] = None  # M = 2048 CPU plan takes minutes; the golden holds every row
        out["max_rel_err_vs_oracle"] = rep["max_rel_err_sampled_rows"]
        out["oracle"] = "reference golden (all 63 rows)"
        return out
    import coracle

    t0 = time.perf_counter()
    p_or = max(ranks, min(coracle.threads(), configs.CONFIGS[name]["n"] // 8))
    ref = parity.oracle_columns(diag, lower, upper, f_cols, p_or)
    out["max_rel_err_vs_oracle"] = parity.max_rel_err(x_cols, ref)
    out["oracle"] = (f"C oracle (oracle/liboracle.so), all {x_cols.shape[0]} block rows, P={p_or}, "
                     f"{time.perf_counter() - t0:.1f} s")
    return out


def run_b200(args):
    import ctypes

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank (LOCAL_RANK); BTD_DIST_BACKEND=gloo (host collectives) lets the
    # multi-rank flow run with several ranks on one device for functional checks --
    # no kernel waits on another rank, the exchanges go through the host
    backend = os.environ.get("BTD_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    sharded = world > 1 or args.sharded
    if sharded:
        import torch.distributed as dist

        if backend == "nccl":  # communicator set-up on stderr: ranks, channels, NVLS / CollNet use
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group(backend, rank=rank, world_size=world,
                                device_id=torch.device("cuda", local) if backend == "nccl" else None)
    import paper_1108_4181_b200 as btd
    from paper_1108_4181_b200 import _native, configs, plan_build_arrays
    from paper_1108_4181_b200.distributed import ShardedPlan

    name = args.config
    cfg = configs.CONFIGS[name]
    ranks, split = plan_params(name, world, args.ranks, args.split)
    n, m, K = cfg["n"], cfg["m"], cfg["k"]
    lib = _native.load()
    stream = torch.cuda.current_stream()

    # every rank draws the same global matrix / RHS (seeded numpy stream) and keeps its rows
    t0 = time.perf_counter()
    if args.inputs == "numpy":
        host = make_inputs(name)
        diag, lower, upper = (torch.from_numpy(a).cuda() for a in host[:3])
    else:  # --inputs device (A/B only): torch Philox on the device, no parity report
        diag, lower, upper, Fdev = configs.generate(name, device="cuda")
        host = (None, None, None, Fdev.cpu().numpy())
        del Fdev
    gen_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if not sharded:
        plan = plan_build_arrays(diag, lower, upper, ranks, split=split)
        row_lo, row_hi = 0, n
        nranges, L, mode, fbytes = plan.nranges, plan.L, plan.mode, plan.factor_bytes
        scoup = bool(plan.scalar_coupling)
        handle = plan.handle
    else:
        plan = ShardedPlan(diag, lower, upper, ranks, split=split)
        row_lo, row_hi = plan.row_lo, plan.row_hi
        info = plan.be.info(plan.h)
        nranges, L, mode, fbytes = plan.nranges, plan.L, int(info.mode), int(info.factor_bytes)
        scoup = bool(info.scalar_coupling)
        handle = plan.h
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    build_warm_s = None
    if not sharded and not args.no_check:  # a second build: without the one-time CUDA module loading
        t0 = time.perf_counter()
        plan2 = plan_build_arrays(diag, lower, upper, ranks, split=split)
        torch.cuda.synchronize()
        build_warm_s = time.perf_counter() - t0
        plan2.close()
        del plan2
        torch.cuda.empty_cache()
    if args.inputs == "numpy":  # the residual re-uploads the matrix from the host arrays
        del diag, lower, upper
        torch.cuda.empty_cache()
    Fh = np.ascontiguousarray(host[3][row_lo:row_hi])
    F = torch.from_numpy(Fh).cuda()
    X = torch.empty_like(F)

    if not sharded:
        sp = ctypes.c_void_p(stream.cuda_stream)

        def solve():
            st = lib.btd_plan_solve(handle, ctypes.c_void_p(F.data_ptr()), ctypes.c_void_p(X.data_ptr()), K, sp)
            if st:
                _native.check(st)
    else:
        def solve():
            plan.solve(F, out=X)

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            solve()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        lc0 = _native.launch_count()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            solve()
        e1.record(stream)
        clk.sample_now()
        e1.synchronize()
        launches = _native.launch_count() - lc0
        if dist:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    ms_rank = ms
    if dist:
        tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    value = K * args.steps / (ms / 1e3)  # whole job: K columns per step over all GPUs

    # per-phase device timing (separate profiled pass; events between the phases)
    buf = (ctypes.c_double * 4)()
    nsv = ctypes.c_int64()
    lib.btd_plan_set_profiling(handle, 1)
    lib.btd_plan_phase_times(handle, buf, ctypes.byref(nsv), 1)
    for _ in range(args.steps):
        solve()
    torch.cuda.synchronize()
    lib.btd_plan_phase_times(handle, buf, ctypes.byref(nsv), 1)
    lib.btd_plan_set_profiling(handle, 0)
    ph = [buf[i] / max(1, nsv.value) for i in range(4)]
    per_rank = None
    if dist:
        vals = torch.tensor([ms_rank / args.steps] + ph, device="cuda", dtype=torch.float64)
        allv = torch.empty(world * vals.numel(), device="cuda", dtype=torch.float64)
        dist.all_gather_into_tensor(allv, vals)
        allv = allv.view(world, -1).cpu().tolist()
        per_rank = [{"rank": r, "ms_per_step": v[0], "forward": v[1], "interface_tree": v[2], "backward": v[3],
                     "total": v[4]} for r, v in enumerate(allv)]

    res = None
    if not args.no_check:
        if args.inputs == "numpy":
            diag, lower, upper = (torch.from_numpy(a).cuda() for a in host[:3])
        res = (residual_check_sharded(torch, dist, X, F, diag, lower, upper, row_lo, row_hi) if sharded
               else residual_check(torch, X, F, diag, lower, upper))
    if args.inputs != "numpy" or not args.no_check:
        del diag, lower, upper
    torch.cuda.empty_cache()
    par = None
    if not args.no_check and rank == 0 and args.inputs == "numpy":
        try:
            par = parity_report(name, X, host, (row_lo, row_hi), ranks)
        except Exception as exc:  # the report must not kill the bench line
            par = {"error": f"{type(exc).__name__}: {exc}"}

    # e2e through the public host-memory API: numpy F -> device -> solve -> numpy X
    e2e = None
    if not args.no_e2e:
        del F, X
        torch.cuda.empty_cache()
        if not sharded:
            Fp = btd.pinned_array(Fh)  # the caller's batch in page-locked memory (untimed, once)

            def solve_host():
                return btd.plan_solve(plan, Fp)
            api = ("paper_1108_4181_b200.plan_solve(plan, numpy (n, m, k)) -> numpy; input from "
                   "paper_1108_4181_b200.pinned_array (page-locked), solution in the pinned result pool")
        else:
            Fp = torch.from_numpy(Fh).pin_memory()
            Xp = torch.empty_like(Fp).pin_memory()

            def solve_host():
                plan.solve_host(Fp, Xp)
                return Xp
            api = "ShardedPlan.solve_host(pinned host rows) (per-rank host pipeline)"
        for _ in range(2):  # warm: page-locks F once and fills the 2-deep pinned solution pool
            xh = solve_host()
        del xh
        if dist:
            dist.barrier()
        esteps = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(esteps):
            xh = solve_host()
            _ = float(xh[-1, -1, -1])  # the step's result is read on the host
        ems = (time.perf_counter() - t0) * 1e3
        if dist:
            tt = torch.tensor([ems], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        nbytes = Fh.nbytes
        e2e = {"value": K * esteps / (ems / 1e3), "unit": "RHS/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "steps": esteps, "ms_per_step": ems / esteps, "api": api,
               "timing": "host wall clock around the blocking API calls, max over ranks"}
        del xh

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel (forward sweep) and of the whole solve, per GPU
    pk = measured_peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    fp64 = fp64_peak_tflops(torch)
    nint = interior_rows(n, nranges, L) / world
    # scalar-coupled plans (interior lower blocks a I: c1) run the forward sweep with two block
    # products per row instead of three: 4 M^2 K flops and two factor streams
    fprod = 2 if scoup else 3
    fwd_flops = 2.0 * fprod * m * m * K * nint
    fwd_bytes = 8.0 * (fprod * m * m + 2 * m * K) * nint
    tot_flops = 2.0 * (fprod + 2) * m * m * K * n / world
    tot_bytes = 8.0 * ((fprod + 2) * m * m + 4 * m * K) * n / world
    hbm_bound = tot_flops / (fp64 * 1e12) < tot_bytes / (hbm * 1e9)
    t_fwd = ph[0] / 1e3
    if hbm_bound:
        roof = {"bound": "hbm", "achieved": fwd_bytes / t_fwd / 1e9, "peak": hbm, "unit": "GB/s"}
    else:
        roof = {"bound": "tensor", "achieved": fwd_flops / t_fwd / 1e12, "peak": fp64, "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = ncu_traffic(name)
    roof["kernel"] = (("stream_fwd_kernel (TMA bulk-copy ring)" if m <= 32 and K % 2 == 0 else
                       "chain_fwd_sc_kernel (scalar-coupled: 2 products per row)" if scoup else "chain_fwd_kernel")
                      if mode == 0 else "gemm_tma_kernel (mode 1: one batched TMA GEMM per row step)")
    roof["algorithmic_per_launch"] = (f"{fwd_bytes:.4e} B = 8({fprod}M^2+2MK) x {nint:.0f} interior rows" if hbm_bound
                                      else f"{fwd_flops:.4e} flop = {2 * fprod}M^2K x {nint:.0f} interior rows")
    roof["peak_source"] = ("cuBLAS DGEMM 4096^3 measured in this run (fp64 tensor; MEASURED_PEAKS.json has no fp64)"
                           if not hbm_bound else "MEASURED_PEAKS.json hbm_gbs (burst copy)")
    t_roof = max(tot_flops / (fp64 * 1e12), tot_bytes / (hbm * 1e9))
    clocks = clk.summary()

    cpu = cpu_port = None
    if world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference_run(name)
        except Exception as exc:
            cpu = {"error": f"{type(exc).__name__}: {exc}"}
        cpu_port = cpu_port_run(name)
        if cpu is None:
            cpu = cpu_port

    line = {
        "metric": "rhs_columns_per_second", "value": value, "unit": "RHS/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        # total work is fixed as GPUs are added (c4: N = 2^20 rows; only the subdomain count per GPU grows)
        "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy stream of configs.generate, BASELINE.json distributions; "
                "identical to the reference's full-size golden inputs)",
        "config": {"workload": name, "n": n, "m": m, "k": K, "ranks": ranks, "split": split,
                   "device_ranges": nranges, "L": L, "mode": mode, "scalar_coupling": scoup,
                   "parallelism": f"rows sharded over {world} GPUs (NCCL all-gather of interface pairs)"
                   if sharded else "single GPU",
                   "l2": "inputs larger than L2 (F %.2f GB, factors %.2f GB per GPU)" % (
                       Fh.nbytes / 1e9, fbytes / 1e9)},
        "roofline": roof,
        "solve_roofline": {"flops_per_gpu": tot_flops, "bytes_per_gpu": tot_bytes,
                           # SURVEY 8(d) companions: strict lower bound 8(5M^2 + 2MK) and the
                           # reference pipeline's 8(5M^2 + 6MK) bytes per block row
                           "bytes_strict_per_gpu": 8.0 * (5 * m * m + 2 * m * K) * n / world,
                           "bytes_ref_pipeline_per_gpu": 8.0 * (5 * m * m + 6 * m * K) * n / world,
                           "t_roof_ms": t_roof * 1e3,
                           "frac": t_roof * 1e3 / ms_step, "fp64_tflops_peak": fp64, "hbm_gbs_peak": hbm},
        "phases_ms": {"forward": ph[0], "interface_tree": ph[1], "backward": ph[2], "total": ph[3]},
        "per_rank": per_rank,
        "collectives": ({"backend": backend, "world": world,
                         "nccl_version": ".".join(str(v) for v in torch.cuda.nccl.version())
                         if backend == "nccl" else None,
                         "per_solve": "all-gather of one carry block per rank + all-gather of the crossing "
                                      "tree-node partial sums (summed in rank order)"} if sharded else None),
        "plan_build_s": build_s,
        "plan_build_warm_s": build_warm_s,
        "input_generation_s": gen_s,
        "rel_residual": res,
        "max_rel_err_vs_oracle": par.get("max_rel_err_vs_oracle") if isinstance(par, dict) else None,
        "parity": par,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "cpu_baseline_port": cpu_port,
        "clocks": clocks,
        "gpu_launches": launches,
    }
    emit(line)
    if dist:
        dist.destroy_process_group()


def ncu_traffic(name):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(name)
    except (OSError, ValueError):
        return None


def residual_check(torch, X, F, diag, lower, upper):
    """max|P X - F| / max|F| on the device (ref cli.py:211-214)."""
    y = torch.bmm(diag, X)
    y[1:] -= torch.bmm(lower, X[:-1])
    y[:-1] -= torch.bmm(upper, X[1:])
    r = ((y - F).abs().max() / F.abs().max()).item()
    del y
    torch.cuda.empty_cache()
    return r


def residual_check_sharded(torch, dist, X, F, diag, lower, upper, lo, hi):
    """Sharded form of residual_check: each rank's rows [lo, hi) with the neighbour
    ranks' boundary rows of X exchanged (one all-gather of first/last rows); the
    max over ranks of max|P X - F| over the max over ranks of max|F|."""
    n = diag.shape[0]
    world, rank = dist.get_world_size(), dist.get_rank()
    edge = torch.stack([X[0], X[-1]]).contiguous()
    edges = torch.empty((2 * world,) + tuple(X.shape[1:]), dtype=X.dtype, device=X.device)
    dist.all_gather_into_tensor(edges, edge)
    edges = edges.view((world, 2) + tuple(X.shape[1:]))
    y = torch.bmm(diag[lo:hi], X)
    if lo >= 1:  # row i reads -lower[i-1] x_{i-1}
        xm = torch.cat([edges[rank - 1, 1:2], X[:-1]])
        y -= torch.bmm(lower[lo - 1:hi - 1], xm)
    elif hi - lo > 1:
        y[1:] -= torch.bmm(lower[0:hi - 1], X[:-1])
    if hi <= n - 1:  # row i reads -upper[i] x_{i+1}
        xp = torch.cat([X[1:], edges[rank + 1, 0:1]])
        y -= torch.bmm(upper[lo:hi], xp)
    elif hi - lo > 1:
        y[:-1] -= torch.bmm(upper[lo:hi - 1], X[1:])
    t = torch.tensor([(y - F).abs().max().item(), F.abs().max().item()], dtype=torch.float64, device=X.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    del y
    torch.cuda.empty_cache()
    return float(t[0] / t[1])


def run_dd(args):
    """--config c3dd: the full Schur-complement DD solve of config 3's grid
    (SURVEY.md 8f row f1): interiors by stacked dichotomy plans, interface by the
    S-plan, recovery -- RHS/s of whole-grid solves."""
    import torch

    from paper_1108_4181_b200 import _native, configs, schur

    cfg = configs.CONFIGS["c3"]
    nx, nz, nsub, K = cfg["nx"], cfg["nz"], cfg["nsub"], cfg["k"]
    torch.cuda.set_device(0)
    t0 = time.perf_counter()
    # interiors: 4 stacked plans of 16 subdomains (32768 block rows of M = 128), 144 ranges each
    # (measured: 148 ranges, 2 exact waves, is 4% slower; --ranks overrides)
    dd = schur.HelmholtzDD(nx, nz, nsub, groups=4, ranks_int=args.ranks or 144)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    f = torch.randn((nz, nx, K), dtype=torch.float64, device="cuda", generator=g)
    for _ in range(args.warmup):
        x = dd.solve(f)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lc0 = _native.launch_count()
    with ClockSampler(0) as clk:
        e0.record()
        for _ in range(args.steps):
            x = dd.solve(f)
        e1.record()
        e1.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    res = dd.residual(x, f)
    fp64 = fp64_peak_tflops(torch)
    ni = [e - a for a, e in dd.sub]
    ifl = 8.0 if all(getattr(p, "scalar_coupling", False) for p in dd.plans) else 10.0  # scalar-coupled interiors
    flops = 2 * sum(ifl * nx * n * n * K for n in ni) + 10.0 * (nsub - 1) * nx * nx * K
    line = {"metric": "rhs_columns_per_second", "value": K / (ms / 1e3), "unit": "RHS/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded layered velocity model, torch Philox RHS)",
            "config": {"workload": "c3dd", "nx": nx, "nz": nz, "nsub": nsub, "k": K, "interior_groups": 4,
                       "interior_ranks": dd.plans[0].nranges},
            "solve_roofline": {"flops": flops, "t_roof_ms": flops / (fp64 * 1e12) * 1e3,
                               "frac": flops / (fp64 * 1e12) * 1e3 / ms, "fp64_tflops_peak": fp64},
            "plan_build_s": build_s, "scalar_coupled_interiors": ifl == 8.0,
            "grid_rel_residual": res, "clocks": clk.summary(),
            "gpu_launches": _native.launch_count() - lc0}
    emit(line)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("BENCH_CONFIG", "c4"), choices=sorted(BENCH_CFG) + ["c3dd"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ranks", type=int, default=0)
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="use the row-sharded NCCL path even on one GPU")
    ap.add_argument("--inputs", default="numpy", choices=["numpy", "device"],
                    help="numpy: the seeded numpy stream (reference-golden inputs, parity report); "
                         "device: torch Philox on the GPU (A/B runs only)")
    args = ap.parse_args()
    _stdout_to_stderr()
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c3dd":
        run_dd(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
