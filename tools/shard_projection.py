"""Per-rank device time of the row-sharded solve at world W, emulated on ONE GPU.

    python tools/shard_projection.py --config c4 --worlds 1 2 4 8 [--split S] [--reps 3]

Every rank's shard plan lives on the one device; a solve runs phase A (local
sweeps) for all ranks, a host-side concatenation stands in for the carry
all-gather, phase B (interface RHS, series sums / crossing partials), the
partials all-gather, phase C (tree levels, recovery) -- the same three C-ABI
calls ShardedPlan makes.  Each rank's phases are timed with CUDA events while
that rank has the GPU to itself, i.e. what the rank's own B200 would do.  The
projected step is max_r A + max_r B + max_r C plus the two all-gathers (their
bytes are printed; on NVSwitch a few-MB all-gather is tens of microseconds and
is NOT included).  No kernel waits on another rank's kernel.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1108_4181_b200 import configs  # noqa: E402
from paper_1108_4181_b200.distributed import NativeBackend  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def project(name, world, split=0, reps=3, ranks=0):
    cfg = configs.CONFIGS[name]
    ranks, sp = bench.plan_params(name, world, ranks, split)
    d, lo, up, F = configs.generate(name, device="cuda")
    n, m, K = cfg["n"], cfg["m"], cfg["k"]
    be = NativeBackend(0)
    hs = []
    for r in range(world):
        h, st, row, rng = be.create(d, lo, up, n, m, ranks, sp, r, world)
        assert st == 0, (st, row, rng)
        hs.append(h)
    allc = torch.cat([be.contrib(h) for h in hs])
    for h in hs:
        st, _ = be.finish(h, allc)
        assert st == 0
    del d, lo, up
    infos = [be.info(h) for h in hs]
    fl = [F[i.row_lo:i.row_hi] for i in infos]
    xl = [torch.empty_like(f) for f in fl]
    sizes = [be.exchange_size(h, K) for h in hs]
    tA = [[] for _ in hs]; tB = [[] for _ in hs]; tC = [[] for _ in hs]
    for it in range(reps + 2):
        carries, parts = [], []
        for r, h in enumerate(hs):
            c = be.empty(sizes[r][0])
            e0, e1 = ev(), ev()
            e0.record(); be.solve_a(h, fl[r], xl[r], K, c); e1.record(); e1.synchronize()
            tA[r].append(e0.elapsed_time(e1)); carries.append(c)
        carry_all = torch.cat(carries)
        for r, h in enumerate(hs):
            pt = be.empty(max(sizes[r][1], 1))
            e0, e1 = ev(), ev()
            e0.record(); be.solve_b(h, carry_all, pt, K); e1.record(); e1.synchronize()
            tB[r].append(e0.elapsed_time(e1)); parts.append(pt[:sizes[r][1]])
        part_all = torch.cat(parts) if parts[0].numel() else be.empty(1)
        for r, h in enumerate(hs):
            e0, e1 = ev(), ev()
            e0.record(); be.solve_c(h, part_all, fl[r], xl[r], K); e1.record(); e1.synchronize()
            tC[r].append(e0.elapsed_time(e1))
    med = lambda v: sorted(v[2:])[len(v[2:]) // 2]
    A = [med(v) for v in tA]; B = [med(v) for v in tB]; C = [med(v) for v in tC]
    step = max(A) + max(B) + max(C)
    out = {"config": name, "world": world, "ranks": ranks, "split": sp,
           "device_ranges_per_gpu": infos[0].range_hi - infos[0].range_lo,
           "phase_ms_max": [max(A), max(B), max(C)], "phase_ms_rank0": [A[0], B[0], C[0]],
           "step_ms": step, "rhs_per_s": K / (step / 1e3),
           "allgather_bytes_per_rank": [sizes[0][0] * 8, sizes[0][1] * 8]}
    for h in hs:
        be.destroy(h)
    del F, fl, xl
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ranks-per-gpu", type=int, default=0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    base = None
    for w in a.worlds:
        r = project(a.config, w, a.split, a.reps, a.ranks_per_gpu * w)
        base = base or (r["rhs_per_s"] if w == 1 else None)
        if base:
            r["projected_efficiency"] = r["rhs_per_s"] / (w * base)
        print(json.dumps(r), flush=True)
