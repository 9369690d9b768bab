#!/usr/bin/env python
"""A/B runner for bench.py variants (replaces round 1's ~30 one-off tools/ab*.sh).

Each variant is LABEL[:ENV=V,ENV=V][:bench args]; every variant runs
``bench.py --steps S --warmup W --no-e2e --no-cpu --no-check`` in a fresh
process with those environment variables and arguments, and one summary line
is printed per variant (RHS/s, ms/step, per-phase ms, solve roofline fraction).

    python tools/ab.py --config c2 base "f20:BTD_CHAIN_VARIANT=20" "p74::--ranks 74"
    python tools/ab.py --config c4 "s37::--split 37" "s74::--split 74" --repeat 3

Variant knobs live in the library as environment variables read at plan build
(BTD_FORCE_MODE, BTD_HOST_CHUNKS, BTD_HOST_MINW, BTD_HOST_SLOTS, ...) or as
bench.py arguments (--ranks, --split, --config)."""

import argparse
import json
import os
import shlex
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(label, env, args, steps, warmup):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", str(steps), "--warmup", str(warmup),
           "--no-e2e", "--no-cpu", "--no-check", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, env=dict(os.environ, **env), cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    if r.returncode or not lines:
        return f"{label}: FAILED rc={r.returncode} {r.stderr[-400:]}"
    d = json.loads(lines[-1])
    c, ph = d["config"], d.get("phases_ms") or {}
    return (f"{label:>12} {c['workload']} P={c.get('ranks')} split={c.get('split')} RHS/s={d['value']:.0f} "
            f"ms={d['ms_per_step']:.3f} fwd={ph.get('forward', 0):.3f} tree={ph.get('interface_tree', 0):.3f} "
            f"bwd={ph.get('backward', 0):.3f} solve_frac={d['solve_roofline']['frac']:.3f} "
            f"kernel_frac={d['roofline']['frac']:.3f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--config", default="c4")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--repeat", type=int, default=1)
    a = ap.parse_args()
    for _ in range(a.repeat):
        for v in a.variants:
            parts = v.split(":", 2)
            label = parts[0]
            env = dict(kv.split("=", 1) for kv in parts[1].split(",") if kv) if len(parts) > 1 else {}
            args = shlex.split(parts[2]) if len(parts) > 2 else []
            if "--config" not in args:
                args = ["--config", a.config, *args]
            print(run(label, env, args, a.steps, a.warmup), flush=True)


if __name__ == "__main__":
    main()
