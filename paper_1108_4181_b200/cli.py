"""``solve`` command on the GPU path.

Mirrors the reference's ``blocktri solve`` (cli.py:171-232): read a BTR1
matrix and BVC1 right-hand sides, build the plan, solve all right-hand sides
as one batch, write ``solution_XXX.bvc`` files and ``solve_report.json``
({command, config, results}), exit 1 if the worst residual
``max|P x - f| / max|f|`` exceeds ``tol``.  Config handling follows the
reference (defaults <- JSON config or an emitted report <- flags, unknown keys
rejected, cli.py:96-150) and so do the exit codes (0 ok, 1 numerical,
2 i/o, 3 config; errors as one JSON line on stderr, cli.py:449-467).

``plan_cache`` follows ref cli.py:183-196: an existing DPLN file bound to this
matrix (and the same ranks/split) is loaded instead of building, anything else
(missing, other matrix, malformed) is rebuilt and the cache rewritten.  GPU plan
files import the device factors directly (io.read_plan); the reference's own
CPU DPLN files are validated and the GPU plan is rebuilt from the matrix.

    python -m paper_1108_4181_b200.cli solve --matrix A.btr --rhs f.bvc --ranks 8 [--split 4]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

from . import errors
from . import io as bio
from .distributed import stage_count

EXIT_OK, EXIT_NUMERICAL, EXIT_IO, EXIT_CONFIG = 0, 1, 2, 3


class ConfigError(errors.BlocktriError):
    """Invalid or unknown configuration keys/values (ref errors.py:80-81)."""


_SCHEMA = {"matrix": str, "rhs": (str, list), "ranks": int, "tol": float, "out": str, "seed": int,
           "plan_cache": str, "split": int}
_DEFAULTS = {"ranks": 1, "tol": 1e-8, "out": ".", "seed": 0, "split": 1}


def _validate(cfg):
    if not isinstance(cfg, dict):
        raise ConfigError("solve: expected an object")
    for key, val in cfg.items():
        if key not in _SCHEMA:
            raise ConfigError(f"solve: unknown key {key!r}")
        want = _SCHEMA[key]
        if want is float:
            ok = isinstance(val, (int, float)) and not isinstance(val, bool)
        elif want is int:
            ok = isinstance(val, int) and not isinstance(val, bool)
        else:
            ok = isinstance(val, want)
        if not ok:
            raise ConfigError(f"solve.{key}: wrong type {type(val).__name__}")


def load_config(path=None, overrides=None):
    cfg = dict(_DEFAULTS)
    if path is not None:
        try:
            with open(path) as fh:
                data = json.load(fh)
        except OSError as exc:
            raise bio.FileFormatError(f"cannot read config: {exc}") from exc
        except json.JSONDecodeError as exc:
            raise ConfigError(f"config is not valid JSON: {exc}") from exc
        if isinstance(data, dict) and "config" in data and "command" in data:
            if data["command"] != "solve":
                raise ConfigError(f"report was produced by {data['command']!r}, not 'solve'")
            data = data["config"]
        _validate(data)
        cfg.update(data)
    if overrides:
        _validate(overrides)
        cfg.update(overrides)
    return cfg


def cmd_solve(cfg):
    from . import dichotomy

    if "matrix" not in cfg or "rhs" not in cfg:
        raise ConfigError("solve needs 'matrix' and 'rhs' paths")
    out = cfg["out"]
    os.makedirs(out, exist_ok=True)
    matrix = bio.read_matrix(cfg["matrix"])
    paths = cfg["rhs"] if isinstance(cfg["rhs"], list) else [cfg["rhs"]]
    vectors = [bio.read_vector(p) for p in paths]
    for v in vectors:
        if v.n != matrix.n or v.m != matrix.m:
            raise ConfigError(f"rhs layout ({v.n},{v.m}) != matrix ({matrix.n},{matrix.m})")
    t0 = time.time()
    plan, cache, cache_hit = None, cfg.get("plan_cache"), False
    if cache and os.path.exists(cache):
        try:
            plan = bio.read_plan(cache, matrix)
            if plan.ranks != cfg["ranks"] or plan.split != cfg["split"]:
                plan = None
            else:
                cache_hit = True
        except bio.FileFormatError:
            plan = None
    if plan is None:
        plan = dichotomy.plan_build(matrix, cfg["ranks"], split=cfg["split"])
        if cache:
            bio.write_plan(cache, plan)
    build_s = time.time() - t0
    batch = np.stack([v.data for v in vectors], axis=2)
    t0 = time.time()
    x = dichotomy.plan_solve(plan, batch)
    solve_s = time.time() - t0
    residuals, sols = [], []
    for i, v in enumerate(vectors):
        xi = np.ascontiguousarray(x[:, :, i])
        r = matrix.apply(xi) - v.data
        den = np.abs(v.data).max() or 1.0
        residuals.append(float(np.abs(r).max() / den))
        p = os.path.join(out, f"solution_{i:03d}.bvc")
        bio.write_vector(p, xi)
        sols.append(p)
    worst = max(residuals)
    results = {"residual": worst, "residuals": residuals, "plan_build_seconds": build_s,
               "solve_seconds": solve_s, "ranks": cfg["ranks"], "stages": stage_count(cfg["ranks"]),
               "solutions": sols, "backend": "b200", "device_ranges": plan.nranges,
               "plan_cache_hit": cache_hit}
    report = {"command": "solve", "config": cfg, "results": results}
    bio.atomic_write(os.path.join(out, "solve_report.json"),
                     (json.dumps(report, indent=2, sort_keys=True) + "\n").encode())
    if worst > cfg["tol"]:
        raise errors.BlocktriError(f"residual {worst:.3e} exceeds tolerance {cfg['tol']:.1e}")
    return results


def _parser():
    ap = argparse.ArgumentParser(prog="paper_1108_4181_b200", description="B200 dichotomy solver")
    sub = ap.add_subparsers(dest="command", required=True)
    ps = sub.add_parser("solve", help="solve BTR1/BVC1 systems on the GPU")
    ps.add_argument("--config")
    ps.add_argument("--out")
    ps.add_argument("--seed", type=int)
    ps.add_argument("--tol", type=float)
    ps.add_argument("--matrix")
    ps.add_argument("--rhs", action="append")
    ps.add_argument("--ranks", type=int)
    ps.add_argument("--split", type=int)
    ps.add_argument("--plan-cache", dest="plan_cache")
    return ap


def _fail(category, exc, code):
    sys.stderr.write(json.dumps({"error": category, "message": str(exc)}) + "\n")
    return code


def main(argv=None):
    args = _parser().parse_args(argv)
    over = {k: getattr(args, k) for k in ("out", "seed", "tol", "matrix", "ranks", "split", "plan_cache")
            if getattr(args, k) is not None}
    if args.rhs:
        over["rhs"] = args.rhs if len(args.rhs) > 1 else args.rhs[0]
    try:
        cmd_solve(load_config(args.config, over))
    except ConfigError as exc:
        return _fail("config", exc, EXIT_CONFIG)
    except (FileNotFoundError, OSError, bio.FileFormatError) as exc:
        return _fail("io", exc, EXIT_IO)
    except errors.BlocktriError as exc:
        return _fail("numerical", exc, EXIT_NUMERICAL)
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
