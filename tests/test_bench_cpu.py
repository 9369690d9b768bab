"""bench.py pieces that run without a GPU: the reference arm's single JSON line
(the unmodified reference's plan_solve from oracle/_ref on the host cores; the
C port of its algorithm when the reference is not built) and the plan-parameter
policy behind every bench line (whole waves of sweep CTAs per GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c0",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "RHS/s" and d["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": "RHS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refcpu

    assert d["cpu_baseline"]["kind"] == ("reference" if refcpu.available() else "port")
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] == d["value"]
    assert d["config"]["workload"] == "c0" and d["steps"] == 2 and d["warmup"] == 1


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c0",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_plan_params_whole_waves(world):
    # c1/c2: 37 ranges per GPU (148 = 4 x 37: every chain grid is whole waves)
    # (18 per GPU on 4 and 8 GPUs: shallower sharded trees)
    for c in ("c1", "c2"):
        ranks, split = bench.plan_params(c, world)
        assert ranks == (37 if world <= 2 else 18) * world and split == 1
    # c4: paired reading of BASELINE (8/16/32/64 subdomains per GPU), one wave of 592 device ranges
    ranks, split = bench.plan_params("c4", world)
    assert ranks == 8 * world * world
    assert ranks // world * split <= 592 and ranks // world * (split + 1) > 592
    # explicit overrides win
    assert bench.plan_params("c4", world, ranks=64, split=37) == (64, 37)
