"""Projected multi-GPU strong scaling WITH the two per-solve all-gathers priced.

Input: the per-rank phase times of the sharded solve measured on one B200
(tools/shard_projection.py -> the "final projections" block of
profiles/r01_shard_projection.txt: every rank's phases A / B / C timed while it
has the GPU alone).  Output: step = max_r A + max_r B + max_r C + 2 all-gathers
(carry blocks, crossing-node partial sums), each priced with a latency /
bandwidth model t = alpha + (W - 1) * bytes_per_rank / bw (ring/NVLS all-gather
moves (W-1)/W of the gathered volume through each GPU).  No multi-GPU box was
available, so alpha is swept over the range NCCL shows for small all-gathers on
one NVSwitch node (8 / 15 / 25 us) and bw = 350 GB/s per GPU.

    python tools/collective_projection.py [profiles/r01_shard_projection.txt]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALPHAS_US = (8.0, 15.0, 25.0)
BW = 350e9


def load(path):
    rows, final = [], False
    for line in open(path):
        if line.startswith("## final projections"):
            final = True
            continue
        if final and line.startswith("{"):
            rows.append(json.loads(line))
    return rows


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_shard_projection.txt")
    rows = load(path)
    base = {r["config"]: r for r in rows if r["world"] == 1}
    print("config world  step_ms(no coll)  " + "  ".join(f"alpha={a:g}us: step_ms eff" for a in ALPHAS_US)
          + "  | one merged exchange (alpha=15us)")
    for r in rows:
        w, name = r["world"], r["config"]
        b1 = base[name]
        t1 = b1["step_ms"]
        cells = []
        for a in ALPHAS_US:
            coll = 0.0
            if w > 1:
                for nbytes in r["allgather_bytes_per_rank"]:
                    if nbytes:
                        coll += a * 1e-3 + (w - 1) * nbytes / BW * 1e3
            step = r["step_ms"] + coll
            cells.append(f"{step:8.3f} {t1 / (w * step):5.3f}")
        merged = r["step_ms"]
        if w > 1:
            merged += 15e-3 + (w - 1) * sum(r["allgather_bytes_per_rank"]) / BW * 1e3
        print(f"{name:6} {w:5d}  {r['step_ms']:16.3f}  " + "  ".join(cells)
              + f"  | {merged:8.3f} {t1 / (w * merged):5.3f}")


if __name__ == "__main__":
    main()
