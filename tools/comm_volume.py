"""Per-solve exchange volume per rank of the sharded solve, old (all-gather of
every range's (base, carry) pair, the reference harness pattern) vs new
(carry shift + partial series sums of crossing tree nodes)."""
import sys
sys.path[:0] = ["oracle", "."]
import blocktri_oracle as O
import bench

def needed(tree, nr, q0, q1):
    need = [0] * (nr + 1)
    for q in range(q0, min(q1, nr - 1) + 1):
        need[q] = 1
    changed = True
    while changed:
        changed = False
        for lo, hi, k, _ in reversed(tree):
            if not need[k]:
                continue
            if lo >= 1 and not need[lo - 1]:
                need[lo - 1] = changed = 1
            if hi + 1 <= nr - 1 and not need[hi + 1]:
                need[hi + 1] = changed = 1
    return need

from paper_1108_4181_b200 import configs
for name in ("c1", "c2", "c3", "c4"):
    cfg = configs.CONFIGS[name]
    for world in (2, 4, 8):
        ranks, split = bench.plan_params(name, world)
        nr = min(cfg["n"], ranks * split)
        mp = cfg["m"]
        K = cfg["k"]
        tree = O.partition_tree(nr)
        nrl = nr // world
        cross = set()
        for r in range(world):
            nd = needed(tree, nr, r * nrl, (r + 1) * nrl)
            for b, (lo, hi, k, _) in enumerate(tree):
                if nd[k] and (lo < r * nrl or hi >= (r + 1) * nrl):
                    cross.add(b)
        blk = mp * K * 8
        old = world * nrl * 2 * blk
        new = world * (1 + len(cross)) * blk
        print(f"{name} world={world} ranges={nr} crossing_nodes={len(cross)}  received/rank/solve: "
              f"old {old/1e6:.1f} MB  new {new/1e6:.2f} MB")
