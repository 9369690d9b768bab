"""Per-kernel share of one solve step from an ncu launch list (btd:: kernels).

usage: launch_shares.py OUT_JSON cfg:launches.csv:plain.log [...]
The plain bench log (--steps 1) reports gpu_launches for one step; the last
that-many launches of the ncu list are the final solve."""
import csv, json, sys

out = {}
for arg in sys.argv[2:]:
    cfg, lcsv, plain = arg.split(":")
    line = [l for l in open(plain) if l.startswith("{")][-1]
    n = int(json.loads(line)["gpu_launches"])
    rows = list(csv.reader(open(lcsv)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    t = []
    for r in rows[hdr + 1:]:
        # only this library's kernels (the bench also runs cuBLAS / torch kernels)
        # (helper kernels in btd_api.cu's anonymous namespace count too: gpu_launches counts them)
        if len(r) > vi and r[mi] == "gpu__time_duration.sum" and ("btd::" in r[ki] or "anonymous namespace" in r[ki]):
            v = float(r[vi].replace(",", ""))
            u = r[ui]
            v = v / 1000.0 if u in ("ns", "nsecond") else (v * 1000.0 if u in ("ms", "msecond") else v)
            t.append((r[ki].split("(")[0][:60], v))
    step = t[-n:]
    tot = sum(v for _, v in step)
    agg = {}
    for k, v in step:
        a = agg.setdefault(k, {"launches": 0, "total_us": 0.0})
        a["launches"] += 1
        a["total_us"] += v
    for a in agg.values():
        a["share"] = round(a["total_us"] / tot, 4)
        a["total_us"] = round(a["total_us"], 1)
    out[cfg] = {"launches_per_step": n, "step_us_serialised": round(tot, 1), "kernels": agg}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps({c: {k: v["share"] for k, v in o["kernels"].items()} for c, o in out.items()}, indent=1))
