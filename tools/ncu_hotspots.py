"""Top SASS instructions by stall samples from an ncu source-page CSV, with opcode totals."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
cols = ["stall_wait", "stall_long_sb", "stall_math", "stall_short_sb", "stall_barrier", "stall_selected"]
byop = collections.Counter(); tot = collections.Counter()
data = [r for r in data if len(r) == len(hdr) and r[0].startswith("0x")]
for r in data:
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    for c in cols:
        v = float(r[ix[c]] or 0)
        byop[(op, c)] += v
        tot[c] += v
print("totals:", dict(tot))
for c in cols:
    top = sorted(((v, op) for (op, cc), v in byop.items() if cc == c), reverse=True)[:5]
    print(f"{c:15s}", ", ".join(f"{op}={v:.0f}" for v, op in top))
# show a window of the hottest wait instructions
best = sorted(range(len(data)), key=lambda i: -float(data[i][ix["stall_wait"]] or 0))[:6]
for i in best:
    lo, hi = max(0, i - 3), min(len(data), i + 2)
    print("----")
    for j in range(lo, hi):
        print(f"{data[j][ix['stall_wait']]:>6s} {data[j][ix['stall_long_sb']]:>6s}  {data[j][ix['Source']].strip()[:90]}")
