"""Per-instruction stall samples of one kernel from `ncu -i rep --page source --csv --print-source sass`:
prints the hottest address window(s) with instruction, executed count and stall breakdown."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
ix = {h: i for i, h in enumerate(hdr)}
cols = ["stall_math", "stall_wait", "stall_short_sb", "stall_long_sb", "stall_barrier", "stall_selected",
        "stall_not_selected", "stall_mio", "stall_branch_resolving", "stall_dispatch", "stall_lg", "stall_no_inst"]
f = lambda r, c: float(r[ix[c]]) if r[ix[c]] not in ("", "-") else 0.0
tot = collections.Counter()
for r in data:
    for c in cols: tot[c] += f(r, c)
S = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print("samples", S, {c: round(v / S, 3) for c, v in tot.most_common()})
ops = collections.Counter(); opsamp = collections.Counter()
for r in data:
    src = r[ix["Source"]].strip(); op = src.split()[0]
    if op.startswith("@"): op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += int(float(r[ix["Instructions Executed"]] or 0)); opsamp[op] += f(r, "Warp Stall Sampling (All Samples)")
print("executed by opcode:", ops.most_common(14))
print("samples by opcode:", [(k, round(v / S, 3)) for k, v in opsamp.most_common(12)])
lo = int(sys.argv[2]) if len(sys.argv) > 2 else None
if lo is not None:
    hi = int(sys.argv[3])
    for r in data[lo:hi]:
        st = " ".join(f"{c[6:]}={int(f(r,c))}" for c in cols if f(r, c) > 0)
        print(f"{r[ix['Address']][-5:]} {int(float(r[ix['Instructions Executed']] or 0)):>9d} {r[ix['Source']].strip()[:60]:60s} {st}")
