"""DMMA dependency distances in the SASS of the chain kernels.

For every DMMA of each matching kernel: how many DMMAs earlier the same accumulator was last
written (1 = back-to-back dependent issue, which exposes the DMMA latency).  Also registers and
spill bytes.  Usage: python tools/sass_dmma_deps.py <cubin|so> [name-substring ...]
"""
import collections
import re
import subprocess
import sys


def main():
    path, pats = sys.argv[1], sys.argv[2:]
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", path], capture_output=True, text=True).stdout
    usage = {}
    cur = None
    for ln in res.splitlines():
        m = re.search(r"Function (\S+):", ln)
        if m:
            cur = m.group(1)
        m = re.search(r"REG:(\d+).*?(?:STACK:(\d+))?", ln)
        if m and cur:
            st = re.search(r"STACK:(\d+)", ln)
            usage[cur] = (int(m.group(1)), int(st.group(1)) if st else 0)
    fn = None
    seqs = collections.OrderedDict()
    for ln in sass.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            fn = m.group(1)
            seqs[fn] = []
            continue
        if fn is None:
            continue
        m = re.search(r"\s(DMMA\.8x8x4)\s+(R\d+),", ln)
        if m:
            seqs[fn].append(m.group(2))
        elif re.search(r"\s(BRA|BAR\.SYNC|EXIT)", ln):
            seqs[fn].append(None)  # block boundary
    for fn, seq in seqs.items():
        if not seq or (pats and not any(p in fn for p in pats)):
            continue
        hist = collections.Counter()
        last = {}
        i = 0
        for r in seq:
            if r is None:
                last = {}
                i = 0
                continue
            d = i - last[r] if r in last else 0
            hist[min(d, 9)] += 1
            last[r] = i
            i += 1
        n = sum(hist.values())
        regs = usage.get(fn, ("?", "?"))
        print(f"{fn[:110]}\n   regs={regs[0]} stack={regs[1]} dmma={n} "
              + " ".join(f"d{k}={hist[k] / n:.2f}" for k in sorted(hist)) + "  (d0 = first in block, d9 = >= 9)")


if __name__ == "__main__":
    main()
