"""Registers / spills per kernel from `python -m paper_1108_4181_b200.build --force -v` stderr."""
import re, subprocess, sys
out = subprocess.run([sys.executable, "-m", "paper_1108_4181_b200.build", "--force", "-v"], capture_output=True, text=True).stderr
cur = None; info = {}
for ln in out.splitlines():
    m = re.search(r"Function properties for (\S+)", ln) or re.search(r"Compiling entry function '(\S+)'", ln)
    if m: cur = m.group(1); info.setdefault(cur, {})
    m = re.search(r"(\d+) bytes spill stores", ln)
    if m and cur: info[cur]["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur: info[cur]["regs"] = int(m.group(1))
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for k, v in sorted(info.items()):
    if pat in k: print(f"{v.get('regs','?'):>4} regs {v.get('spill',0):>5} spill  {k}")
