"""Registers / spills per kernel from build/obj/kernels.ptxas.txt (nvcc -Xptxas -v output).

    python tools/ptxas_summary.py [regex]
"""
import re
import subprocess
import sys
from pathlib import Path

txt = (Path(__file__).resolve().parent.parent / "build" / "obj" / "kernels.ptxas.txt").read_text()
pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
cur = None
rows = []
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows.append([cur, m.groups(), None])
    m = re.search(r"Used (\d+) registers", line)
    if m and rows and rows[-1][2] is None:
        rows[-1][2] = m.group(1)
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.split("\n")
for (mangled, (stk, st, ld), reg), name in zip(rows, names):
    if pat and not pat.search(name):
        continue
    print(f"{reg:>4} regs  stack {stk:>3}  spill st/ld {st:>3}/{ld:<3}  {name}")
