"""Registers / spills per kernel instance from an `nvcc -Xptxas -v` log: python scripts/ptxas_regs.py log [filter]."""
import re, sys
t = open(sys.argv[1]).read()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for m in re.finditer(r"Function properties for (\S+)\n\s*(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\nptxas info\s*: Used (\d+) registers", t):
    n = m.group(1)
    if flt not in n:
        continue
    k = re.findall(r"Li(\d+)E", n)
    print(n[:40], k, "stack", m.group(2), "spill st", m.group(3), "ld", m.group(4), "regs", m.group(5))
