"""Summarise registers/spills per sweep instance from paper_1707_02347_b200/_build/ptxas.log."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1707_02347_b200/_build/ptxas.log").read().splitlines()
cur, sp = None, 0
rows = []
for l in log:
    if "Compiling entry" in l:
        m = re.search(r"sweep_kernelILi(\d)ELi(\d)ELb([01])ELi(\d)ELi(\d)ELi(\d+)E", l)
        cur = "R=%s TK=%s wave=%s ndim=%s VY=%s NWY=%s" % m.groups() if m else None
    m2 = re.search(r"(\d+) bytes spill stores", l)
    if m2:
        sp = int(m2.group(1))
    m3 = re.search(r"Used (\d+) registers", l)
    if m3 and cur:
        rows.append((cur, int(m3.group(1)), sp))
for r in sorted(rows):
    print("%-40s regs %3d spill %d" % r)
