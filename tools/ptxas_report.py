"""Summarise registers/spills per kernel instance from paper_1707_02347_b200/_build/ptxas.log."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1707_02347_b200/_build/ptxas.log").read()
rows = []
# ptxas prints: Compiling entry function 'NAME' ... / N bytes stack frame, S bytes spill stores ... / Used R registers
for m in re.finditer(r"Compiling entry function '([^']+)'[^\n]*\n(?:[^\n]*\n){0,3}?\s*(\d+) bytes stack frame, (\d+) bytes spill stores[^\n]*\n[^\n]*Used (\d+) registers", log):
    name, _, spill, regs = m.groups()
    a = re.search(r"sweep_kernelILi(\d)ELi(\d)ELb([01])ELi(\d)ELi(\d)ELi(\d+)E", name)
    b = re.search(r"sweep1_kernelILi(\d)ELb([01])ELi(\d)ELi(\d+)E", name)
    if a:
        key = "tiled  R=%s TK=%s wave=%s ndim=%s VY=%s NWY=%s" % a.groups()
    elif b:
        key = "untile R=%s TK=1 wave=%s ndim=%s NCW=%s" % b.groups()
    else:
        continue
    rows.append((key, int(regs), int(spill)))
for r in sorted(set(rows)):
    print("%-48s regs %3d spill %d" % r)
