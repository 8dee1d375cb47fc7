#!/usr/bin/env python
"""Aggregate the per-instruction warp-stall samples of an ncu source page (SASS view).

    ncu -i REP --page source --csv --print-source sass > x.csv; python tools/ncu_stalls.py x.csv [topN]

Prints the stall-reason totals, the instructions with the most samples (with their reason mix),
and samples grouped by SASS opcode."""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot = collections.Counter()
    per = []
    byop = collections.Counter()
    allsmp = 0
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        try:
            n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        allsmp += n
        mix = {k: int(r[ix[k]] or 0) for k in reasons}
        for k, v in mix.items():
            tot[k] += v
        src = r[ix["Source"]]
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        byop[op.split(".")[0]] += n
        per.append((n, r[ix["Address"]], src, mix))
    print(f"total samples {allsmp}")
    for k, v in tot.most_common():
        if v:
            print(f"  {k:28s} {v:8d} {100.0 * v / max(1, allsmp):5.1f}%")
    print("by opcode:")
    for k, v in byop.most_common(15):
        print(f"  {k:12s} {v:8d} {100.0 * v / max(1, allsmp):5.1f}%")
    print("top instructions:")
    for n, a, src, mix in sorted(per, reverse=True)[:top]:
        m = ", ".join(f"{k[6:]}={v}" for k, v in sorted(mix.items(), key=lambda x: -x[1])[:3] if v)
        print(f"  {n:7d} {a:>6s} {src[:60]:60s} {m}")


if __name__ == "__main__":
    main()
