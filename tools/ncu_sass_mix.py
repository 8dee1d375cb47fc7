"""Instruction mix and stall samples per SASS opcode (and the top source lines) of an ncu report.

    python tools/ncu_sass_mix.py REP.ncu-rep [--lines]
"""
import collections
import csv
import io
import subprocess
import sys


def rows(path, extra=()):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", *extra],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(path, lines=False):
    r = rows(path)
    hi = next(i for i, x in enumerate(r) if x and x[0] == "Address")
    h = r[hi]
    ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    op = collections.Counter()
    st = collections.Counter()
    tot_i = tot_s = 0
    for x in r[hi + 1:]:
        if len(x) < len(h) or not x[0].startswith("0x"):
            continue
        m = x[1].split()
        if not m:
            continue
        k = m[0] if not m[0].startswith("@") else m[1]
        k = k.split(".")[0]
        n = int(x[ie] or 0)
        s = int(x[ss] or 0)
        op[k] += n
        st[k] += s
        tot_i += n
        tot_s += s
    print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
    for k, n in op.most_common(30):
        print(f"  {k:12s} {n:14,d} {n / tot_i:7.2%}   stalls {st[k] / max(tot_s, 1):7.2%}")
    if lines:
        r = rows(path, ("--print-source", "cuda,sass"))
        cur = None
        agg = collections.Counter()
        sagg = collections.Counter()
        hdr = None
        for x in r:
            if x and x[0] == "Line No":
                hdr = x
                continue
            if hdr is None or len(x) < 6:
                continue
            if x[0]:
                cur = (x[0], x[1][:90])
                continue
            try:
                agg[cur] += int(x[hdr.index("Instructions Executed")] or 0)
                sagg[cur] += int(x[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            except (ValueError, IndexError):
                pass
        print("top source lines by instructions executed:")
        for k, n in agg.most_common(25):
            print(f"  {n:14,d} {n / tot_i:6.2%} stalls {sagg[k] / max(tot_s, 1):6.2%}  L{k[0]}: {k[1]}")


if __name__ == "__main__":
    main(sys.argv[1], "--lines" in sys.argv)
