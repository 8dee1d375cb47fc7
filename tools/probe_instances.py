"""Run every compiled kernel instance once on a small grid (each in its own subprocess, so a
faulting instance cannot take down the others) and compare bit-exactly with the oracle.

    python tools/probe_instances.py [--only ndim,order,time_order,tk]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def one(ndim, order, time_order, tk):
    import numpy as np
    import workloads as W
    from harness import gpu_run, oracle_run
    if ndim == 2:
        p = W.problem("C1", n=(45, 37, 1), nt=5)
    else:
        p = W.problem("C2", n=(45, 37, 21), nt=5)
    d = dict(p.__dict__, space_order=order)
    if time_order == 2:
        q = W.problem("C3", n=p.n, nt=5, sponge=3)
        d = dict(q.__dict__, space_order=order, src=((22, 18, p.n[2] // 2),), ndim=ndim)
    p = W.Problem(**d)
    g = gpu_run(p, t_kernel=tk)
    o = oracle_run(p)
    return all(np.array_equal(a, b) for a, b in zip(g, o))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--child", default=None)
    a = ap.parse_args()
    if a.child:
        nd, o, to, tk = map(int, a.child.split(","))
        ok = one(nd, o, to, tk)
        print("RESULT", json.dumps({"cfg": a.child, "bitwise": ok}))
        return
    from paper_1707_02347_b200.build import instances
    cfgs = [(nd, 2 * R, 2 if w else 1, TK) for (nd, w, R, TK, *_rest) in instances()]
    if a.only:
        cfgs = [tuple(map(int, a.only.split(",")))]
    for c in cfgs:
        key = ",".join(map(str, c))
        r = subprocess.run([sys.executable, __file__, "--child", key], capture_output=True, text=True,
                           timeout=300)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
        if line:
            print(line[0][7:], flush=True)
        else:
            err = (r.stderr.strip().splitlines() or ["?"])[-1]
            print(json.dumps({"cfg": key, "error": err[-200:]}), flush=True)


if __name__ == "__main__":
    main()
