"""Short run of one config through the public API, for ncu captures (no timing claims).

    python tools/prof_run.py --config C5 --tk 1 --nt 6
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--tk", type=int, default=1)
    ap.add_argument("--nt", type=int, default=6)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--grid", default=None, help="interior grid override, e.g. 512x512x512")
    a = ap.parse_args()
    import torch
    import workloads as W
    from paper_1707_02347_b200.dist import SlabRunner
    p = W.problem(a.config, n=tuple(int(v) for v in a.grid.split("x")) if a.grid else None)
    r = SlabRunner(p, t_kernel=a.tk, device=0)
    host = r.host_inputs(a.nt, pin=False)
    dev = r.to_device(host)
    for _ in range(a.reps):
        r.reset_state(dev)
        r.run(dev, a.nt)
    torch.cuda.synchronize()
    print("ok", a.config, a.tk, a.nt)


if __name__ == "__main__":
    main()
