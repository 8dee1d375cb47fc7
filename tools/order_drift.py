#!/usr/bin/env python
"""fp32 evaluation-order drift at full size (reading Q8), oracle only:
C3 (512^3, SO8, 500 steps) in fp64 (canonical order), fp32 canonical (O1) and fp32 in the paper's
printed order (O1-literal); writes tests/golden/order_drift_C3.json with the rel-L2 of each fp32
result against fp64 and against each other.

    python tools/order_drift.py [C3]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as W  # noqa: E402


def rel(g, w):
    g = np.asarray(g, np.float64)
    w = np.asarray(w, np.float64)
    return float(np.sqrt(((g - w) ** 2).sum() / (w * w).sum()))


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    p = W.problem(cfg)
    t0 = time.time()
    _, c64, _ = oracle.run_problem(p, dtype=np.float64)
    _, c32, _ = oracle.run_problem(p)
    _, l32, _ = oracle.run_problem(p, kind="literal")
    doc = {"config": cfg, "grid": list(p.n), "nt": p.nt, "space_order": p.space_order,
           "written_by": "tools/order_drift.py (oracle only)",
           "rel_l2_fp32_canonical_vs_fp64": rel(c32, c64),
           "rel_l2_fp32_literal_vs_fp64": rel(l32, c64),
           "rel_l2_fp32_literal_vs_fp32_canonical": rel(l32, c32),
           "seconds": round(time.time() - t0, 1)}
    with open(os.path.join(ROOT, "tests", "golden", f"order_drift_{cfg}.json"), "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
