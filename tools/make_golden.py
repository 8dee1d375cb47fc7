#!/usr/bin/env python
"""Write the full-nt oracle fixtures tests/golden/fullnt_<cfg>.{json,npz}.

Calls ONLY oracle/ and workloads/ (no product code): O1 (the canonical untiled loop nest) runs
config C3 / C4 / C5 at its full nt from the seeded inputs, and the fixture stores
  * SHA-256 of the interior bytes of u^{nt} and u^{nt-1} (fp32, (nz, ny, nx) C order) -- the GPU
    path computes the canonical order, so its fields must hash identically (bitwise parity);
  * the fp64 L2 norms of both fields and of the receiver trace;
  * a strided sample of both fields (every s-th point per axis, float32) and the full receiver
    trace, for element-wise diagnostics and a sampled rel-L2 when the digests differ;
  * for C3 and C5 (--literal): the rel-L2 between O1 and O1-literal (the paper's printed update
    expression and term order) at full nt -- the fp32 drift bound of reading Q8.

    python tools/make_golden.py C3 C5 C4 [--literal C3 C5]

The paper's correctness check compares whole runs, tiled against untiled.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as W  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
STRIDE = {"C3": 16, "C4": 32, "C5": 24}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def norm(a: np.ndarray) -> float:
    a = np.asarray(a, dtype=np.float64)
    return float(np.sqrt((a * a).sum()))


def rel(g, w) -> float:
    g = np.asarray(g, np.float64)
    w = np.asarray(w, np.float64)
    d = np.sqrt((w * w).sum())
    return float(np.sqrt(((g - w) ** 2).sum()) / d) if d > 0 else float(np.sqrt(((g - w) ** 2).sum()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--literal", nargs="*", default=[])
    a = ap.parse_args()
    os.makedirs(GOLDEN, exist_ok=True)
    for cfg in a.configs:
        p = W.problem(cfg)
        t0 = time.time()
        P, C, tr = oracle.run_problem(p)
        secs = time.time() - t0
        s = STRIDE[cfg]
        doc = {
            "config": cfg, "grid": list(p.n), "nt": p.nt, "space_order": p.space_order,
            "written_by": "tools/make_golden.py (oracle O1 only)",
            "oracle_threads": oracle.num_threads(), "oracle_seconds": round(secs, 1),
            "sha256_u_nt": sha(C), "sha256_u_nt_minus_1": sha(P),
            "norm_u_nt": norm(C), "norm_u_nt_minus_1": norm(P), "norm_trace": norm(tr),
            "nrec": int(tr.shape[1]), "sample_stride": s,
        }
        if cfg in a.literal:
            t1 = time.time()
            Pl, Cl, trl = oracle.run_problem(p, kind="literal")
            doc["literal"] = {
                "what": "O1-literal (paper's printed expression/term order, P:1678-1708) vs O1, fp32, full nt",
                "rel_l2_u_nt": rel(Cl, C), "rel_l2_u_nt_minus_1": rel(Pl, P),
                "rel_l2_trace": rel(trl, tr) if tr.size else 0.0,
                "max_abs_u_nt": float(np.abs(Cl.astype(np.float64) - C).max()),
                "seconds": round(time.time() - t1, 1)}
            del Pl, Cl, trl
        np.savez_compressed(os.path.join(GOLDEN, f"fullnt_{cfg}.npz"),
                            u_nt=C[::s, ::s, ::s].copy(), u_nt_minus_1=P[::s, ::s, ::s].copy(),
                            trace=tr.astype(np.float32))
        with open(os.path.join(GOLDEN, f"fullnt_{cfg}.json"), "w") as f:
            json.dump(doc, f, indent=1)
        print(json.dumps(doc), flush=True)
        del P, C, tr


if __name__ == "__main__":
    main()
