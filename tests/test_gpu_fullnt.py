"""Full-length parity on the BASELINE grids: every config runs its whole nt on the GPU, in the
launch configuration bench.py times (planner T_k) and with the time-tiled T_k = 2 pass, and the
final fields must hash to the SHA-256 digests the CPU oracle O1 wrote for the same seeded inputs
(tests/golden/fullnt_<cfg>.json, written by tools/make_golden.py, which calls only oracle/ and
workloads/).  The paper's correctness check compares whole runs, tiled against untiled
(P:1817-1839); the north star asks for <= 1e-5 relative L2 after nt steps on every config -- the
GPU path computes the canonical order, so the bar here is bit equality, with the sampled rel-L2 and
the receiver traces (C5) checked element-wise as well."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import workloads as W
from harness import gpu_run, rel_l2

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden(cfg):
    path = os.path.join(GOLDEN, f"fullnt_{cfg}.json")
    if not os.path.exists(path):
        pytest.skip(f"no full-nt fixture for {cfg} (tools/make_golden.py {cfg})")
    doc = json.load(open(path))
    arr = np.load(os.path.join(GOLDEN, f"fullnt_{cfg}.npz"))
    return doc, arr


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


@pytest.mark.parametrize("cfg", ["C3", "C5", "C4"])
@pytest.mark.parametrize("tk", ["bench", 2])
def test_full_nt_matches_oracle_digest(cfg, tk):
    doc, arr = _golden(cfg)
    p = W.problem(cfg)
    assert [int(v) for v in doc["grid"]] == list(p.n) and doc["nt"] == p.nt
    if tk == "bench":
        from paper_1707_02347_b200.planner import plan
        tk = plan(p.time_order, p.radius, p.n).t_kernel
    gp, gc, gt = gpu_run(p, t_kernel=tk)
    s = doc["sample_stride"]
    # element-wise on the strided sample (diagnostic first, so a mismatch reports its size)
    err_s = max(rel_l2(gc[::s, ::s, ::s], arr["u_nt"]), rel_l2(gp[::s, ::s, ::s], arr["u_nt_minus_1"]))
    assert err_s <= 1e-5, f"sampled rel-L2 {err_s:.3e}"
    if doc["nrec"]:
        assert gt.shape == arr["trace"].shape
        assert rel_l2(gt, arr["trace"]) <= 1e-5
        assert np.array_equal(gt, arr["trace"]), "receiver traces differ"
    assert np.array_equal(gc[::s, ::s, ::s], arr["u_nt"])
    # whole fields, bit for bit
    assert _sha(gc) == doc["sha256_u_nt"], "u^nt differs from the oracle"
    assert _sha(gp) == doc["sha256_u_nt_minus_1"], "u^(nt-1) differs from the oracle"
    n_c = float(np.sqrt((gc.astype(np.float64) ** 2).sum()))
    assert abs(n_c - doc["norm_u_nt"]) <= 1e-12 * max(1.0, doc["norm_u_nt"])
