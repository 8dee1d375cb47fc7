"""CPU checks of the bench.py contract that need no GPU: the reference arm (the oracle, the one
other place bench.py may run oracle/) prints one JSON line with the keys the driver reads, and
under torchrun the non-zero ranks print nothing and exit 0.  Also: the roofline bookkeeping
(algorithmic bytes per launch) and the kernel naming the bench line reports."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                       text=True, env=e, timeout=300)
    return r


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GPts/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_nonzero_rank_is_silent():
    r = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "3"],
             env={"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_alg_bytes_and_kernel_names():
    import bench
    import workloads as W
    c5, c2 = W.problem("C5"), W.problem("C2")
    assert bench._alg_bytes_per_point_launch(c5, False, 1) == 20      # u^{n-1}, u^n, a, c, u^{n+1}
    assert bench._alg_bytes_per_point_launch(c5, True, 2) == 24       # + one more output level
    assert bench._alg_bytes_per_point_launch(c2, False, 1) == 8
    assert bench._kernel_name(c5, 1).startswith("st::sweep1s_kernel<R=6")
    assert bench._kernel_name(W.problem("C3"), 2).startswith("st::sweepx_kernel<R=4")
    assert bench._kernel_name(W.problem("C4"), 1).startswith("st::sweep1s_kernel<R=8")
