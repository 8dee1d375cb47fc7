"""GPU parity of the time-tiled T_k = 2 exchange pass (sweepx.cuh: L1 tiles compute u^{n+1} and
publish per-plane progress, L2 tiles on the grid skewed r rows up compute u^{n+2} from the L1
tiles' stores) against the CPU oracle, bit for bit, on shapes that force its scheduling corner
cases: several z-chunks (ST_EXCH_CHUNKS; a chunk's L1 tiles also compute the r planes on each
side), ragged x/y/z extents, sources and receivers on tile-row boundaries and on the skewed L2 rows
and chunk-boundary planes, odd step counts (a final T = 1 pass), and repeated runs of one plan
(progress words and ticket carried across launches)."""
from __future__ import annotations

import numpy as np
import pytest

import workloads as W
from harness import gpu_run, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


def _wave(n, nt, order, sponge=3, src=None, rec=None):
    p = W.problem("C3", n=n, nt=nt, sponge=sponge)
    return W.Problem(**{**p.__dict__, "space_order": order,
                        "src": tuple(src) if src is not None else p.src,
                        "rec": tuple(rec) if rec is not None else ()})


def _same(p, **kw):
    gp, gc, gt = gpu_run(p, t_kernel=2, **kw)
    op, oc, ot = oracle_run(p)
    err = max(rel_l2(gc, oc), rel_l2(gp, op), rel_l2(gt, ot) if ot.size else 0.0)
    assert err <= 1e-5, err
    assert np.array_equal(gc, oc), f"u^nt differs (rel-L2 {rel_l2(gc, oc):.3e})"
    assert np.array_equal(gp, op), f"u^(nt-1) differs (rel-L2 {rel_l2(gp, op):.3e})"
    assert np.array_equal(gt, ot), "receiver traces differ"


@pytest.mark.parametrize("order,n,nt,chunks", [
    (6, (96, 61, 31), 8, 2),
    (8, (150, 100, 40), 9, 3),
    (8, (150, 100, 40), 10, 1),
    (12, (130, 90, 33), 7, 2),
    (12, (130, 90, 33), 6, 1),
    (14, (100, 70, 36), 5, 2),
    (16, (70, 52, 34), 5, 3),
])
def test_exchange_chunks_and_edges(monkeypatch, order, n, nt, chunks):
    monkeypatch.setenv("ST_EXCH_CHUNKS", str(chunks))
    r = order // 2
    nx, ny, nz = n
    zc = min((nz + chunks - 1) // chunks, nz - 1)     # first plane of the second chunk
    # rows at L1 tile-row edges (multiples of 16 and 24) and at the skewed L2 edges (minus r)
    src = [(nx // 2, ny // 2, nz // 2), (1, 24 - r, zc), (nx - 2, 16, 2)]
    rec = [(nx // 2, 24, nz // 2), (3, 24 - r - 1, zc - 1), (nx - 1, ny - 1, nz - 1),
           (0, 16 - r, 1), (63, 48 - r, nz // 2), (64, 47, 5)]
    _same(_wave(n, nt, order, src=src, rec=rec))


def test_exchange_repeated_runs():
    """One plan, several runs: the ticket and progress words carry over between launches."""
    p = _wave((90, 60, 30), 12, 8, rec=[(45, 30, 15), (2, 10, 3)])
    _same(p, splits=[4, 2, 6])
