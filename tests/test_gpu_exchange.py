"""GPU parity of the exchange-tiled T_k = 2 kernel (sweept.cuh) against the CPU oracle, bit for
bit, on shapes that force its scheduling corner cases: band cuts (ST_EXCH_SLOTS caps the tiles a
band may hold, so small grids get many bands, down to one tile row per band), several z-chunks
(ST_EXCH_CHUNKS), ragged x/y/z extents, sources and receivers on band-cut rows and chunk-boundary
planes, odd step counts (a final T = 1 pass), and repeated runs of one plan (progress counters and
ticket carried across launches)."""
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


@pytest.mark.parametrize("order,n,nt,slots,chunks", [
    (2, (70, 50, 20), 9, 2, 4),
    (4, (96, 61, 31), 8, 3, 2),
    (8, (150, 100, 40), 9, 6, 3),
    (8, (150, 100, 40), 10, 1000, 1),
    (12, (130, 90, 33), 7, 3, 2),
    (12, (130, 90, 33), 6, 4, 1),
    (14, (100, 70, 36), 5, 2, 2),
])
def test_exchange_bands_chunks(monkeypatch, order, n, nt, slots, chunks):
    monkeypatch.setenv("ST_EXCH_SLOTS", str(slots))
    monkeypatch.setenv("ST_EXCH_CHUNKS", str(chunks))
    r = order // 2
    nx, ny, nz = n
    # sources / receivers on rows and planes next to tile-row, band and chunk boundaries
    zc = (nz + chunks - 1) // chunks          # first plane of the second chunk
    zc = min(zc, nz - 1)
    src = [(nx // 2, ny // 2, nz // 2), (1, 14 - r, zc), (nx - 2, 13, 2)]
    rec = [(nx // 2, 14, nz // 2), (3, 14 - r - 1, zc - 1), (nx - 1, ny - 1, nz - 1),
           (0, 27, 1), (63, 28, nz // 2), (64, 14 + 14 - r, 5)]
    _same(_wave(n, nt, order, src=src, rec=rec))


def test_exchange_heat_bands(monkeypatch):
    monkeypatch.setenv("ST_EXCH_SLOTS", "5")
    monkeypatch.setenv("ST_EXCH_CHUNKS", "3")
    _same(W.problem("C2", n=(131, 70, 45), nt=11))


def test_exchange_repeated_runs(monkeypatch):
    """One plan, several runs: the ticket and progress words carry over between launches."""
    monkeypatch.setenv("ST_EXCH_SLOTS", "4")
    p = _wave((90, 60, 30), 12, 8, rec=[(45, 30, 15), (2, 10, 3)])
    _same(p, splits=[4, 2, 6])
