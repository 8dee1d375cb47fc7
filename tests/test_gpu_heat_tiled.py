"""GPU parity of the register-resident heat time-tiled kernel (sweeph, DESIGN.md §6 G5) against the
CPU oracle O1: every level of the pass lives in the registers of one warp, x neighbours by SHFL,
y neighbours beyond a warp's strip through a boundary-row ring, one CTA barrier per step.

The corners this exercises: ragged tiles in x and y (the output tile is the region shrunk by the
rim HX/HY, so the last tile column/row is partial), grids smaller than one tile, z-chunk edges
(ST_CHUNKS forces many chunks, each with its own 2*T_k*r warm-up), the global z boundary inside a
level's range (levels zero there: Dirichlet), sources on tile rims and domain edges injected in
every redundant copy, receivers sampled only by the owning tile, run composition with remainder
T = 1 passes, snapshots (the SAVE instance), anisotropic spacing, and the full C2 grid.  Bar:
bitwise equality with O1 (the kernel evaluates the canonical per-point order)."""
import numpy as np
import pytest

import workloads as W
from harness import gpu_run, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


def _heat(n, nt, src=(), rec=(), dx=(1.0, 1.0, 1.0), init="uniform"):
    p = W.problem("C2", n=n, nt=nt)
    d = dict(p.__dict__, src=tuple(src), rec=tuple(rec), dx=tuple(dx), init=init,
             f_peak=15.0 if src else None)
    return W.Problem(**d)


def _check(p, tk, splits=None):
    gp, gc, gt = gpu_run(p, t_kernel=tk, splits=splits)
    op, oc, ot = oracle_run(p)
    assert max(rel_l2(gc, oc), rel_l2(gp, op)) <= 1e-5
    assert np.array_equal(gc, oc), f"u^nt max |diff| {np.abs(gc - oc).max()}"
    assert np.array_equal(gp, op), f"u^nt-1 max |diff| {np.abs(gp - op).max()}"
    if ot.size:
        assert np.array_equal(gt, ot), f"trace max |diff| {np.abs(gt - ot).max()}"


@pytest.mark.parametrize("tk", [2, 3, 4])
@pytest.mark.parametrize("n,nt", [((131, 70, 45), 13), ((64, 64, 20), 8), ((5, 3, 4), 9),
                                  ((200, 190, 33), 12), ((57, 121, 9), 11)])
def test_heat_tiled_ragged(tk, n, nt):
    _check(_heat(n, nt), tk)


@pytest.mark.parametrize("tk", [2, 3, 4])
def test_heat_tiled_sources_receivers(tk):
    nx, ny, nz = 97, 83, 29
    src = [(nx // 2, ny // 2, nz // 2), (0, 0, 0), (nx - 1, ny - 1, nz - 1), (55, 3, 14),
           (56, 56, 1), (2, 60, 27), (nx // 2, ny // 2, nz // 2)]
    rec = [(0, 0, 0), (nx - 1, ny - 1, nz - 1), (nx // 2, ny // 2, nz // 2), (56, 55, 3),
           (1, 57, 28), (60, 4, 14)]
    _check(_heat((nx, ny, nz), 14, src=src, rec=rec, init="zero"), tk)


@pytest.mark.parametrize("tk", [3, 4])
@pytest.mark.parametrize("chunks", ["2", "5", "9"])
def test_heat_tiled_z_chunks(monkeypatch, tk, chunks):
    monkeypatch.setenv("ST_CHUNKS", chunks)
    _check(_heat((70, 66, 61), 10, src=[(30, 30, 20), (10, 50, 40)], rec=[(31, 30, 21)]), tk)


@pytest.mark.parametrize("tk", [3, 4])
def test_heat_tiled_run_composition(tk):
    _check(_heat((90, 75, 31), 17), tk, splits=[5, 7, 5])


@pytest.mark.parametrize("tk", [2, 4])
def test_heat_tiled_anisotropic(tk):
    _check(_heat((80, 72, 40), 12, dx=(1.0, 1.25, 0.8)), tk)


@pytest.mark.parametrize("tk,every", [(4, 4), (4, 2), (3, 6)])
def test_heat_tiled_snapshots(tk, every):
    import torch
    from paper_1707_02347_b200 import Stencil
    p = _heat((77, 69, 23), 12, src=[(30, 30, 10)], rec=[(31, 30, 11)])
    st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=tk)
    up, uc = W.initial_fields(p)
    P = st.embed(torch.from_numpy(up).cuda())
    C = st.embed(torch.from_numpy(uc).cuda())
    wav = torch.from_numpy(W.wavelet(p, p.nt)).cuda()
    nsnap = p.nt // every
    snaps = torch.full((nsnap,) + st.shape, float("nan"), device="cuda")
    st.run(P, C, p.nt, src=list(p.src), wavelet=wav, rec=list(p.rec), save_every=every,
           snapshots=snaps)
    st.sync()
    for j in range(1, nsnap + 1):
        _, want, _ = oracle_run(p, nt=j * every)
        assert np.array_equal(st.interior(snaps[j - 1]).cpu().numpy(), want), j
    _, want_c, _ = oracle_run(p)
    assert np.array_equal(st.interior(C).cpu().numpy(), want_c)
    st.close()


@pytest.mark.parametrize("tk", [3, 4])
def test_C2_full_tiled(tk):
    _check(W.problem("C2"), tk)
