"""O2 (the paper's skewed time-tiled schedule) reproduces O1 (the untiled loop
nest) BIT-EXACTLY -- "every point's operands are identical values under any
legal order" -- and an under-skewed tiling (skew < radius) does
not.  Also checks the buffered-time reading Q13 (modulo-B buffers)."""
import itertools

import numpy as np
import pytest

import oracle
import workloads as W


def _case(name, n, nt, sponge=None):
    return W.problem(name, n=n, nt=nt, sponge=sponge)


def _with_points(p, src, rec):
    return W.Problem(**{**p.__dict__, "src": tuple(src), "rec": tuple(rec)})


CASES = [
    ("heat2d", lambda: _case("C1", (23, 17, 1), 9)),
    ("heat3d", lambda: _case("C2", (13, 11, 10), 7)),
    ("wave_so8", lambda: _with_points(_case("C3", (14, 13, 12), 9, sponge=3),
                                       [(7, 6, 5), (2, 3, 9)], [(1, 1, 1), (7, 6, 5), (12, 11, 10)])),
    ("wave_so4", lambda: _with_points(W.Problem(**{**_case("C3", (12, 15, 11), 10, sponge=2).__dict__,
                                                   "space_order": 4}),
                                       [(6, 7, 5)], [(6, 7, 5), (0, 14, 10)])),
]


@pytest.mark.parametrize("case", [c[0] for c in CASES])
@pytest.mark.parametrize("Tt,Tz,Ty,B", [(1, 4, 4, 2), (2, 4, 8, 3), (4, 8, 4, 2), (4, 8, 8, 6),
                                         (8, 16, 16, 3), (100, 8, 8, 2)])
def test_skewed_equals_untiled_bitwise(case, Tt, Tz, Ty, B):
    p = dict(CASES)[case]()
    P1, C1, t1 = oracle.run_problem(p, kind="untiled")
    P2, C2, t2 = oracle.run_problem(p, kind="skewed", Tt=Tt, Tz=Tz, Ty=Ty, B=B)
    assert np.array_equal(C1, C2) and np.array_equal(P1, P2)
    assert np.array_equal(t1, t2)
    assert np.abs(C1).max() > 0


@pytest.mark.parametrize("case", ["heat3d", "wave_so8"])
def test_underskewed_tiling_differs(case):
    """Negative control: skew < radius breaks the dependences -> mismatch."""
    p = dict(CASES)[case]()
    _, C1, _ = oracle.run_problem(p, kind="untiled")
    for skew in range(0, p.radius):
        _, C2, _ = oracle.run_problem(p, kind="skewed", Tt=4, Tz=4, Ty=4, B=3, skew=skew)
        assert not np.array_equal(C1, C2), skew


def test_buffer_smaller_than_time_tile_is_legal():
    """Q13: with skew >= r, B = 2 (< time tile) is still bit-exact; the paper's 'tile <= buffer'
     is sufficient, not necessary."""
    p = dict(CASES)["wave_so8"]()
    _, C1, _ = oracle.run_problem(p, kind="untiled")
    for Tt in (3, 5, 9):
        _, C2, _ = oracle.run_problem(p, kind="skewed", Tt=Tt, Tz=6, Ty=5, B=2)
        assert np.array_equal(C1, C2)


def test_run_composition_bitwise():
    """run(a); run(b) == run(a+b) (step0 indexes the wavelet), O1."""
    p = dict(CASES)["wave_so8"]()
    r = p.radius
    import workloads as Wm
    vel = oracle.embed(Wm.velocity(p), 3, r); vel[vel == 0] = 1500
    a, c = oracle.medium(vel, oracle.embed(Wm.damp(p), 3, r), p.dt)
    wv = Wm.wavelet(p, p.nt)
    cf = oracle.fd_weights(p.space_order)

    def fresh():
        return oracle.embed(np.zeros((p.n[2], p.n[1], p.n[0])), 3, r), oracle.embed(np.zeros((p.n[2], p.n[1], p.n[0])), 3, r)
    P, C = fresh()
    ta = oracle.run_untiled(3, p.n, p.space_order, cf, p.dx, 2, p.dt, P, C, a, c, nt=4, step0=0,
                            src=p.src, wavelet=wv, rec=p.rec)
    tb = oracle.run_untiled(3, p.n, p.space_order, cf, p.dx, 2, p.dt, P, C, a, c, nt=5, step0=4,
                            src=p.src, wavelet=wv, rec=p.rec)
    P2, C2 = fresh()
    tt = oracle.run_untiled(3, p.n, p.space_order, cf, p.dx, 2, p.dt, P2, C2, a, c, nt=9, step0=0,
                            src=p.src, wavelet=wv, rec=p.rec)
    assert np.array_equal(C, C2) and np.array_equal(P, P2)
    assert np.array_equal(np.concatenate([ta, tb]), tt)


# ----------------------------------------------------------------------------- O3: z-slab schedule
@pytest.mark.parametrize("time_order,order", [(2, 8), (2, 4), (1, 2)])
@pytest.mark.parametrize("nslab,tc", [(2, 1), (3, 2), (4, 3), (2, 4)])
def test_slab_schedule_equals_untiled(time_order, order, nslab, tc):
    """O3 (the library's z-slab decomposition: ghost planes r*T_c of u^n and r*(T_c-1) of u^{n-1}
    refreshed every T_c steps, redundant shrinking regions, sources injected in ghost planes too,
    owner-only receivers) reproduces O1 bit for bit (S:458 pattern)."""
    r = order // 2
    nz = nslab * max(4, r * tc)
    if time_order == 2:
        p = W.problem("C3", n=(14, 12, nz), nt=11, sponge=2)
        p = W.Problem(**{**p.__dict__, "space_order": order,
                         "src": ((7, 6, nz // nslab - 1), (3, 2, nz // 2)),
                         "rec": ((7, 6, nz // nslab), (1, 1, 0), (13, 11, nz - 1))})
    else:
        p = W.problem("C2", n=(13, 11, nz), nt=9)
    want = oracle.run_problem(p)
    got = oracle.run_problem(p, kind="slabs", nslab=nslab, tc=tc)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_slab_schedule_shallow_ghost_differs():
    """Negative control: a ghost zone one plane shallower than r*T_c changes the result."""
    p = W.problem("C2", n=(13, 11, 24), nt=9)
    want = oracle.run_problem(p)
    got = oracle.run_problem(p, kind="slabs", nslab=3, tc=3, ghost=2)
    assert not np.array_equal(got[1], want[1])
