"""GPU parity: the CUDA path (C ABI through the Python binding) vs the CPU oracle, element by
element, on the same seeded inputs (workloads/).

Bar (north_star): relative L2 <= 1e-5 in fp32 for u^{nt}, u^{nt-1} and the receiver traces.
Because both sides evaluate the same canonical per-point order (include/stencil.h, SURVEY
§8(c)) with flushed denormals, we also assert bitwise equality, which is the stronger claim
(any legal schedule reproduces the untiled result exactly)."""
import numpy as np
import pytest

import workloads as W
from harness import gpu_run, oracle_run, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _check(p, t_kernel=1, nt=None, splits=None, bitwise=True):
    gp, gc, gt = gpu_run(p, nt=nt, t_kernel=t_kernel, splits=splits)
    op, oc, ot = oracle_run(p, nt=nt)
    errs = [rel_l2(gc, oc), rel_l2(gp, op)]
    if ot.size:
        errs.append(rel_l2(gt, ot))
    assert max(errs) <= TOL, errs
    assert np.abs(oc).max() > 0
    if bitwise:
        assert np.array_equal(gc, oc), f"max |diff| {np.abs(gc - oc).max()}"
        assert np.array_equal(gp, op)
        assert np.array_equal(gt, ot)


def _wave(name, n, nt, sponge, order=None, src=None, rec=None):
    p = W.problem(name, n=n, nt=nt, sponge=sponge)
    d = dict(p.__dict__)
    if order:
        d["space_order"] = order
    if src is not None:
        d["src"] = tuple(src)
    if rec is not None:
        d["rec"] = tuple(rec)
    return W.Problem(**d)


# ----------------------------------------------------------------------------- C1 / C2 heat
@pytest.mark.parametrize("tk", [1, 2, 4])
def test_C1_heat2d_full(tk):
    _check(W.problem("C1"), t_kernel=tk)


@pytest.mark.parametrize("tk", [1, 2, 4])
def test_heat3d_ragged(tk):
    _check(W.problem("C2", n=(131, 70, 45), nt=13), t_kernel=tk)


@pytest.mark.parametrize("tk", [1, 4])
def test_C2_heat3d_full(tk):
    _check(W.problem("C2"), t_kernel=tk)


@pytest.mark.parametrize("order", [2, 4, 6, 10, 14, 16])
def test_heat3d_orders(order):
    p = W.problem("C2", n=(67, 41, 29), nt=6)
    _check(W.Problem(**{**p.__dict__, "space_order": order}))


# ----------------------------------------------------------------------------- wave
@pytest.mark.parametrize("order", [2, 4, 6, 8, 10, 12, 14, 16])
@pytest.mark.parametrize("tk", [1, 2])
def test_wave_orders_ragged(order, tk):
    n = (97, 75, 60)
    src = [(48, 37, 30), (0, 0, 0), (96, 74, 59), (48, 37, 30)]
    rec = [(1, 2, 3), (48, 37, 30), (95, 70, 2), (63, 31, 30), (64, 32, 31), (30, 60, 58)]
    _check(_wave("C3", n, 17, 8, order=order, src=src, rec=rec), t_kernel=tk)


@pytest.mark.parametrize("order", [10, 12, 16])
@pytest.mark.parametrize("sponge", [6, 0])
def test_wave_undamped_tiles(order, sponge):
    """The static-ring untiled kernel loads the a box only where a tile's plane holds a point
    with a != -1 (a == -1 exactly where damp = 0; the medium kernel's tile flags).  A grid wide
    enough for tiles (64 columns x 24 or 16 rows) that lie wholly inside the sponge-free interior,
    next to tiles and planes that do not, and the same grid with no damping at all (every flag
    set, boundary tiles included); sources in a skipped tile, in a damped tile and on the edge."""
    n = (200, 110, 40)
    src = [(100, 60, 20), (3, 4, 2), (199, 109, 39), (64, 48, 6)]
    rec = [(100, 60, 20), (65, 49, 7), (127, 71, 33), (128, 72, 34), (2, 100, 20), (190, 30, 5)]
    _check(_wave("C5", n, 11, sponge, order=order, src=src, rec=rec), t_kernel=1)


@pytest.mark.parametrize("order", [12, 14, 16])
@pytest.mark.parametrize("dx", [(10.0, 10.0, 10.0), (10.0, 12.5, 8.0)])
def test_wave_isotropic_and_anisotropic_weights(order, dx):
    """The isotropic-weight instance (one weight per k, launched when the per-axis weights are
    bitwise equal: r >= 7) and the general one (anisotropic spacing) both match the oracle."""
    p = _wave("C3", (70, 50, 40), 9, 6, order=order, src=[(35, 25, 20)], rec=[(35, 25, 20), (3, 4, 5)])
    _check(W.Problem(**{**p.__dict__, "dx": dx, "dt": 4e-4}))


@pytest.mark.parametrize("tk", [1, 2])
def test_wave_tiny_grid(tk):
    """Grid smaller than one tile in every direction."""
    _check(_wave("C3", (5, 3, 4), 9, 1, order=4, src=[(2, 1, 1)], rec=[(4, 2, 3)]), t_kernel=tk)


def test_wave_2d():
    p = W.problem("C1", nt=15)
    d = dict(p.__dict__, time_order=2, space_order=8, dt=8e-4, dx=(10.0, 10.0, 10.0), init="zero",
             layers=(1500.0, 2500.0, 3500.0, 4500.0), f_peak=15.0, sponge=10, src=((64, 64, 0),),
             rec=((10, 10, 0), (64, 64, 0)))
    _check(W.Problem(**d))


@pytest.mark.parametrize("tk", [1, 2])
def test_run_composition(tk):
    """run(a) + run(b) + run(c) == run(a+b+c) == oracle (odd chunks exercise the swap path)."""
    p = _wave("C3", (70, 66, 40), 12, 6, src=[(35, 33, 20)], rec=[(35, 33, 20), (10, 10, 10)])
    _check(p, t_kernel=tk, splits=[3, 5, 4])


@pytest.mark.parametrize("tk", [1, 2])
def test_run_composition_reused_medium(tk):
    """Later chunks pass vel = damp = None (the plan keeps the medium of the first chunk) and
    identical src/rec lists (the plan keeps its uploaded tables): still bit-exact."""
    p = _wave("C3", (70, 66, 40), 12, 6, src=[(35, 33, 20)], rec=[(35, 33, 20), (10, 10, 10)])
    gp, gc, gt = gpu_run(p, t_kernel=tk, splits=[3, 5, 4], reuse_medium=True)
    op, oc, ot = oracle_run(p)
    assert np.array_equal(gc, oc) and np.array_equal(gp, op) and np.array_equal(gt, ot)


def test_vel_null_without_medium_is_estate():
    import torch
    from paper_1707_02347_b200 import Stencil
    p = _wave("C3", (40, 36, 30), 4, 4)
    st = Stencil(3, p.n, p.space_order, 2, p.dt, p.dx)
    P, C = st.empty(), st.empty()
    with pytest.raises(RuntimeError, match="ST_ESTATE|medium"):
        st.run(P, C, 2)
    st.close()


def test_nt_zero_is_noop():
    import torch
    from paper_1707_02347_b200 import Stencil
    p = W.problem("C2", n=(20, 20, 20), nt=0)
    st = Stencil(3, p.n, 2, 1, p.dt, p.dx)
    _, uc = W.initial_fields(p)
    C = st.embed(torch.from_numpy(uc).cuda())
    P = st.empty()
    before = C.clone()
    st.run(P, C, 0)
    st.sync()
    assert torch.equal(C, before)


# ----------------------------------------------------------------------------- full sizes
# Full BASELINE grids, in the launch configuration bench.py times (t_kernel as bench), with a
# step count the oracle finishes in seconds; the full step counts are covered by the
# schedule-invariance tests below (bitwise vs the untiled GPU run).
@pytest.mark.parametrize("name,nt,tk", [("C3", 12, 2), ("C5", 6, 1), ("C4", 3, 1)])
def test_full_grid_vs_oracle(name, nt, tk):
    import psutil
    p = W.problem(name)
    need = 10 * 4 * (p.n[0] + 16) * (p.n[1] + 16) * (p.n[2] + 16)   # oracle + generator arrays
    if psutil.virtual_memory().available < need:
        pytest.skip(f"host RAM below {need / 2**30:.0f} GiB for the {name} oracle")
    _check(p, t_kernel=tk, nt=nt)


@pytest.mark.parametrize("name,tk", [("C3", 2), ("C5", 2)])
def test_full_run_schedule_invariance(name, tk):
    """Full grid AND full nt: time-tiled == untiled bitwise; traces too."""
    p = W.problem(name)
    a = gpu_run(p, t_kernel=1)
    b = gpu_run(p, t_kernel=tk)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert np.isfinite(a[1]).all() and np.abs(a[1]).max() > 0


@pytest.mark.parametrize("name,tk,nt", [("C5", 1, 600), ("C3", 2, 300), ("C4", 1, 100)])
def test_run_to_run_determinism(name, tk, nt):
    """Two runs of the bench launch configuration give identical bits (catches shared-memory races
    that the short oracle runs cannot see: the field is non-zero only near the source early on)."""
    p = W.problem(name)
    a = gpu_run(p, nt=nt, t_kernel=tk)
    b = gpu_run(p, nt=nt, t_kernel=tk)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert np.abs(a[1]).max() > 0


# ----------------------------------------------------------------------------- paper replica
@pytest.mark.parametrize("tk", [1, 2])
def test_paper_replica_scaled(tk):
    """Source-free SO8 AWE with the paper's dt, h and Gaussian initial field (NEXT-2 i), ragged grid."""
    _check(W.problem("P256", n=(70, 45, 38), nt=13, sponge=5), t_kernel=tk)


@pytest.mark.parametrize("name,nt", [("P256", 8), ("P384", 4)])
def test_paper_replica_full_grid(name, nt):
    _check(W.problem(name), nt=nt, t_kernel=1)


# ----------------------------------------------------------------------------- snapshots (save mode)
@pytest.mark.parametrize("tk,every,order", [(1, 3, 8), (2, 3, 8), (2, 4, 8), (1, 1, 8),
                                            (1, 3, 12), (2, 2, 12), (1, 2, 16), (2, 4, 16)])
def test_snapshots_match_oracle(tk, every, order):
    """stencil_run_save: snapshot j holds u^{j*every} bit-exactly (oracle run of j*every steps);
    the run's final state is unchanged by saving (SURVEY §8(f) NEXT-2 ii).  SO12/SO16 cover the
    snapshot-store instances of the static-ring untiled kernel and of the exchange pass."""
    import torch
    from paper_1707_02347_b200 import Stencil
    p = _wave("C3", (45, 38, 30), 10, 5, order=order, src=[(22, 19, 15)], rec=[(20, 20, 20)])
    st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=tk)
    up, uc = W.initial_fields(p)
    P = st.embed(torch.from_numpy(up).cuda())
    C = st.embed(torch.from_numpy(uc).cuda())
    vel = st.embed(torch.from_numpy(W.velocity(p)).cuda())
    damp = st.embed(torch.from_numpy(W.damp(p)).cuda())
    wav = torch.from_numpy(W.wavelet(p, p.nt)).cuda()
    nsnap = p.nt // every
    snaps = torch.full((nsnap,) + st.shape, float("nan"), device="cuda")
    st.run(P, C, p.nt, vel=vel, damp=damp, src=list(p.src), wavelet=wav, rec=list(p.rec),
           save_every=every, snapshots=snaps)
    st.sync()
    for j in range(1, nsnap + 1):
        _, want, _ = oracle_run(p, nt=j * every)
        got = st.interior(snaps[j - 1]).cpu().numpy()
        assert np.array_equal(got, want), j
    _, want_c, _ = oracle_run(p)
    assert np.array_equal(st.interior(C).cpu().numpy(), want_c)
    st.close()


# ----------------------------------------------------------------------------- G4 resident 2-D
@pytest.mark.parametrize("resident", ["spb", "1", "2", "off"])
@pytest.mark.parametrize("order,n", [(2, (77, 53, 1)), (8, (64, 40, 1)), (16, (41, 47, 1)),
                                     (4, (128, 128, 1))])
def test_2d_wave_resident_vs_per_step(monkeypatch, resident, order, n):
    """2-D wave through the whole-run cluster-resident kernel (G4: rows split over up to 8 CTAs,
    DSMEM halo push every spb steps, redundant halo rows in between; ST_RES_SPB caps spb) and,
    with ST_NO_RESIDENT, through the per-step sweeps: ragged odd widths, sources on the first/last
    column (pair lo/hi element) and on CTA-boundary rows, duplicate sources, receivers on corners
    -- bit-exact vs the oracle either way."""
    if resident == "off":
        monkeypatch.setenv("ST_NO_RESIDENT", "1")
    elif resident != "spb":
        monkeypatch.setenv("ST_RES_SPB", resident)
    nx, ny, _ = n
    p = W.problem("C1", n=n, nt=13)
    d = dict(p.__dict__, time_order=2, space_order=order, dt=8e-4, dx=(10.0, 12.0, 10.0), init="zero",
             layers=(1500.0, 2500.0, 3500.0, 4500.0), f_peak=15.0, sponge=6,
             src=((nx // 2, ny // 2, 0), (0, 3, 0), (nx - 1, ny - 2, 0), (nx // 2, ny // 2, 0),
                  (5, 7, 0), (6, 8, 0), (nx - 3, 16, 0)),
             rec=((0, 0, 0), (nx - 1, ny - 1, 0), (nx // 2, ny // 2, 0), (1, ny - 1, 0)))
    _check(W.Problem(**d))


@pytest.mark.parametrize("resident", [True, False])
def test_2d_heat_resident_eigenmode(monkeypatch, resident):
    if not resident:
        monkeypatch.setenv("ST_NO_RESIDENT", "1")
    p = W.problem("C1", n=(99, 128, 1), nt=37)
    _check(W.Problem(**dict(p.__dict__, init="eigenmode")))


# ----------------------------------------------------------------------------- band/interior split
@pytest.mark.parametrize("order", [8, 12, 16])
def test_t1_band_interior_split(monkeypatch, order):
    """ST_SPLIT_T1: every step as lo band + hi band + interior launches (the split the
    library-owned NCCL exchange overlaps with the transfer, include/stencil.h), bit-exact, with
    sources and receivers on band planes."""
    monkeypatch.setenv("ST_SPLIT_T1", "1")
    r = order // 2
    n = (70, 50, 40)
    src = [(35, 25, 20), (3, 4, r - 1), (66, 45, n[2] - r)]
    rec = [(10, 10, 0), (20, 30, r), (40, 20, n[2] - 1), (35, 25, n[2] - r - 1)]
    _check(_wave("C3", n, 9, 5, order=order, src=src, rec=rec))


# ----------------------------------------------------------------------------- library-owned exchange
@pytest.mark.parametrize("t_comm,t_kernel,heat", [(1, 1, False), (3, 1, False), (4, 2, False),
                                                  (8, 4, True), (6, 3, True)])
def test_lib_exchange_single_rank(t_comm, t_kernel, heat):
    """st_config.nccl_id on a one-rank plan: the library-owned time loop (T_c periods, NCCL group
    calls with no neighbours, comm-stream joins, trace zeroing and ncclAllReduce) runs for real on
    one GPU and stays bit-exact; the multi-rank transfers need >= 2 GPUs."""
    import torch
    from paper_1707_02347_b200 import Stencil
    from paper_1707_02347_b200.stencil import nccl_unique_id
    p = _wave("C3", (60, 44, 36), 11, 5, src=[(30, 22, 18)], rec=[(30, 22, 18), (5, 40, 2), (59, 0, 35)])
    if heat:   # the heat time-tiled kernel (sweeph) inside the library's period loop
        p = W.Problem(**{**W.problem("C2", n=(60, 44, 36), nt=19).__dict__, "f_peak": 15.0,
                         "src": p.src, "rec": p.rec})
    st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=t_kernel,
                 t_comm=t_comm, nccl_id=nccl_unique_id())
    assert st.lib_exchange
    up, uc = W.initial_fields(p)
    P = st.embed(torch.from_numpy(up).cuda())
    C = st.embed(torch.from_numpy(uc).cuda())
    vel = st.embed(torch.from_numpy(W.velocity(p)).cuda()) if not heat else None
    damp = st.embed(torch.from_numpy(W.damp(p)).cuda()) if not heat else None
    wav = torch.from_numpy(W.wavelet(p, p.nt)).cuda()
    trace = torch.full((p.nt, len(p.rec)), float("nan"), device="cuda")   # the library zeroes it
    st.run(P, C, p.nt, vel=vel, damp=damp, src=list(p.src), wavelet=wav, rec=list(p.rec), trace=trace)
    st.sync()
    op, oc, ot = oracle_run(p)
    assert np.array_equal(st.interior(C).cpu().numpy(), oc)
    assert np.array_equal(st.interior(P).cpu().numpy(), op)
    assert np.array_equal(trace.cpu().numpy(), ot)
    st.close()


# ----------------------------------------------------------------------------- CUDA graph replay (bench C1 path)
@pytest.mark.parametrize("wave", [False, True])
def test_cuda_graph_replay_2d(wave):
    """bench.py replays the 2-D step (stencil_run_from the stored initial pair: one resident
    launch) as a CUDA graph captured on the plan's stream: the captured library launches must
    reproduce the oracle bit for bit on every replay (heat: C1; wave: 2-D SO8 with a source,
    medium derived inside the step), and the stored initial pair stays untouched."""
    import torch
    from paper_1707_02347_b200.dist import SlabRunner
    if wave:
        p = W.problem("C1", n=(96, 80, 1), nt=15)
        p = W.Problem(**dict(p.__dict__, time_order=2, space_order=8, dt=8e-4, dx=(10.0, 10.0, 10.0),
                             init="zero", layers=(1500.0, 2500.0, 3500.0, 4500.0), f_peak=15.0,
                             sponge=6, src=((48, 40, 0),)))
    else:
        p = W.problem("C1")
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    try:
        r = SlabRunner(p, t_kernel=1, device=0)
        host = r.host_inputs(p.nt, pin=False)
        dev = r.to_device(host, p.nt)

        init = (dev["_init_prev"].clone(), dev["_init_cur"].clone())

        def step():
            r.run_from_init(dev, p.nt)
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        op, oc, _ = oracle_run(p)
        for _ in range(3):
            dev["u_cur"].zero_()
            g.replay()
            torch.cuda.synchronize()
            assert np.array_equal(r.stencil.interior(dev["u_cur"]).cpu().numpy(), oc)
            assert np.array_equal(r.stencil.interior(dev["u_prev"]).cpu().numpy(), op)
        assert torch.equal(init[1], dev["_init_cur"]) and torch.equal(init[0], dev["_init_prev"])
        r.stencil.close()
    finally:
        torch.cuda.set_stream(torch.cuda.default_stream())


# ----------------------------------------------------------------------------- stencil_run_from
@pytest.mark.parametrize("case", ["heat2d", "wave2d", "wave2d_steps", "wave3d", "heat3d_tk4"])
def test_run_from_kept_initial_pair(monkeypatch, case):
    """stencil_run_from: outputs start as NaN garbage, the run starts from the kept initial pair
    (resident 2-D kernel loads it itself; per-step 2-D sweeps and 3-D plans copy it first); the
    result is the oracle's bit for bit, twice in a row (repeated simulations), and the initial
    fields are unchanged.  An initial field overlapping an output is ST_EINVAL."""
    import torch
    from paper_1707_02347_b200 import Stencil
    from paper_1707_02347_b200._lib import StencilError
    tk = 1
    if case == "heat2d":
        p = W.problem("C1", n=(99, 128, 1), nt=23)
    elif case.startswith("wave2d"):
        if case == "wave2d_steps":
            monkeypatch.setenv("ST_NO_RESIDENT", "1")
        p = W.problem("C1", n=(77, 53, 1), nt=13)
        p = W.Problem(**dict(p.__dict__, time_order=2, space_order=8, dt=8e-4, dx=(10.0, 12.0, 10.0),
                             init="zero", layers=(1500.0, 2500.0, 3500.0, 4500.0), f_peak=15.0,
                             sponge=6, src=((38, 26, 0), (0, 3, 0)), rec=((0, 0, 0), (76, 52, 0))))
    elif case == "wave3d":
        p = _wave("C3", (45, 38, 30), 7, 5, src=[(22, 19, 15)], rec=[(20, 20, 20)])
    else:
        p, tk = W.problem("C2", n=(64, 48, 40), nt=10), 4
    st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=tk)
    up, uc = W.initial_fields(p)
    I0 = st.embed(torch.from_numpy(up).cuda())
    I1 = st.embed(torch.from_numpy(uc).cuda())
    keep = (I0.clone(), I1.clone())
    wave = p.time_order == 2
    vel = st.embed(torch.from_numpy(W.velocity(p)).cuda()) if wave else None
    damp = st.embed(torch.from_numpy(W.damp(p)).cuda()) if wave else None
    wav = torch.from_numpy(W.wavelet(p, p.nt)).cuda() if p.src else None
    op, oc, ot = oracle_run(p)
    P, C = st.empty(), st.empty()
    for _ in range(2):
        P.fill_(float("nan")); C.fill_(float("nan"))
        tr = st.run(P, C, p.nt, vel=vel, damp=damp, src=list(p.src), wavelet=wav, rec=list(p.rec),
                    init=(I0 if wave else None, I1))
        st.sync()
        assert np.array_equal(st.interior(C).cpu().numpy(), oc)
        assert np.array_equal(st.interior(P).cpu().numpy(), op)
        if p.rec:
            assert np.array_equal(tr.cpu().numpy(), ot)
    assert torch.equal(I0, keep[0]) and torch.equal(I1, keep[1])
    with pytest.raises(StencilError):       # init_cur overlapping u_prev
        st.run(P, C, 1, vel=vel, damp=damp, src=list(p.src), wavelet=wav, rec=list(p.rec),
               init=(I0 if wave else None, P))
    st.close()


# ----------------------------------------------------------------------------- pipelined e2e (bench)
@pytest.mark.parametrize("case", ["wave3d", "heat2d"])
def test_host_pipelined_runs(case):
    """SlabRunner.run_host_pipelined (bench.py's e2e): uploads, runs and read-backs of successive
    simulations overlap on three streams over two device slots; every step's host result is the
    oracle's bit for bit (checked on the last two steps, one per slot)."""
    import torch
    from paper_1707_02347_b200.dist import SlabRunner
    if case == "wave3d":
        p = _wave("C3", (45, 38, 30), 9, 5, src=[(22, 19, 15)], rec=[(20, 20, 20), (3, 4, 5)])
    else:
        p = W.problem("C1", n=(99, 128, 1), nt=23)
    r = SlabRunner(p, t_kernel=1, device=0)
    host = r.host_inputs(p.nt, pin=True)
    devs = [r.to_device(host, p.nt), r.to_device(host, p.nt)]
    streams = (torch.cuda.Stream(), torch.cuda.Stream())
    op, oc, ot = oracle_run(p)
    for steps in (1, 2, 5):
        for d in devs:
            d["u_cur"].fill_(float("nan"))
        out = r.run_host_pipelined(host, devs, p.nt, steps, streams)
        torch.cuda.synchronize()
        assert np.array_equal(out[0].numpy().reshape(oc.shape), oc)
        if p.rec:
            assert np.array_equal(out[1].numpy(), ot)
        if steps > 1:           # the other slot's result too
            other = r._out_bufs[(steps - 2) % 2]
            assert np.array_equal(other[0].numpy().reshape(oc.shape), oc)
    r.stencil.close()
