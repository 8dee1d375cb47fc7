"""The library's z-slab path (rank/nranks plans, ghost planes, shrinking valid ranges, sources in
ghost zones, owner-only receivers) on ONE GPU: N slab plans run one after another in a single
process; between periods their ghost planes are exchanged with the same exchange plan as the
NCCL path (dist.local_exchange).  No kernel ever waits on another, so sequential execution is
exact.  The assembled owned planes must equal the single-domain oracle bit-for-bit."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


def _problem(order=8, nz=48):
    p = W.problem("C5", n=(70, 45, nz), nt=13, sponge=5)
    return W.Problem(**{**p.__dict__, "space_order": order,
                        "src": ((35, 22, nz // 2), (10, 40, nz // 2 - 1)),
                        "rec": ((35, 22, nz // 2), (35, 22, nz // 2 - 1), (1, 1, 0), (69, 44, nz - 1),
                                (33, 20, nz // 4))})


def _run_slabs(p, world, tk, tc, no_swap=False):
    from paper_1707_02347_b200 import Stencil
    from paper_1707_02347_b200.dist import local_exchange
    plans, fields = [], []
    wav = torch.from_numpy(W.wavelet(p)).cuda()
    for rk in range(world):
        st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=tk, t_comm=tc,
                     rank=rk, nranks=world, no_swap=no_swap)
        has_lo, has_hi = rk > 0, rk < world - 1
        z0 = st.z_range[0]
        lo = z0 - (st.G if has_lo else 0)
        hi = z0 + st.nz_local + (st.G if has_hi else 0)
        gl = z0 - lo
        f = {}
        up, uc = W.initial_fields(p, lo, hi)
        f["u_prev"] = st.embed(torch.from_numpy(up).cuda(), ghost_lo=gl)
        f["u_cur"] = st.embed(torch.from_numpy(uc).cuda(), ghost_lo=gl)
        if p.time_order == 2:
            f["vel"] = st.embed(torch.from_numpy(W.velocity(p, lo, hi)).cuda(), ghost_lo=gl)
            f["damp"] = st.embed(torch.from_numpy(W.damp(p, lo, hi)).cuda(), ghost_lo=gl)
        f["trace"] = torch.zeros((p.nt, len(p.rec)), dtype=torch.float32, device="cuda")
        plans.append(st)
        fields.append(f)
    G, nzl = plans[0].G, plans[0].nz_local
    done = 0
    while done < p.nt:
        n = min(tc, p.nt - done)
        local_exchange(fields, G, nzl, p.radius, n, need_prev=p.time_order == 2)
        for st, f in zip(plans, fields):
            first = done == 0           # later chunks reuse the plan's medium (vel = NULL)
            st.run(f["u_prev"], f["u_cur"], n, vel=f.get("vel") if first else None,
                   damp=f.get("damp") if first else None, step0=done,
                   src=list(p.src), wavelet=wav, rec=list(p.rec), trace=f["trace"][done:done + n])
            if st.swapped():            # no_swap plans: exchange references, as SlabRunner does
                assert no_swap
                f["u_prev"], f["u_cur"] = f["u_cur"], f["u_prev"]
        done += n
    torch.cuda.synchronize()
    P = np.concatenate([st.interior(f["u_prev"]).cpu().numpy() for st, f in zip(plans, fields)])
    C = np.concatenate([st.interior(f["u_cur"]).cpu().numpy() for st, f in zip(plans, fields)])
    T = sum(f["trace"] for f in fields).cpu().numpy()
    for st in plans:
        st.close()
    return P, C, T


@pytest.mark.parametrize("world,tk,tc", [(2, 1, 1), (2, 1, 3), (3, 2, 2), (4, 2, 2), (2, 2, 6), (4, 1, 3),
                                          (8, 1, 1)])
def test_emulated_slabs_bitwise(world, tk, tc):
    p = _problem(nz=64 if world == 8 else 48)
    got = _run_slabs(p, world, tk, tc)
    want = oracle.run_problem(p)
    assert np.abs(want[1]).max() > 0
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@pytest.mark.parametrize("world,tk,tc", [(2, 1, 1), (4, 1, 1), (3, 2, 2), (2, 1, 3)])
def test_emulated_slabs_no_swap(world, tk, tc):
    """SlabRunner's mode: no_swap plans (odd pass counts return the pair swapped, the caller swaps
    references), medium derived on the first chunk only."""
    p = _problem()
    got = _run_slabs(p, world, tk, tc, no_swap=True)
    want = oracle.run_problem(p)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def _run_fused(p, world, steps_per_sim=None, sims=1):
    """Fused halo push on one GPU: N no_swap slab plans whose peers are the other plans' buffers
    (same process), run one step each in rank order.  The initial ghost planes come from the
    seeded global fields (embedded with the slab's ghosts); there is no exchange call at all.
    sims > 1 repeats the simulation from the initial state with the same plans (the counters keep
    counting, as in the bench's warm-up + timed simulations)."""
    from paper_1707_02347_b200 import Stencil
    plans, fields, init = [], [], []
    wav = torch.from_numpy(W.wavelet(p)).cuda()
    for rk in range(world):
        st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=1, t_comm=1,
                     rank=rk, nranks=world, no_swap=True)
        z0 = st.z_range[0]
        lo = z0 - (st.G if rk > 0 else 0)
        hi = z0 + st.nz_local + (st.G if rk < world - 1 else 0)
        gl = z0 - lo
        f = {}
        up, uc = W.initial_fields(p, lo, hi)
        f["u_prev"] = st.embed(torch.from_numpy(up).cuda(), ghost_lo=gl)
        f["u_cur"] = st.embed(torch.from_numpy(uc).cuda(), ghost_lo=gl)
        if p.time_order == 2:
            f["vel"] = st.embed(torch.from_numpy(W.velocity(p, lo, hi)).cuda(), ghost_lo=gl)
            f["damp"] = st.embed(torch.from_numpy(W.damp(p, lo, hi)).cuda(), ghost_lo=gl)
        f["trace"] = torch.zeros((p.nt, len(p.rec)), dtype=torch.float32, device="cuda")
        init.append((f["u_prev"].clone(), f["u_cur"].clone()))
        plans.append(st)
        fields.append(f)
    ab = [(f["u_prev"], f["u_cur"]) for f in fields]
    for rk, st in enumerate(plans):
        for side, peer in ((0, rk - 1), (1, rk + 1)):
            if 0 <= peer < world:
                st.set_peer(side, ab[rk][0], ab[rk][1], ab[peer][0].data_ptr(), ab[peer][1].data_ptr(),
                            plans[peer].peer_counters())
    for sim in range(sims):
        for f, (ip, ic) in zip(fields, init):
            f["u_prev"].copy_(ip)
            f["u_cur"].copy_(ic)
            f["trace"].zero_()
        for n in range(p.nt):
            for st, f in zip(plans, fields):
                st.run(f["u_prev"], f["u_cur"], 1, vel=f["vel"] if n == 0 else None,
                       damp=f["damp"] if n == 0 else None, step0=n, src=list(p.src), wavelet=wav,
                       rec=list(p.rec), trace=f["trace"][n:n + 1])
                if st.swapped():
                    f["u_prev"], f["u_cur"] = f["u_cur"], f["u_prev"]
    torch.cuda.synchronize()
    P = np.concatenate([st.interior(f["u_prev"]).cpu().numpy() for st, f in zip(plans, fields)])
    C = np.concatenate([st.interior(f["u_cur"]).cpu().numpy() for st, f in zip(plans, fields)])
    T = sum(f["trace"] for f in fields).cpu().numpy()
    for st in plans:
        st.close()
    return P, C, T


@pytest.mark.parametrize("world,order,sims", [(2, 8, 1), (3, 12, 1), (4, 4, 2), (4, 16, 1)])
def test_fused_halo_push_bitwise(world, order, sims):
    """NEXT-1: the sweep stores its band planes straight into the neighbours' ghost zones and
    signals them; the next step's producer waits for the counters.  Bit-exact vs the oracle."""
    p = _problem(order=order, nz=48)
    got = _run_fused(p, world, sims=sims)
    want = oracle.run_problem(p)
    assert np.abs(want[1]).max() > 0
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@pytest.mark.parametrize("world,order", [(2, 8), (3, 12)])
def test_fused_halo_push_ipc_processes(world, order, tmp_path):
    """The fused push across PROCESSES (one per rank, all on cuda:0): peers' buffers and counters
    are CUDA IPC mappings (stencil_ipc_export/open), the ranks take turns step by step (gloo
    barriers; no kernel waits on an unfinished one).  Bit-exact vs the oracle."""
    import os
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ipc_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(rk), str(world), str(port), str(tmp_path),
                               str(order), "48"], stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for rk in range(world)]
    outs = []
    try:
        for pr in procs:
            outs.append(pr.communicate(timeout=240)[0].decode(errors="replace"))
    finally:
        for pr in procs:
            if pr.poll() is None:
                pr.kill()
    for rk, (pr, out) in enumerate(zip(procs, outs)):
        assert pr.returncode == 0, f"rank {rk} failed:\n{out[-3000:]}"
    p = _problem(order=order, nz=48)
    res = [np.load(tmp_path / f"rank{rk}.npz") for rk in range(world)]
    got = (np.concatenate([r["P"] for r in res]), np.concatenate([r["C"] for r in res]),
           sum(r["T"] for r in res))
    want = oracle.run_problem(p)
    assert np.abs(want[1]).max() > 0
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_fused_halo_push_rejects_bad_plans():
    from paper_1707_02347_b200 import Stencil
    from paper_1707_02347_b200._lib import StencilError
    p = _problem()
    st = Stencil(3, p.n, 8, 2, p.dt, p.dx, t_kernel=1, t_comm=1, rank=0, nranks=2)   # no no_swap
    a, b = st.empty(), st.empty()
    with pytest.raises(StencilError, match="ST_NO_SWAP"):
        st.set_peer(1, a, b, a.data_ptr(), b.data_ptr(), st.peer_counters())
    st.close()
    st = Stencil(3, p.n, 8, 2, p.dt, p.dx, t_kernel=1, t_comm=2, rank=0, nranks=2, no_swap=True)
    with pytest.raises(StencilError, match="t_comm"):
        st.set_peer(1, a, b, a.data_ptr(), b.data_ptr(), st.peer_counters())
    st.close()
    st = Stencil(3, p.n, 8, 2, p.dt, p.dx, t_kernel=1, t_comm=1, rank=0, nranks=2, no_swap=True)
    with pytest.raises(StencilError, match="neighbour"):
        st.set_peer(0, a, b, a.data_ptr(), b.data_ptr(), st.peer_counters())   # rank 0 has no lo
    st.close()


def test_ghost_deeper_than_slab_rejected():
    from paper_1707_02347_b200 import Stencil
    from paper_1707_02347_b200._lib import ST_EINVAL, StencilError
    p = _problem()
    with pytest.raises(StencilError) as e:
        Stencil(3, p.n, 8, 2, p.dt, p.dx, t_kernel=1, t_comm=4, rank=0, nranks=4)   # 16 > 12 planes
    assert e.value.status == ST_EINVAL


@pytest.mark.parametrize("order", [2, 12, 16])
def test_emulated_slabs_orders(order):
    p = _problem(order=order, nz=64)
    got = _run_slabs(p, 2, 1, 2)
    want = oracle.run_problem(p)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@pytest.mark.parametrize("order,tc", [(12, 1), (16, 2)])
def test_emulated_slabs_undamped_tiles(order, tc):
    """z-slab plans on a grid with tiles wholly inside the sponge-free interior: the a == -1 tile
    flags (a box not loaded) are per slab plane, ghost planes included."""
    p = W.problem("C5", n=(200, 80, 48), nt=9, sponge=5)
    p = W.Problem(**{**p.__dict__, "space_order": order, "src": ((100, 40, 24), (70, 30, 23)),
                     "rec": ((100, 40, 24), (65, 25, 23), (1, 1, 0), (199, 79, 47))})
    got = _run_slabs(p, 2, 1, tc)
    want = oracle.run_problem(p)
    assert np.abs(want[1]).max() > 0
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@pytest.mark.parametrize("world,tk,tc", [(2, 4, 4), (3, 3, 6), (2, 2, 4), (4, 4, 8)])
def test_emulated_slabs_heat_tiled(world, tk, tc):
    """Heat z-slabs on the register-resident time-tiled kernel (sweeph): ghost zones of depth
    r*T_c, passes over shrinking plane ranges that start inside a neighbour's ghost zone (levels
    are computed there, not zeroed), sources in ghost zones, owner-only receivers."""
    nz = 48 if world == 3 else 64
    p = W.problem("C2", n=(70, 45, nz), nt=17)
    p = W.Problem(**{**p.__dict__, "f_peak": 15.0,
                     "src": ((35, 22, nz // 2), (10, 40, nz // 2 - 1), (5, 5, 1)),
                     "rec": ((35, 22, nz // 2), (1, 1, 0), (69, 44, nz - 1), (33, 20, nz // 4))})
    got = _run_slabs(p, world, tk, tc)
    want = oracle.run_problem(p)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
