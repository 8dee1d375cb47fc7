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
        f["vel"] = st.embed(torch.from_numpy(W.velocity(p, lo, hi)).cuda(), ghost_lo=gl)
        f["damp"] = st.embed(torch.from_numpy(W.damp(p, lo, hi)).cuda(), ghost_lo=gl)
        f["trace"] = torch.zeros((p.nt, len(p.rec)), dtype=torch.float32, device="cuda")
        plans.append(st)
        fields.append(f)
    G, nzl = plans[0].G, plans[0].nz_local
    done = 0
    while done < p.nt:
        n = min(tc, p.nt - done)
        local_exchange(fields, G, nzl, p.radius, n, need_prev=True)
        for st, f in zip(plans, fields):
            first = done == 0           # later chunks reuse the plan's medium (vel = NULL)
            st.run(f["u_prev"], f["u_cur"], n, vel=f["vel"] if first else None,
                   damp=f["damp"] if first else None, step0=done,
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
