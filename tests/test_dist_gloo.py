"""Multi-process CPU test of the z-slab path (gloo, world sizes 2 and 3): the SAME halo_exchange
(paper_1707_02347_b200/dist.py) the GPUs use over NCCL moves the ghost planes between ranks, each
rank advances its slab T_c steps with the CPU oracle (treating the slab ends as boundaries --
the error enters at radius planes per step and never reaches the owned planes), and the
assembled owned planes and rank-summed traces must equal the single-domain oracle BITWISE."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    p = W.problem("C5", n=(23, 19, 36), nt=11, sponge=3)
    return W.Problem(**{**p.__dict__, "space_order": 4,
                        "src": ((11, 9, 12), (4, 4, 11)),     # near the 3-rank slab boundary z=12
                        "rec": ((11, 9, 12), (11, 9, 11), (3, 3, 0), (20, 15, 35), (5, 6, 24))})


def _slab_step(p, fields, rank, world, G, nzl, z0, nt, step0, wav, trace):
    """Advance the slab (incl. existing ghost planes) nt steps with the oracle."""
    r = p.radius
    has_lo, has_hi = rank > 0, rank < world - 1
    lo = G - (G if has_lo else 0)
    hi = G + nzl + (G if has_hi else 0)
    g_lo = z0 - (G if has_lo else 0)           # global plane of array plane `lo`
    nx, ny = p.n[0], p.n[1]
    sub_n = (nx, ny, hi - lo)
    P = oracle.embed(fields["u_prev"][lo:hi, :, :nx].numpy(), 3, r)
    C = oracle.embed(fields["u_cur"][lo:hi, :, :nx].numpy(), 3, r)
    vel = oracle.embed(W.velocity(p, g_lo, g_lo + hi - lo), 3, r)
    vel[vel == 0] = 1.0
    a, c = oracle.medium(vel, oracle.embed(W.damp(p, g_lo, g_lo + hi - lo), 3, r), p.dt)
    src = [(x, y, z - g_lo) for (x, y, z) in p.src if g_lo <= z < g_lo + hi - lo]
    sidx = [i for i, (x, y, z) in enumerate(p.src) if g_lo <= z < g_lo + hi - lo]
    rec = [(x, y, z - g_lo) for (x, y, z) in p.rec if z0 <= z < z0 + nzl]       # owned only
    ridx = [i for i, (x, y, z) in enumerate(p.rec) if z0 <= z < z0 + nzl]
    tr = oracle.run_untiled(3, sub_n, p.space_order, oracle.fd_weights(p.space_order), p.dx, 2, p.dt,
                            P, C, a, c, nt=nt, step0=step0, src=src,
                            wavelet=wav[:, sidx] if src else None, rec=rec)
    fields["u_prev"][lo:hi, :, :nx] = torch.from_numpy(oracle.extract(P, 3, sub_n, r))
    fields["u_cur"][lo:hi, :, :nx] = torch.from_numpy(oracle.extract(C, 3, sub_n, r))
    for k, i in enumerate(ridx):
        trace[step0:step0 + nt, i] = torch.from_numpy(tr[:, k])


def _worker(rank, world, port, tc, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1707_02347_b200.dist import halo_exchange
        p = _problem()
        r = p.radius
        nzl = p.n[2] // world
        G = r * tc
        z0 = rank * nzl
        X = (p.n[0] + 31) // 32 * 32
        Z = nzl + 2 * G
        fields = {k: torch.zeros((Z, p.n[1], X), dtype=torch.float32) for k in ("u_prev", "u_cur")}
        wav = W.wavelet(p)
        trace = torch.zeros((p.nt, len(p.rec)), dtype=torch.float32)
        done = 0
        while done < p.nt:
            n = min(tc, p.nt - done)
            halo_exchange(fields, rank, world, G, nzl, r, n, need_prev=True)
            _slab_step(p, fields, rank, world, G, nzl, z0, n, done, wav, trace)
            done += n
        dist.all_reduce(trace)
        own = fields["u_cur"][G:G + nzl, :, :p.n[0]].contiguous()
        ownp = fields["u_prev"][G:G + nzl, :, :p.n[0]].contiguous()
        gath = [torch.zeros_like(own) for _ in range(world)]
        gathp = [torch.zeros_like(own) for _ in range(world)]
        dist.all_gather(gath, own)
        dist.all_gather(gathp, ownp)
        if rank == 0:
            q.put((torch.cat(gathp).numpy(), torch.cat(gath).numpy(), trace.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,tc", [(2, 1), (2, 3), (3, 2), (3, 4)])
def test_slab_decomposition_gloo_bitwise(world, tc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tc, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p = _problem()
    want = oracle.run_problem(p)
    assert np.abs(want[1]).max() > 0
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_exchange_plan_depths():
    from paper_1707_02347_b200.dist import exchange_plan
    ops = exchange_plan(rank=1, world=3, G=12, nzl=20, radius=4, nt=3)
    # u_cur: depth 12, u_prev: depth 8, both neighbours, send/recv pairs
    assert ("send", 0, "u_cur", 12, 12) in ops and ("recv", 0, "u_cur", 0, 12) in ops
    assert ("send", 2, "u_cur", 20, 12) in ops and ("recv", 2, "u_cur", 32, 12) in ops
    assert ("send", 0, "u_prev", 12, 8) in ops and ("recv", 2, "u_prev", 32, 8) in ops
    assert len(ops) == 8
    assert exchange_plan(rank=0, world=1, G=4, nzl=8, radius=4, nt=1) == []
    ops0 = exchange_plan(rank=0, world=2, G=4, nzl=8, radius=4, nt=1)
    assert ops0 == [("send", 1, "u_cur", 8, 4), ("recv", 1, "u_cur", 12, 4)]
