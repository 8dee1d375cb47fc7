"""One rank of tests/test_gpu_slabs.py::test_fused_halo_push_ipc_processes: a z-slab plan in its
OWN process, all ranks on cuda:0, the neighbours' field buffers and counters reached through
stencil_ipc_export / stencil_ipc_open (CUDA IPC), as SlabRunner.enable_fused does across GPUs.

The ranks take turns: rank k runs step n only after rank k-1's step n has completed (device
synchronised, then a gloo barrier), so no kernel ever waits on one that has not finished -- two
contexts time-slicing one GPU must not spin on each other (B200_PROFILING.md).  What this covers
that the one-process test cannot: the IPC handles (offsets inside torch's segments, one mapping
per allocation), pushes and counter updates landing in another process's memory, and reading
them back there.

usage: ipc_worker.py RANK WORLD PORT OUTDIR ORDER NZ"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np                      # noqa: E402
import torch                            # noqa: E402
import torch.distributed as dist        # noqa: E402

import workloads as W                   # noqa: E402


def main():
    rank, world, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    outdir, order, nz = sys.argv[4], int(sys.argv[5]), int(sys.argv[6])
    from test_gpu_slabs import _problem
    from paper_1707_02347_b200 import Stencil
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    p = _problem(order=order, nz=nz)
    wav = torch.from_numpy(W.wavelet(p)).cuda()
    st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=1, t_comm=1,
                 rank=rank, nranks=world, no_swap=True)
    z0 = st.z_range[0]
    lo = z0 - (st.G if rank > 0 else 0)
    hi = z0 + st.nz_local + (st.G if rank < world - 1 else 0)
    gl = z0 - lo
    up, uc = W.initial_fields(p, lo, hi)
    f = {"u_prev": st.embed(torch.from_numpy(up).cuda(), ghost_lo=gl),
         "u_cur": st.embed(torch.from_numpy(uc).cuda(), ghost_lo=gl),
         "vel": st.embed(torch.from_numpy(W.velocity(p, lo, hi)).cuda(), ghost_lo=gl),
         "damp": st.embed(torch.from_numpy(W.damp(p, lo, hi)).cuda(), ghost_lo=gl),
         "trace": torch.zeros((p.nt, len(p.rec)), dtype=torch.float32, device="cuda")}
    a, b = f["u_prev"], f["u_cur"]
    mine = (st.ipc_export(a.data_ptr()), st.ipc_export(b.data_ptr()), st.ipc_export(st.peer_counters()))
    blobs = [None] * world
    dist.all_gather_object(blobs, mine)
    for side, peer in ((0, rank - 1), (1, rank + 1)):
        if 0 <= peer < world:
            pa, pb, pc = (st.ipc_open(x) for x in blobs[peer])
            st.set_peer(side, a, b, pa, pb, pc)
    torch.cuda.synchronize()
    dist.barrier()
    for n in range(p.nt):
        for turn in range(world):
            if turn == rank:
                st.run(f["u_prev"], f["u_cur"], 1, vel=f["vel"] if n == 0 else None,
                       damp=f["damp"] if n == 0 else None, step0=n, src=list(p.src), wavelet=wav,
                       rec=list(p.rec), trace=f["trace"][n:n + 1])
                if st.swapped():
                    f["u_prev"], f["u_cur"] = f["u_cur"], f["u_prev"]
                torch.cuda.synchronize()
            dist.barrier()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"),
             P=st.interior(f["u_prev"]).cpu().numpy(), C=st.interior(f["u_cur"]).cpu().numpy(),
             T=f["trace"].cpu().numpy())
    dist.barrier()          # peers keep their buffers mapped until every rank has read its result
    st.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
