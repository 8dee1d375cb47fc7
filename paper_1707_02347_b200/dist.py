"""z-slab decomposition over GPUs.

One process per GPU.  The global grid is split into z-slabs of n_z/G interior planes; each rank
stores G = radius*T_c ghost planes on both sides (layout: include/stencil.h).  Once per period of
T_c steps the ranks exchange ghost planes with their z-neighbours -- depth radius*T_c of u^n and
radius*(T_c-1) of u^{n-1} -- as contiguous plane slabs (z is the slowest axis, so no packing) with
torch.distributed point-to-point send/recv (NCCL over NVLink on GPUs, gloo on CPU for tests), then
the CUDA library advances T_c steps over the shrinking valid region without further exchange.
Receiver traces are written by the owning rank only and summed across ranks at the end.

`halo_exchange` is device-agnostic (CPU or CUDA tensors) so the exchange plan is tested on CPU
with gloo (tests/test_dist_gloo.py) exactly as it runs on the GPUs.
"""
from __future__ import annotations

import os
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch
import torch.distributed as dist


def init_from_env(gpus: int = 1, backend: str = "nccl") -> Tuple[int, int, int]:
    """(rank, world, local_rank) from torchrun's environment; initialises the process group when
    world > 1 (rendezvous defaults to 127.0.0.1)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if gpus not in (None, 0) and world != gpus and world > 1:
        raise RuntimeError(f"--gpus {gpus} but WORLD_SIZE={world}")
    return rank, world, local


def exchange_plan(rank: int, world: int, G: int, nzl: int, radius: int, nt: int,
                  depth_prev: Optional[int] = None) -> List[Tuple[str, int, str, int, int]]:
    """Messages for one exchange before `nt` steps: (op, peer, field, plane_begin, plane_count) in
    array-plane coordinates.  u_cur needs radius*nt ghost planes, u_prev radius*(nt-1)."""
    dc = radius * nt
    dp = radius * (nt - 1) if depth_prev is None else depth_prev
    assert dc <= G, "ghost zone too shallow for nt steps"
    ops = []
    for field, d in (("u_cur", dc), ("u_prev", dp)):
        if d <= 0:
            continue
        if rank > 0:          # lower neighbour: send my lowest owned planes, receive its highest
            ops.append(("send", rank - 1, field, G, d))
            ops.append(("recv", rank - 1, field, G - d, d))
        if rank < world - 1:  # upper neighbour
            ops.append(("send", rank + 1, field, G + nzl - d, d))
            ops.append(("recv", rank + 1, field, G + nzl, d))
    return ops


def halo_exchange(fields: Dict[str, torch.Tensor], rank: int, world: int, G: int, nzl: int,
                  radius: int, nt: int, need_prev: bool = True, group=None) -> int:
    """Exchange ghost planes of fields['u_cur'] (and fields['u_prev'] when need_prev) in place.
    Returns the bytes this rank sent."""
    if world <= 1:
        return 0
    plan = exchange_plan(rank, world, G, nzl, radius, nt, None if need_prev else 0)
    p2p = []
    sent = 0
    for op, peer, field, z0, cnt in plan:
        view = fields[field][z0:z0 + cnt]
        assert view.is_contiguous()
        if op == "send":
            p2p.append(dist.P2POp(dist.isend, view, peer, group))
            sent += view.numel() * view.element_size()
        else:
            p2p.append(dist.P2POp(dist.irecv, view, peer, group))
    if p2p:
        for r in dist.batch_isend_irecv(p2p):
            r.wait()
    return sent


def local_exchange(fields_per_rank: List[Dict[str, torch.Tensor]], G: int, nzl: int, radius: int,
                   nt: int, need_prev: bool = True) -> None:
    """The same exchange plan executed by plain tensor copies between slabs held by ONE process
    (all slabs on one device, or peer copies between devices).  Owned planes are read and ghost
    planes written, so the copy order is irrelevant."""
    world = len(fields_per_rank)
    for i in range(world):
        for op, peer, field, zr, cnt in exchange_plan(i, world, G, nzl, radius, nt,
                                                      None if need_prev else 0):
            if op != "recv":
                continue
            for op2, peer2, field2, zs, cnt2 in exchange_plan(peer, world, G, nzl, radius, nt,
                                                              None if need_prev else 0):
                if op2 == "send" and peer2 == i and field2 == field:
                    assert cnt2 == cnt
                    fields_per_rank[i][field][zr:zr + cnt].copy_(fields_per_rank[peer][field][zs:zs + cnt])


class SlabRunner:
    """Runs a workloads.Problem on this rank's z-slab through the CUDA library, exchanging ghost
    planes every T_c steps.  world == 1 degenerates to a single stencil_run per simulation."""

    def __init__(self, problem, rank: int = 0, world: int = 1, t_kernel: int = 1, t_comm: int = 1,
                 device: int = 0, fused: bool = False, lib_exchange: bool = False):
        from .stencil import Stencil, nccl_unique_id
        self.p = problem
        self.rank, self.world = rank, world
        self.tk = t_kernel
        self.tc = t_comm if world > 1 else max(1, t_kernel)
        self.device = device
        # lib_exchange: the library owns the NCCL communicator and the whole time loop
        # (st_config.nccl_id); rank 0 makes the id, the process group broadcasts it
        nccl_id = None
        self.lib_exchange = lib_exchange and world > 1
        if self.lib_exchange:
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
        self.stencil = Stencil(problem.ndim, problem.n, problem.space_order, problem.time_order,
                               problem.dt, problem.dx, t_kernel=t_kernel, t_comm=self.tc, rank=rank,
                               nranks=world, device=device, no_swap=True, nccl_id=nccl_id)
        st = self.stencil
        self.G = st.G
        self.nzl = st.nz_local
        self.z0 = st.z_range[0]
        self.has_lo, self.has_hi = rank > 0, rank < world - 1
        self.field_bytes = st.X * st.Y * st.Z * 4
        self.wave = problem.time_order == 2
        self._timing = False
        # fused halo push (include/stencil.h): T_c = T_k = 1 only; enabled by enable_fused()
        self.fused_capable = fused and world > 1 and t_kernel == 1 and self.tc == 1
        self.fused = False

    @property
    def nz_local(self):
        return self.nzl

    # ------------------------------------------------------------------ inputs
    def _slab_planes(self):
        """Global interior plane range stored by this rank (owned + existing ghost planes)."""
        lo = self.z0 - (self.G if self.has_lo else 0)
        hi = self.z0 + self.nzl + (self.G if self.has_hi else 0)
        return lo, hi

    def host_inputs(self, nt: int, pin: bool = True) -> Dict[str, torch.Tensor]:
        """Seeded inputs of this slab in the padded layout, on the host (pinned)."""
        import workloads as W
        p, st = self.p, self.stencil
        lo, hi = self._slab_planes() if p.ndim == 3 else (0, 1)
        ghost_lo = self.z0 - lo if p.ndim == 3 else 0
        out = {}

        def put(arr):
            t = torch.zeros(st.shape, dtype=torch.float32, pin_memory=pin)
            z = st.G - ghost_lo
            t[z:z + arr.shape[0], :, :p.n[0]] = torch.from_numpy(arr)
            return t
        up, uc = W.initial_fields(p, lo, hi)
        out["u_prev"], out["u_cur"] = put(up), put(uc)
        if self.wave:
            out["vel"] = put(W.velocity(p, lo, hi))
            out["damp"] = put(W.damp(p, lo, hi))
        if p.src:
            w = torch.from_numpy(W.wavelet(p, nt))
            out["wavelet"] = w.pin_memory() if pin else w
        return out

    def to_device(self, host: Dict[str, torch.Tensor], nt: int = None) -> Dict[str, torch.Tensor]:
        """Device copies of host_inputs(nt); the receiver trace is sized for nt steps (default: the
        wavelet's row count, else the problem's nt), so run(dev, nt) never writes past it."""
        dev = {k: v.to(f"cuda:{self.device}", non_blocking=True) for k, v in host.items()}
        dev["_init_cur"] = dev["u_cur"].clone()
        dev["_init_prev"] = dev["u_prev"].clone()
        if nt is None:
            nt = host["wavelet"].shape[0] if "wavelet" in host else self.p.nt
        if self.p.rec:
            dev["trace"] = torch.zeros((max(1, nt), len(self.p.rec)), dtype=torch.float32,
                                       device=f"cuda:{self.device}")
        return dev

    def enable_fused(self, dev, group=None):
        """Fused halo push: every rank exports (IPC) its two field buffers and its inbound
        counters, all-gathers the blobs over the process group and registers its z-neighbours'
        with the library; from then on a run's sweep stores its band planes straight into the
        neighbours' ghost zones and only the first chunk of each simulation calls NCCL."""
        if not self.fused_capable:
            return False
        st = self.stencil
        a, b = dev["u_prev"], dev["u_cur"]
        mine = (st.ipc_export(a.data_ptr()), st.ipc_export(b.data_ptr()),
                st.ipc_export(st.peer_counters()))
        blobs = [None] * self.world
        dist.all_gather_object(blobs, mine, group=group)
        for side, peer in ((0, self.rank - 1), (1, self.rank + 1)):
            if 0 <= peer < self.world:
                pa, pb, pc = (st.ipc_open(x) for x in blobs[peer])
                st.set_peer(side, a, b, pa, pb, pc)
        dist.barrier(group=group)
        self.fused = True
        return True

    def reset_state(self, dev):
        dev["u_cur"].copy_(dev["_init_cur"])
        if self.wave:           # heat reads only u^n: its u_prev is output-only (include/stencil.h)
            dev["u_prev"].copy_(dev["_init_prev"])

    def run_from_init(self, dev, nt: int):
        """One simulation from the stored initial pair (the bench step): on one rank
        stencil_run_from (the 2-D resident kernel loads the pair itself: one launch, no copy; other
        plans copy it on the plan's stream), else reset_state + run."""
        if self.world > 1 or self.fused or self.lib_exchange:
            self.reset_state(dev)
            return self.run(dev, nt)
        p, st = self.p, self.stencil
        trace = dev.get("trace")
        if trace is not None:
            trace = trace[:nt]          # one rank owns every receiver: every entry is written
        st.run(dev["u_prev"], dev["u_cur"], nt, vel=dev.get("vel"), damp=dev.get("damp"), step0=0,
               src=list(p.src), wavelet=dev.get("wavelet"), rec=list(p.rec), trace=trace,
               init=(dev["_init_prev"] if self.wave else None, dev["_init_cur"]))
        if st.swapped():
            dev["u_prev"], dev["u_cur"] = dev["u_cur"], dev["u_prev"]
        return trace

    def _inputs(self):
        # heat reads only u^n (its u_prev is output-only, include/stencil.h): u_prev is not an input
        return ("u_prev", "u_cur", "vel", "damp", "wavelet") if self.wave else ("u_cur", "wavelet")

    def upload(self, host, dev):
        for k in self._inputs():
            if k in host:
                dev[k].copy_(host[k], non_blocking=True)

    def download(self, dev, trace, slot: int = 0):
        """Asynchronous copy of u^{n+nt} (owned interior) and the trace into pinned host buffers
        (one pair per slot, so pipelined steps never share a destination); returns them."""
        st = self.stencil
        if not hasattr(self, "_out_bufs"):
            self._out_bufs = {}
        if slot not in self._out_bufs:
            self._out_bufs[slot] = (
                torch.empty(st.interior(dev["u_cur"]).shape, dtype=torch.float32, pin_memory=True),
                torch.empty(trace.shape, dtype=torch.float32, pin_memory=True) if trace is not None else None)
        out_h, tr_h = self._out_bufs[slot]
        out_h.copy_(st.interior(dev["u_cur"]), non_blocking=True)
        if trace is not None:
            tr_h.copy_(trace, non_blocking=True)
        return out_h, tr_h

    def run_host_pipelined(self, host, devs, nt: int, steps: int, streams):
        """steps simulations, each from the pinned host inputs to pinned host results, pipelined
        over the device input slots devs (to_device copies): step k uploads into slot k % len(devs)
        on streams[0] while step k-1 runs on the plan's stream, and downloads on streams[1] while
        step k+1 runs.  A slot is re-uploaded only after its previous results were read back.
        Every step still copies all of its inputs in and its result out (bench.py e2e)."""
        import torch
        comp = self.stencil.stream
        h2d, d2h = streams
        free = [None] * len(devs)
        res = None
        h2d.wait_stream(comp)           # the first upload starts after the work already queued
        for k in range(steps):
            i = k % len(devs)
            d = devs[i]
            with torch.cuda.stream(h2d):
                if free[i] is not None:
                    h2d.wait_event(free[i])
                self.upload(host, d)
                up = torch.cuda.Event()
                up.record(h2d)
            with torch.cuda.stream(comp):
                comp.wait_event(up)
                tr = self.run(d, nt)
                done = torch.cuda.Event()
                done.record(comp)
            with torch.cuda.stream(d2h):
                d2h.wait_event(done)
                res = self.download(d, tr, slot=i)
                free[i] = torch.cuda.Event()
                free[i].record(d2h)
        comp.wait_stream(d2h)
        return res

    def io_bytes(self, host) -> Tuple[int, int]:
        h2d = sum(host[k].numel() * 4 for k in self._inputs() if k in host)
        n_out = self.p.n[0] * self.p.n[1] * (self.nzl if self.p.ndim == 3 else 1)
        d2h = 4 * (n_out + (self.p.nt * len(self.p.rec) if self.p.rec else 0))
        return h2d, d2h

    # ------------------------------------------------------------------ run
    def set_timing(self, on: bool = True):
        self._timing = on
        self.stencil.set_timing(on)

    def timing(self):
        """(sweep_ms, sweep_launches, tiled_launches, aux_launches) summed over every run since the
        previous query or set_timing (waits for the last run; the runs themselves never sync)."""
        return self.stencil.timing()

    def run(self, dev, nt: int):
        """Advance the slab by nt steps (exchange every T_c steps when world > 1); returns the
        (rank-summed) receiver trace tensor or None."""
        p, st = self.p, self.stencil
        trace = dev.get("trace")
        if trace is not None:
            trace = trace[:nt]
            trace.zero_()
        if self.lib_exchange:
            # one C-ABI call: the library exchanges every T_c steps (overlapped at T_c = 1) and
            # sums the trace over the ranks itself
            st.run(dev["u_prev"], dev["u_cur"], nt, vel=dev.get("vel"), damp=dev.get("damp"),
                   step0=0, src=list(p.src), wavelet=dev.get("wavelet"), rec=list(p.rec), trace=trace)
            if st.swapped():
                dev["u_prev"], dev["u_cur"] = dev["u_cur"], dev["u_prev"]
            return trace
        done = 0
        while done < nt:
            n = min(self.tc, nt - done) if self.world > 1 else nt - done
            # fused: the sweeps push the ghost planes themselves; NCCL only before the first step
            # (it also orders this simulation's reset after the neighbours' last pushes)
            if self.world > 1 and (not self.fused or done == 0):
                halo_exchange(dev, self.rank, self.world, self.G, self.nzl, p.radius, n,
                              need_prev=self.wave)
            # the medium a, c is derived once per simulation (first chunk); later chunks reuse it
            first = done == 0
            st.run(dev["u_prev"], dev["u_cur"], n, vel=dev.get("vel") if first else None,
                   damp=dev.get("damp") if first else None,
                   step0=done, src=list(p.src), wavelet=dev.get("wavelet"), rec=list(p.rec),
                   trace=None if trace is None else trace[done:done + n])
            if st.swapped():      # odd pass count (T_c = 1): swap references, not 2 fields of HBM
                dev["u_prev"], dev["u_cur"] = dev["u_cur"], dev["u_prev"]
            done += n
        if trace is not None and self.world > 1:
            dist.all_reduce(trace)
        return trace

    def close(self):
        self.stencil.close()
