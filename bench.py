#!/usr/bin/env python
"""Benchmark of the time-tiled FD stencil sweep (BASELINE.json metric: GPts/s and achieved HBM
GB/s vs roofline, 1/2/4/8 GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--tk auto] [--tc 4]
    python bench.py --impl reference ...        # the CPU oracle arm (host cores)

One bench *step* = one full simulation of the workload through the public API: stencil_run of
the config's nt time steps over the whole grid (all SURVEY §8(a) rows: medium precompute,
star stencil, leapfrog/heat update, source injection, receiver sampling, time tiling, halo
exchange every T_c steps when N > 1).  Inputs are synthetic (workloads/), seeded, generated once
on the host; `value` is timed with inputs resident in HBM; `e2e` re-times the same step with
host pinned buffers copied in (u_prev, u_cur, vel, damp, wavelet) and results copied out
(final u_cur and the receiver traces) inside the timed region.
Fields (>= 512 MiB each) exceed the 126 MB L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

# The paper's own runs of the replica workloads (derived from P:2001-2003 and
# P:2112-2116): GPts/s over the padded (N+20)^3 array, time-tiled and Devito auto-tuned blocking,
# on a 4-core i7-6700K.  Context only (another machine, padded-point count).
PAPER_GPTS = {"P256": (0.921, 0.672), "P256L": (0.818, 0.635), "P384": (0.793, 0.575)}
METRIC = "GPts/s (grid-point updates/sec)"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured copy (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _alg_bytes_per_point_launch(p: W.Problem, tiled: bool, tk: int) -> int:
    """Algorithmic HBM bytes per interior point per sweep launch.
    wave: T=1 reads u^{n-1}, u^n, a, c and writes u^{n+1} (in place) = 20 B;
          T_k pass reads u^{n-1}, u^n, a, c, writes u^{n+T_k-1}, u^{n+T_k} = 24 B.
    heat: read u^n, write u^{n+T} = 8 B (+4 on the final pass, ignored)."""
    if p.time_order == 2:
        return 24 if tiled else 20
    return 8


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()            # wait for the first sample so the timed region is covered
            while not self.lines and time.time() - t0 < 10:
                time.sleep(0.05)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


_OVERRIDE = {}


def _problem(cfg: str, gpus: int) -> W.Problem:
    p = W.problem(cfg, gpus=gpus) if cfg == "C5" else W.problem(cfg)
    if _OVERRIDE.get("so"):
        p = W.Problem(**{**p.__dict__, "space_order": int(_OVERRIDE["so"])})
    if _OVERRIDE.get("n"):
        n = tuple(int(v) for v in _OVERRIDE["n"].split("x"))
        p = W.Problem(**{**p.__dict__, "n": n,
                         "src": tuple((n[0] // 2, n[1] // 2, n[2] // 2) for _ in p.src),
                         "rec": tuple(r for r in p.rec if r[0] < n[0] and r[1] < n[1] and r[2] < n[2])})
    return p


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_1707_02347_b200 import Stencil
    from paper_1707_02347_b200.dist import SlabRunner, init_from_env

    rank, world, local = init_from_env(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    p = _problem(args.config, world)
    from paper_1707_02347_b200.planner import plan
    pl = plan(p.time_order, p.radius, p.n, nranks=world, ndim=p.ndim)
    tk = pl.t_kernel if args.tk == "auto" else int(args.tk)
    from paper_1707_02347_b200.stencil import supported
    if not supported(p.ndim, p.time_order, p.radius, tk):
        ok = [t for t in (1, 2, 4, 8) if supported(p.ndim, p.time_order, p.radius, t)]
        raise SystemExit(f"bench.py: t_kernel={tk} is not built for {args.config} "
                         f"(ndim={p.ndim}, time_order={p.time_order}, radius={p.radius}); "
                         f"compiled depths: {ok} (DESIGN.md §6: wave time tiles are T_k <= 2)")
    if world > 1:
        tc = pl.t_comm if args.tc is None else max(tk, args.tc)
        tc = tc if tc % tk == 0 else tk * ((tc + tk - 1) // tk)
    else:
        tc = tk
    nt = p.nt if args.nt is None else args.nt
    # --graph (2-D, one rank): replay the step (stencil_run_from the stored initial fields) as a CUDA
    # graph captured on the plan's own stream.  Off by default: the step is one resident launch,
    # and direct calls let programmatic dependent launch overlap each launch with the previous
    # kernel, which replays of a one-node graph do not (C1: 14.1 vs 16.4 us per step, DESIGN §6 G4)
    use_graph = (p.ndim == 2 and world == 1 and args.graph)
    plan_stream = torch.cuda.Stream(device=local) if use_graph else torch.cuda.current_stream(local)
    if use_graph:
        torch.cuda.set_stream(plan_stream)     # every torch op, event and replay on the plan's stream
    runner = SlabRunner(p, rank=rank, world=world, t_kernel=tk, t_comm=tc, device=local,
                        fused=args.fused_halo, lib_exchange=args.lib_exchange)
    st = runner.stencil
    # ---- host inputs (pinned) for this rank's slab, then resident device copies ----------------
    host = runner.host_inputs(nt, pin=True)
    dev_in = runner.to_device(host, nt)
    fused = runner.enable_fused(dev_in) if args.fused_halo else False

    def step_resident():
        # one simulation from the stored initial fields (a device copy of them is part of the
        # step, except where the 2-D resident kernel loads them itself: stencil_run_from)
        return runner.run_from_init(dev_in, nt)

    step_direct = step_resident
    graph = None
    if use_graph:
        # warm, then capture one step on the plan's stream; if the library's launch sequence cannot
        # be captured, fall back to direct calls
        for _ in range(3):
            step_resident()
        torch.cuda.synchronize()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=plan_stream):
                step_resident()
            torch.cuda.synchronize()
            graph = g
        except Exception as ex:          # noqa: BLE001 -- report and run uncaptured
            print(f"bench.py: CUDA graph capture failed ({ex}); direct calls", file=sys.stderr)
            torch.cuda.synchronize()
    if graph is not None:
        def step_resident():            # noqa: F811 -- the captured step (stencil_run_from)
            graph.replay()

    # clock sampler first (its start waits for the first nvidia-smi sample, an idle gap that would
    # let the SM clock drop), then the warm-up steps right before the timed region
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step_resident()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step_resident()
    e1.record(stream)
    torch.cuda.synchronize()
    t_ms = e0.elapsed_time(e1)
    # the same K steps again with the library's per-run sweep events on the plan's stream (no host
    # sync): the roofline's per-launch kernel time.  A separate pass because timed events serialise
    # the stream and would inflate the step time of launch-bound runs (C1: +7 us per 18 us step).
    runner.set_timing(True)
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        step_direct()
    torch.cuda.synchronize()
    sweep_ms, sweep_launches, tiled, aux = runner.timing()   # summed over the timed runs
    runner.set_timing(False)
    if world > 1:
        dist.barrier()
    ck = clocks.stop()
    # max over ranks
    if world > 1:
        t = torch.tensor([t_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
    pts = float(p.points) * nt * args.steps          # all ranks' interior updates
    value = pts / (t_ms * 1e-3) / 1e9

    # ---- e2e: host pinned inputs in, results out, through the public API ---------------------
    # default: pipelined over two device input slots (step k+1's upload and step k-1's read-back
    # overlap step k's run, on their own streams; SlabRunner.run_host_pipelined); --e2e-serial:
    # upload, run, read back one after the other on one stream
    # auto: serial for the launch-bound 2-D runs (C1: a 14 us run; the three-stream choreography's
    # host cost per step exceeds it -- 3.8 vs 8.5 GPts/s measured), pipelined for 3-D
    e2e_serial = args.e2e == "serial" or (args.e2e == "auto" and p.ndim == 2)
    if e2e_serial:
        def e2e_steps(k):
            for _ in range(k):
                runner.upload(host, dev_in)
                tr = runner.run(dev_in, nt)
                runner.download(dev_in, tr)
    else:
        dev_slots = [dev_in, runner.to_device(host, nt)]
        io_streams = (torch.cuda.Stream(device=local), torch.cuda.Stream(device=local))

        def e2e_steps(k):
            runner.run_host_pipelined(host, dev_slots, nt, k, io_streams)
    e2e_steps(max(1, args.warmup))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    e2e_steps(args.steps)
    e3.record(stream)
    torch.cuda.synchronize()
    t_e2e = e2.elapsed_time(e3)
    if world > 1:
        t = torch.tensor([t_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
    e2e_value = pts / (t_e2e * 1e-3) / 1e9
    h2d, d2h = runner.io_bytes(host)

    # ---- roofline of the dominant kernel (the sweep): algorithmic bytes / launch duration ----
    peak, peak_src = _peaks()
    n_local = float(p.n[0] * p.n[1] * runner.nz_local)
    tiled_frac = tiled / max(1, sweep_launches)
    bpp = (tiled_frac * _alg_bytes_per_point_launch(p, True, tk)
           + (1 - tiled_frac) * _alg_bytes_per_point_launch(p, False, tk))
    per_launch_ms = sweep_ms / max(1, sweep_launches)
    achieved = bpp * n_local / (per_launch_ms * 1e-3) / 1e9
    traffic = _ncu_traffic(args.config, tk)
    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "GPts/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms / args.steps, 3),
            "higher_is_better": True, "scaling": "weak" if args.config == "C5" else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (workloads/, seeded)",
            "config": {
                "workload": f"{args.config}: {_describe(p)}",
                "grid": list(p.n), "nt_per_step": nt, "space_order": p.space_order,
                "time_order": p.time_order, "t_kernel": tk, "t_comm": tc if world > 1 else None,
                "schedule": pl.reason if args.tk == "auto" else f"t_kernel={tk} forced by --tk (planner: {pl.reason})",
                "parallelism": f"z-slabs x{world}" if world > 1 else "single GPU",
                "step_launch": ("CUDA graph replay of one captured step (stencil_run_from the stored initial fields)"
                                if graph is not None else "direct API calls"),
                "halo": (None if world == 1 else
                         "fused push: sweep stores band planes into peer ghost zones (P2P)" if fused
                         else "library-owned NCCL exchange (bands overlapped with the interior)"
                         if runner.lib_exchange
                         else "NCCL send/recv of contiguous ghost planes every T_c steps"),
                "l2": "inputs larger than L2 (fields %.0f MiB each, L2 126 MB); no flush" % (
                    runner.field_bytes / 2**20),
            },
            "e2e": {"value": round(e2e_value, 3), "unit": "GPts/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "schedule": ("serial: upload, run, read back" if e2e_serial else
                                 "pipelined: 2 device input slots; step k+1's H2D and step k-1's "
                                 "D2H overlap step k's run (own streams)")},
            "gpu_launches": int(sweep_launches + aux),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         # DRAM bytes of the committed ncu capture over THIS run's launch time:
                         # below `frac` where the kernel moves fewer bytes than the algorithmic
                         # figure (the untiled wave kernel skips the a box where a == -1)
                         "traffic_frac": (None if traffic is None or world > 1 else
                                          round(traffic / (per_launch_ms * 1e-3) / 1e9 / peak, 4)),
                         "kernel": _kernel_name(p, tk), "alg_bytes_per_point_launch": bpp,
                         "per_launch_ms": round(per_launch_ms, 4), "peak_source": peak_src},
            "clocks": ck,
        }
        if args.config in PAPER_GPTS:
            tt, blk = PAPER_GPTS[args.config]
            pad = ((p.n[0] + 8) / p.n[0]) ** 3        # padded (N+20)^3 vs updated (N+12)^3 points
            out["paper_context"] = {
                "paper_time_tiled_gpts_padded": tt, "paper_blocked_gpts_padded": blk,
                "paper_time_tiled_gpts_updated": round(tt / pad, 4),
                "ratio_vs_paper_time_tiled": round(value / (tt / pad), 1),
                "paper_hardware": "Intel i7-6700K, 4 cores, icc -O3 (P:1581-1637)",
                "note": "BASELINE.md derived throughput; different machine and point count"}
    runner.close()
    return out


def _describe(p: W.Problem) -> str:
    phys = "heat" if p.time_order == 1 else "acoustic wave (damped leapfrog)"
    return (f"{phys}, SO{p.space_order}, {p.n[0]}x{p.n[1]}x{p.n[2]} fp32, {p.nt} steps"
            + (f", {len(p.src)} Ricker source(s) {p.f_peak:g} Hz" if p.src else "")
            + (f", {len(p.rec)} receivers" if p.rec else "")
            + (f", {p.sponge}-pt sponge" if p.sponge else ""))


def _kernel_name(p: W.Problem, tk: int) -> str:
    """Name of the compiled sweep instance a pass of this problem launches (build.instances());
    2-D grids that fit a thread-block cluster's shared memory run the resident kernel (G4)."""
    if p.ndim == 2 and not os.environ.get("ST_NO_RESIDENT"):
        return f"st::resident2d_kernel<R={p.radius}, wave={int(p.time_order == 2)}> (whole run)"
    from paper_1707_02347_b200.build import instances
    names = {0: "st::sweep_kernel", 1: "st::sweep1_kernel", 2: "st::sweep2_kernel", 3: "st::sweep1s_kernel",
             4: "st::sweepx_kernel", 5: "st::sweeph_kernel"}
    for (ndim, wave, R, TK, VY, NWY, kind) in instances():
        if (ndim, wave, R, TK) == (p.ndim, int(p.time_order == 2), p.radius, tk):
            return f"{names.get(kind, f'kind{kind}')}<R={R}, T_k={TK}>"
    return "st::sweep_kernel"


def _ncu_traffic(cfg: str, tk: int):
    """dram bytes (read+write) per sweep launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        v = d.get(f"{cfg}_tk{tk}")
        return None if v is None else float(v["dram_bytes_per_launch"])
    except Exception:
        return None


def _oracle_inputs(cfg: str):
    """The oracle's own inputs for the config (untimed): embedded fields, medium, wavelet."""
    import oracle
    p = _problem(cfg, 1)
    r = p.radius
    up, uc = W.initial_fields(p)
    P0 = oracle.embed(up, p.ndim, r)
    C0 = oracle.embed(uc, p.ndim, r)
    a = c = None
    if p.time_order == 2:
        vel = oracle.embed(W.velocity(p), p.ndim, r)
        vel[vel == 0] = 1.0
        a, c = oracle.medium(vel, oracle.embed(W.damp(p), p.ndim, r), p.dt)
        del vel
    wv = W.wavelet(p) if p.src else None
    return p, P0, C0, a, c, wv


def _cpu_info():
    """CPU model, logical cores, and the oracle's OpenMP thread count (PAPER states its machine,
    P:1581-1588; so does this baseline)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    import oracle
    return {"cpu_model": model, "nproc": os.cpu_count(), "omp_threads": oracle.num_threads()}


_ONE_THREAD = r"""
import sys, time
sys.path.insert(0, sys.argv[1])
import numpy as np, oracle, workloads as W
p = W.problem("C3")
r = p.radius
P = oracle.embed(np.zeros((p.n[2], p.n[1], p.n[0]), np.float32), 3, r)
C = P.copy()
vel = oracle.embed(W.velocity(p), 3, r); vel[vel == 0] = 1.0
a, c = oracle.medium(vel, oracle.embed(W.damp(p), 3, r), p.dt)
wv = W.wavelet(p)
t0 = time.perf_counter()
oracle.run_untiled(3, p.n, p.space_order, oracle.fd_weights(p.space_order), p.dx, 2, p.dt, P, C, a, c,
                   nt=2, src=list(p.src), wavelet=wv)
dt = time.perf_counter() - t0
print(p.points * 2 / dt / 1e9, oracle.num_threads())
"""


def one_thread_rate():
    """The oracle O1 on ONE host thread: C3 (SO8 512^3), 2 time steps."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        r = subprocess.run([sys.executable, "-c", _ONE_THREAD, ROOT], capture_output=True, text=True,
                           env=env, timeout=600)
        v, th = r.stdout.strip().split()[-2:]
        return {"value": round(float(v), 4), "unit": "GPts/s", "threads": int(th),
                "sample": "C3 full grid 512^3 SO8, 2 of 500 time steps, OMP_NUM_THREADS=1"}
    except Exception as e:   # reported, not fatal: the baseline is context
        return {"value": None, "error": str(e)[:200]}


def cpu_baseline(cfg: str, seconds: float = 15.0):
    """The oracle O1 as it stands, on this host's cores, on a bounded sample of the workload:
    the full grid for as many time steps as fit in ~`seconds` (>= 1); input generation and the
    state copies untimed."""
    import oracle
    ins = _oracle_inputs(cfg)
    p = ins[0]
    one = _oracle_timed(*ins, nt=1)                # calibration step
    steps = max(1, min(p.nt, int(seconds / max(one, 1e-3))))
    dt = _oracle_timed(*ins, nt=steps)
    out = {"value": round(p.points * steps / dt / 1e9, 4), "unit": "GPts/s", "cores": oracle.num_threads(),
           "kind": "oracle",
           "sample": f"{cfg} full grid {p.n[0]}x{p.n[1]}x{p.n[2]}, {steps} of {p.nt} time steps from the "
                     f"seeded initial state (O1 loop nest only; input generation and state copies untimed)"}
    out.update(_cpu_info())
    out["one_thread"] = one_thread_rate()
    return out


def _oracle_timed(p, P0, C0, a, c, wv, nt):
    """Seconds of O1 for nt steps from the initial state; the state copies are not timed."""
    import oracle
    P, C = P0.copy(), C0.copy()
    t0 = time.perf_counter()
    oracle.run_untiled(p.ndim, p.n, p.space_order, oracle.fd_weights(p.space_order), p.dx,
                       p.time_order, p.dt, P, C, a, c, nt=nt, src=list(p.src), wavelet=wv,
                       rec=list(p.rec))
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the CPU oracle arm, timed per bench step on a bounded sample (the
    config's full grid for --ref-steps time steps; state copies outside the timed region)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle
    ins = _oracle_inputs(args.config)
    p = ins[0]
    sample_steps = args.ref_steps
    for _ in range(args.warmup):
        _oracle_timed(*ins, nt=sample_steps)
    dt = sum(_oracle_timed(*ins, nt=sample_steps) for _ in range(args.steps))
    value = p.points * sample_steps * args.steps / dt / 1e9
    sample = (f"{args.config} full grid {p.n[0]}x{p.n[1]}x{p.n[2]}, {sample_steps} of {p.nt} time steps per "
              f"bench step (bounded sample of the workload; state copies untimed)")
    cb = {"value": round(value, 4), "unit": "GPts/s", "cores": oracle.num_threads(), "kind": "oracle",
          "sample": sample}
    cb.update(_cpu_info())
    return {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GPts/s",
            "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3 / args.steps, 3), "higher_is_better": True,
            "scaling": "weak" if args.config == "C5" else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (workloads/, seeded)",
            "config": {"workload": f"{args.config}: {_describe(p)}", "grid": list(p.n),
                       "nt_per_step": sample_steps, "space_order": p.space_order},
            "cpu_baseline": cb,
            "e2e": {"value": round(value, 4), "unit": "GPts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=list(W.CONFIG_NAMES))
    ap.add_argument("--tk", default="auto")
    ap.add_argument("--tc", type=int, default=None, help="halo depth in steps for N > 1 (default: planner)")
    ap.add_argument("--nt", type=int, default=None, help="override time steps per bench step")
    ap.add_argument("--so", type=int, default=None, help="override the space order (study runs only)")
    ap.add_argument("--grid", default=None, help="override the interior grid, e.g. 512x512x512 (study runs only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-steps", type=int, default=5, help="time steps per reference bench step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e", choices=("auto", "pipelined", "serial"), default="auto",
                    help="e2e schedule: pipelined over two device input slots, or upload/run/read back "
                         "serially (auto: serial for 2-D, pipelined for 3-D)")
    ap.add_argument("--graph", action="store_true", help="2-D runs: replay a CUDA graph of the step instead of calling the API per step")
    ap.add_argument("--fused-halo", action="store_true",
                    help="N > 1, T_c = T_k = 1: halo exchange fused into the sweep over peer memory")
    ap.add_argument("--lib-exchange", action="store_true",
                    help="N > 1: the library owns the NCCL halo exchange and the time loop "
                         "(st_config.nccl_id; boundary bands overlapped with the interior at T_c = 1)")
    args = ap.parse_args()
    _OVERRIDE.update(so=args.so, n=args.grid)
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    out = run_gpu(args)
    if out is not None:
        if out["n_gpus"] == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args.config)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
