"""Where the e2e time of a config goes (bench.py e2e): per-step device time of uploads alone,
read-backs alone, runs alone, uploads + read-backs together, and the pipelined loop.
    python tools/e2e_probe.py C2 [steps]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import workloads as W
from paper_1707_02347_b200.dist import SlabRunner
from paper_1707_02347_b200.planner import plan

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = W.problem(cfg)
tk = plan(p.time_order, p.radius, p.n, nranks=1, ndim=p.ndim).t_kernel
r = SlabRunner(p, t_kernel=tk, device=0)
host = r.host_inputs(p.nt, pin=True)
devs = [r.to_device(host, p.nt), r.to_device(host, p.nt)]
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
comp = r.stencil.stream
tr0 = r.run(devs[0], p.nt)
print("pinned:", {k: v.is_pinned() for k, v in host.items()}, "bytes in/out:", r.io_bytes(host))


def timed(label, fn):
    fn(2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    h2d.wait_stream(comp); d2h.wait_stream(comp)
    th = time.perf_counter()
    fn(K)
    th = time.perf_counter() - th
    comp.wait_stream(h2d); comp.wait_stream(d2h)
    e1.record(comp)
    torch.cuda.synchronize()
    print(f"{label:34s} device {e0.elapsed_time(e1) / K:8.3f} ms/step   host enqueue {1e3 * th / K:8.3f} ms/step")


def ups(k):
    with torch.cuda.stream(h2d):
        for i in range(k):
            r.upload(host, devs[i % 2])


def downs(k):
    with torch.cuda.stream(d2h):
        for i in range(k):
            r.download(devs[i % 2], tr0, slot=i % 2)


def runs(k):
    with torch.cuda.stream(comp):
        for i in range(k):
            r.run(devs[i % 2], p.nt)


def both(k):
    ups(k); downs(k)


def all3(k):
    ups(k); downs(k); runs(k)


timed("upload only (h2d stream)", ups)
timed("read-back only (d2h stream)", downs)
timed("run only", runs)
timed("upload + read-back (2 streams)", both)
timed("upload + read-back + run (no deps)", all3)
timed("pipelined (run_host_pipelined)", lambda k: r.run_host_pipelined(host, devs, p.nt, k, (h2d, d2h)))


def serial(k):
    for i in range(k):
        r.upload(host, devs[0]); t = r.run(devs[0], p.nt); r.download(devs[0], t)


with torch.cuda.stream(comp):
    timed("serial (one stream)", serial)
