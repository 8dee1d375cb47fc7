"""Host vs device time of the C1 bench step (reset + run; run_from_init direct and graph-replayed), for the launch-overhead analysis:
plain loop, with the library's per-run timing events, and with bench.py's nvidia-smi sampler."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import workloads as W
from paper_1707_02347_b200.dist import SlabRunner
from bench import ClockSampler

p = W.problem("C1")
s = torch.cuda.Stream(); torch.cuda.set_stream(s)      # the plan's stream (graph capture below)
r = SlabRunner(p, t_kernel=1, device=0)
host = r.host_inputs(p.nt, pin=False)
dev = r.to_device(host)


def loop(label, N, fn):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(N):
        fn()
    e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"{label:40s} N={N:5d} host {1e6*(t1-t0)/N:6.1f} us/step  device {1e3*e0.elapsed_time(e1)/N:6.1f} us/step")


def step():
    r.reset_state(dev)
    r.run(dev, p.nt)


for N in (5, 50, 2000):
    loop("reset+run", N, step)
loop("run only", 2000, lambda: r.run(dev, p.nt))
for N in (5, 50, 2000):
    loop("run_from_init (stencil_run_from)", N, lambda: r.run_from_init(dev, p.nt))
# the bench step: the run_from_init call captured once and replayed as a CUDA graph
for _ in range(3):
    r.run_from_init(dev, p.nt)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    r.run_from_init(dev, p.nt)
for N in (5, 50, 2000):
    loop("run_from_init, graph replay", N, g.replay)
r.set_timing(True)
for N in (5, 50):
    loop("reset+run, timing events", N, step)
    r.timing()
cs = ClockSampler(0); cs.start()
for N in (5, 50):
    loop("reset+run, timing + nvidia-smi", N, step)
    r.timing()
cs.stop()
r.set_timing(False)
