"""Test helpers: run one workloads.Problem through the CUDA library (C ABI via the Python
binding) and through the CPU oracle, on identical seeded inputs."""
from __future__ import annotations

import numpy as np

import oracle
import workloads as W


def rel_l2(got, want) -> float:
    g = np.asarray(got, dtype=np.float64)
    w = np.asarray(want, dtype=np.float64)
    den = np.sqrt((w * w).sum())
    num = np.sqrt(((g - w) ** 2).sum())
    return float(num / den) if den > 0 else float(num)


def gpu_run(p: W.Problem, nt=None, t_kernel=1, splits=None, reuse_medium=False):
    """Run p on cuda:0; `splits` = list of nt chunks (run composition; with reuse_medium the
    chunks after the first pass vel = damp = None and reuse the plan's medium).  Returns interior
    (u_prev, u_cur, trace) as numpy arrays."""
    import torch
    from paper_1707_02347_b200 import Stencil
    nt = p.nt if nt is None else nt
    st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=t_kernel)
    up, uc = W.initial_fields(p)
    P = st.embed(torch.from_numpy(up).cuda())
    C = st.embed(torch.from_numpy(uc).cuda())
    vel = damp = None
    if p.time_order == 2:
        vel = st.embed(torch.from_numpy(W.velocity(p)).cuda())
        damp = st.embed(torch.from_numpy(W.damp(p)).cuda())
    wav = torch.from_numpy(W.wavelet(p, nt)).cuda() if p.src else None
    traces = []
    done = 0
    for chunk in (splits or [nt]):
        keep = reuse_medium and done > 0
        tr = st.run(P, C, chunk, vel=None if keep else vel, damp=None if keep else damp, step0=done,
                    src=list(p.src), wavelet=wav,
                    rec=list(p.rec))
        if tr is not None:
            traces.append(tr)
        done += chunk
    st.sync()
    torch.cuda.synchronize()
    trace = torch.cat(traces).cpu().numpy() if traces else np.zeros((nt, 0), np.float32)
    out = st.interior(P).cpu().numpy(), st.interior(C).cpu().numpy(), trace
    st.close()
    return out


def oracle_run(p: W.Problem, nt=None):
    return oracle.run_problem(p, nt=nt)
