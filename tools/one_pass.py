#!/usr/bin/env python
"""Run a config's sweep `runs` times (default 2) for nt steps with a given t_kernel -- a short,
deterministic command for ncu / compute-sanitizer captures.

    python tools/one_pass.py C3 2 [nt=2] [runs=2]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import workloads as W
    from paper_1707_02347_b200 import Stencil
    cfg, tk = sys.argv[1], int(sys.argv[2])
    nt = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    runs = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    p = W.problem(cfg)
    st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=tk)
    P, C = st.empty(), st.empty()
    vel = damp = None
    if p.time_order == 2:
        vel = st.embed(torch.from_numpy(W.velocity(p)).cuda())
        damp = st.embed(torch.from_numpy(W.damp(p)).cuda())
    else:
        _, uc = W.initial_fields(p)
        C = st.embed(torch.from_numpy(uc).cuda())
    wav = torch.from_numpy(W.wavelet(p, nt)).cuda() if p.src else None
    for _ in range(runs):
        st.run(P, C, nt, vel=vel, damp=damp, src=list(p.src), wavelet=wav, rec=list(p.rec))
    st.sync()
    torch.cuda.synchronize()
    print(f"ok {cfg} t_kernel={tk} nt={nt} runs={runs}")


if __name__ == "__main__":
    main()
