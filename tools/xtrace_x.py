#!/usr/bin/env python
"""Event-trace diagnosis of the two-role exchange pass (sweepx.cuh built with -DST_XTRACE).

    ST_LIB=paper_1707_02347_b200/_varlib/libstencil_xtx.so python tools/xtrace_x.py C3 [nt]
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pct(name, a):
    a = np.asarray(a, dtype=np.float64)
    a = a[np.isfinite(a)]
    if a.size:
        print(f"{name:44s} n {a.size:7d} p10 {np.percentile(a,10):8.2f} p50 {np.percentile(a,50):8.2f} "
              f"p90 {np.percentile(a,90):8.2f} p99 {np.percentile(a,99):8.2f} us")


def main():
    import torch
    import workloads as W
    from paper_1707_02347_b200 import Stencil, _lib
    cfg = sys.argv[1]
    nt = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    p = W.problem(cfg)
    st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=2)
    P, C = st.empty(), st.empty()
    vel = st.embed(torch.from_numpy(W.velocity(p)).cuda())
    damp = st.embed(torch.from_numpy(W.damp(p)).cuda())
    wav = torch.from_numpy(W.wavelet(p, nt)).cuda()
    for _ in range(2):
        st.run(P, C, nt, vel=vel, damp=damp, src=list(p.src), wavelet=wav)
    st.sync()
    f = _lib.load().stencil_xtrace
    f.restype = ctypes.c_int64
    K, NT = 1024, 8192
    buf = np.zeros(NT * K * 12, dtype=np.uint64)
    NI = 18   # ints per XTile
    tiles = np.zeros(NT * NI, dtype=np.int32)
    n = f(st._h, buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(buf.nbytes),
          tiles.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(tiles.nbytes))
    tr = buf[: n * K * 12].reshape(n, K, 12).astype(np.int64)
    td = tiles[: n * NI].reshape(n, NI)
    role, zb, ze, nd = td[:, 2], td[:, 3], td[:, 4], td[:, 7]
    t0 = tr[:, 0, 6][tr[:, 0, 6] > 0].min()
    print(f"tiles {n}: L1 {int((role == 0).sum())} L2 {int((role == 1).sum())}")
    # publication: saw -> release returned
    pub = []
    for i in range(n):
        k = ze[i] - zb[i]
        e = tr[i, :k]
        ok = (e[:, 0] > 0) & (e[:, 1] > 0)
        pub.append((e[ok, 1] - e[ok, 0]) / 1e3)
    pct("publisher: saw stored -> release returned", np.concatenate(pub))
    # L2 wait: for arrival a (plane zb - r + a) wait start -> satisfied; and vs deps' release time
    r = p.space_order // 2
    waits, vis, lag = [], [], []
    for i in np.where(role == 1)[0]:
        deps = td[i, 8:8 + nd[i]]
        for a in range(ze[i] - zb[i] + 2 * r):
            ts, te = tr[i, a, 2], tr[i, a, 3]
            if ts > 0 and te > 0:
                waits.append((te - ts) / 1e3)
                pl = zb[i] - r + a
                rel = [tr[d, pl - zb[d], 1] for d in deps if 0 <= pl - zb[d] < K]
                rel = [x for x in rel if x > 0]
                if rel:
                    vis.append((te - max(rel)) / 1e3)
    pct("L2 producer wait (start -> satisfied)", waits)
    pct("L2 satisfied - last dep release returned", vis)
    thr = []
    for i in np.where(role == 0)[0]:
        e = tr[i]
        ok = (e[:, 4] > 0) & (e[:, 5] > 0)
        thr.append((e[ok, 5] - e[ok, 4]) / 1e3)
    if thr:
        pct("L1 throttle waits", np.concatenate(thr))
    # lag: L2 tile vs its partner L1 (by index) release time of the same plane
    lags = []
    for i in np.where(role == 0)[0]:
        j = td[i, 17]
        if j < 0:
            continue
        for k in range(0, ze[j] - zb[j], 8):
            pl = zb[j] + k
            a = tr[i, pl - zb[i], 1]
            b = tr[j, k, 1]
            if a > 0 and b > 0:
                lags.append((b - a) / 1e3)
    pct("L2 release(p) - partner L1 release(p)", lags)
    starts = (tr[:, 0, 6] - t0) / 1e3
    print("tile start spread (us): L1", np.percentile(starts[role == 0], [0, 50, 100]).round(1),
          "L2", np.percentile(starts[role == 1], [0, 50, 100]).round(1))


if __name__ == "__main__":
    main()
