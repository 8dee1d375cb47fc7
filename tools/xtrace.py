#!/usr/bin/env python
"""Event-trace diagnosis of the exchange-tiled kernel (sweept.cuh built with -DST_XTRACE).

    python tools/xtrace.py build                      # here: builds _varlib/libstencil_xtrace.so
    ST_LIB=paper_1707_02347_b200/_varlib/libstencil_xtrace.so python tools/xtrace.py run C3 [nt]

Per (tile, plane k) the kernel stamps %globaltimer at: 0 producer-X saw l1done(k), 1 neighbours'
progress satisfied, 2 box TMA issued (after the free-slot wait), 3 consumer warp 0 got box(k),
4 warp 0 finished level 2 of k, 5 warp 0 stored level 1 of k, 6 tile start, 7 warp 0 starts
waiting for box(k).  Prints latency percentiles of each stage.
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    if sys.argv[1] == "build":
        from paper_1707_02347_b200.build import build_variant
        print(build_variant("xtrace", defines=["-DST_XTRACE"], verbose=False))
        return
    import torch
    import workloads as W
    from paper_1707_02347_b200 import Stencil, _lib
    cfg = sys.argv[2]
    nt = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    p = W.problem(cfg)
    st = Stencil(p.ndim, p.n, p.space_order, p.time_order, p.dt, p.dx, t_kernel=2)
    P, C = st.empty(), st.empty()
    vel = st.embed(torch.from_numpy(W.velocity(p)).cuda())
    damp = st.embed(torch.from_numpy(W.damp(p)).cuda())
    wav = torch.from_numpy(W.wavelet(p, nt)).cuda()
    for _ in range(2):
        st.run(P, C, nt, vel=vel, damp=damp, src=list(p.src), wavelet=wav)
    st.sync()
    lib = _lib.load()
    f = lib.stencil_xtrace
    f.restype = ctypes.c_int64
    K = 1024
    nbytes = 4096 * K * 12 * 8
    buf = np.zeros(nbytes // 8, dtype=np.uint64)
    tiles = np.zeros(4096 * 12, dtype=np.int32)
    n = f(st._h, buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(nbytes),
          tiles.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(tiles.nbytes))
    tr = buf[: n * K * 12].reshape(n, K, 12).astype(np.int64)
    td = tiles[: n * 12].reshape(n, 12)
    nk = td[:, 7] - td[:, 6]
    print(f"tiles {n}, planes per tile {sorted(set(nk.tolist()))}")
    t0 = tr[:, 0, 6][tr[:, 0, 6] > 0].min()
    starts = (tr[:, 0, 6] - t0) / 1e3
    ends = np.array([(tr[i, nk[i] - 1, 4] - t0) / 1e3 for i in range(n)])
    print(f"pass span {ends.max():.1f} us; tile duration median {np.median(ends - starts):.1f} us"
          f" min {np.min(ends - starts):.1f} max {np.max(ends - starts):.1f}")

    def pct(name, a):
        a = a[np.isfinite(a)]
        if a.size:
            print(f"{name:42s} p10 {np.percentile(a,10):8.2f} p50 {np.percentile(a,50):8.2f} "
                  f"p90 {np.percentile(a,90):8.2f} p99 {np.percentile(a,99):8.2f} us")
    L = []
    for i in range(n):
        k = nk[i]
        e = tr[i, :k].astype(np.float64)
        L.append(e)
    E = np.concatenate(L)
    ok = (E[:, :6] > 0).all(axis=1)
    E = E[ok]
    pct("l1 stored(w0) -> X saw l1done", (E[:, 0] - E[:, 5]) / 1e3)
    pct("X saw l1done -> deps satisfied", (E[:, 1] - E[:, 0]) / 1e3)
    pct("deps -> TMA issued (slot wait)", (E[:, 2] - E[:, 1]) / 1e3)
    pct("TMA issued -> w0 has box", (E[:, 3] - E[:, 2]) / 1e3)
    pct("w0 waits for box (start->got)", (E[:, 3] - E[:, 7]) / 1e3)
    pct("w0 level-2 compute (got box->done)", (E[:, 4] - E[:, 3]) / 1e3)
    d = np.diff(E[:, 4])
    pct("w0 plane period (level-2 done->done)", d[(d > 0) & (d < 1e7)] / 1e3)
    pct("l1 stored(k) -> l2 done(k)", (E[:, 4] - E[:, 5]) / 1e3)
    pct("l1done seen -> published (release issued)", (E[:, 8] - E[:, 0]) / 1e3)
    # visibility latency: my deps satisfied(k) - max over deps of their publish(k)
    lat, lead = [], []
    for i in range(n):
        deps = [d for d in td[i, 8:12] if d >= 0]
        if not deps:
            continue
        for k in range(nk[i]):
            pub = max(tr[d, k, 8] for d in deps)
            if pub > 0 and tr[i, k, 1] > 0:
                lat.append((tr[i, k, 1] - pub) / 1e3)
                lead.append((pub - tr[i, k, 8]) / 1e3)
    pct("deps satisfied - last dep published", np.array(lat))
    pct("last dep published - my publish", np.array(lead))


if __name__ == "__main__":
    main()
