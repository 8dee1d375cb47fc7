"""CPU ORACLE for the time-stepped FD stencil sweep -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  The CUDA product path
(paper_1707_02347_b200/) never imports it and shares no code with it; both
take their inputs from workloads/ only.

Contents
  fd_weights(order)        standard central 2nd-derivative weights, closed form
                           (the paper's SO8 constants at
                           P:1682-1707 are 0.046208 x these).
  medium(vel, damp, dt)    a, c of the damped leapfrog, oracle.cpp.
  run_untiled(...)         O1, the plain untiled loop nest.
  run_literal(...)         O1-literal: the paper's printed wave expression and term order
                           (P:1678-1708), to bound fp32 order drift (reading Q8).
  run_slabs(...)           O3: the GPU's z-slab schedule (ghost depth r*T_c, exchange every T_c
                           steps, shrinking redundant regions), plain loops; bitwise O1.
  run_skewed(...)          O2, the paper's skewed time-tiled schedule.
  embed/extract            oracle layout <-> interior arrays.

Parity status: every function here is pinned by a `-m "not gpu"` test in
tests/test_oracle_pins.py / tests/test_oracle_schedules.py, except receiver
traces with non-symmetric geometry (pinned only by symmetry; see DESIGN.md
"parity unpinned" list).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction
from math import factorial
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so (g++, OpenMP, no FP contraction, FMA instructions)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-fopenmp", "-ffp-contract=off", "-mfma", "-fPIC", "-shared",
               "-o", _SO, _SRC]
        subprocess.check_call(cmd)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        L = ctypes.c_long
        I = ctypes.c_int
        D = ctypes.c_double
        common = [I, L, L, L, I, P, P, I, D, P, P, P, P, I, L, I, P, P, I, P, P, I]
        for nm in ("oracle_run_untiled_f32", "oracle_run_untiled_f64"):
            f = getattr(lib, nm)
            f.argtypes = common
            f.restype = I
        for nm in ("oracle_run_skewed_f32", "oracle_run_skewed_f64"):
            f = getattr(lib, nm)
            f.argtypes = common + [I, I, I, I, I]
            f.restype = I
        lib.oracle_run_slabs_f32.argtypes = common + [I, I, I]
        lib.oracle_run_slabs_f32.restype = I
        for nm in ("oracle_run_literal_f32", "oracle_run_literal_f64"):
            f = getattr(lib, nm)
            f.argtypes = [I, L, L, L, I, P, P, D, P, P, P, P, I, L, I, P, P, I, P, P, I]
            f.restype = I
        for nm in ("oracle_medium_f32", "oracle_medium_f64"):
            f = getattr(lib, nm)
            f.argtypes = [L, P, P, D, P, P, I]
            f.restype = None
        lib.oracle_num_threads.restype = I
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


# ----------------------------------------------------------------------------- FD weights
def fd_weights_exact(order: int):
    """Central 2nd-derivative weights c_0..c_m (m = order/2) as exact Fractions.

    Closed form (Taylor expansion of sum_k c_k (u(x+kh)+u(x-kh))):
        c_k = 2 (-1)^(k+1) (m!)^2 / (k^2 (m-k)! (m+k)!),  k = 1..m
        c_0 = -2 sum_{k>=1} c_k
    """
    if order < 2 or order % 2:
        raise ValueError("space order must be even and >= 2")
    m = order // 2
    c = [Fraction(0)] * (m + 1)
    for k in range(1, m + 1):
        c[k] = Fraction(2 * (-1) ** (k + 1) * factorial(m) ** 2,
                        k * k * factorial(m - k) * factorial(m + k))
    c[0] = -2 * sum(c[1:])
    return c


def fd_weights(order: int) -> np.ndarray:
    return np.array([float(x) for x in fd_weights_exact(order)], dtype=np.float64)


# ----------------------------------------------------------------------------- layout
def halo_shape(ndim: int, n, r: int):
    nx, ny, nz = n
    return ((nz + 2 * r) if ndim == 3 else 1, ny + 2 * r, nx + 2 * r)


def embed(interior: np.ndarray, ndim: int, r: int, dtype=np.float32) -> np.ndarray:
    """Interior (nz, ny, nx) -> oracle layout with a zero halo of r."""
    nz, ny, nx = interior.shape
    out = np.zeros(halo_shape(ndim, (nx, ny, nz), r), dtype=dtype)
    if ndim == 3:
        out[r:r + nz, r:r + ny, r:r + nx] = interior
    else:
        out[0, r:r + ny, r:r + nx] = interior[0]
    return out


def extract(arr: np.ndarray, ndim: int, n, r: int) -> np.ndarray:
    nx, ny, nz = n
    if ndim == 3:
        return arr[r:r + nz, r:r + ny, r:r + nx].copy()
    return arr[:, r:r + ny, r:r + nx].copy()


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _pts(pts: Sequence) -> np.ndarray:
    a = np.zeros((max(len(pts), 1), 3), dtype=np.int64)
    for i, p in enumerate(pts):
        a[i] = p
    return a


# ----------------------------------------------------------------------------- medium
def medium(vel: np.ndarray, damp: Optional[np.ndarray], dt: float, dtype=np.float32, ftz: bool = True):
    """(a, c) per point (P:1678-1708 rewritten; see oracle.cpp header)."""
    vel = np.ascontiguousarray(vel, dtype=dtype)
    eta = None if damp is None else np.ascontiguousarray(damp, dtype=dtype)
    a = np.empty_like(vel)
    c = np.empty_like(vel)
    fn = _load().oracle_medium_f32 if dtype == np.float32 else _load().oracle_medium_f64
    fn(vel.size, _ptr(vel), _ptr(eta), float(dt), _ptr(a), _ptr(c), int(ftz))
    return a, c


# ----------------------------------------------------------------------------- runs
def _run(kind: str, ndim, n, order, coeffs, h, time_order, dt, P, C, a, c, nt, step0,
         src, wavelet, rec, ftz, extra=()):
    dtype = P.dtype
    assert C.dtype == dtype and P.flags.c_contiguous and C.flags.c_contiguous
    r = order // 2
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    assert coeffs.shape == (r + 1,)
    h = np.ascontiguousarray(h, dtype=np.float64)
    src = list(src or [])
    rec = list(rec or [])
    src_a, rec_a = _pts(src), _pts(rec)
    if src:
        wavelet = np.ascontiguousarray(wavelet, dtype=dtype)
        assert wavelet.shape[1] == len(src) and wavelet.shape[0] >= step0 + nt
    trace = np.zeros((nt, max(len(rec), 1)), dtype=dtype)
    if time_order == 2:
        a = np.ascontiguousarray(a, dtype=dtype)
        c = np.ascontiguousarray(c, dtype=dtype)
    suffix = "f32" if dtype == np.float32 else "f64"
    fn = getattr(_load(), f"oracle_run_{kind}_{suffix}")
    rc = fn(ndim, n[0], n[1], n[2], r, _ptr(coeffs), _ptr(h), time_order, float(dt),
            _ptr(P), _ptr(C), _ptr(a) if time_order == 2 else None,
            _ptr(c) if time_order == 2 else None, nt, step0, len(src), _ptr(src_a),
            _ptr(wavelet) if src else None, len(rec), _ptr(rec_a), _ptr(trace), int(ftz), *extra)
    if rc != 0:
        raise ValueError(f"oracle_run_{kind} rejected its arguments (rc={rc})")
    return trace[:, :len(rec)]


def run_untiled(ndim, n, order, coeffs, h, time_order, dt, P, C, a=None, c=None, nt=1, step0=0,
                src=(), wavelet=None, rec=(), ftz=True):
    """O1: advance (P, C) = (u^{n-1}, u^n) in place by nt steps; returns trace [nt, nrec]."""
    return _run("untiled", ndim, n, order, coeffs, h, time_order, dt, P, C, a, c, nt, step0,
                src, wavelet, rec, ftz)


def run_skewed(ndim, n, order, coeffs, h, time_order, dt, P, C, a=None, c=None, nt=1, step0=0,
               src=(), wavelet=None, rec=(), ftz=True, Tt=4, Tz=8, Ty=8, B=3, skew=None):
    """O2: the paper's skewed time-tiled order; skew defaults to the radius."""
    skew = order // 2 if skew is None else skew
    return _run("skewed", ndim, n, order, coeffs, h, time_order, dt, P, C, a, c, nt, step0,
                src, wavelet, rec, ftz, extra=(Tt, Tz, Ty, B, skew))


def run_slabs(ndim, n, order, coeffs, h, time_order, dt, P, C, a=None, c=None, nt=1, step0=0,
              src=(), wavelet=None, rec=(), ftz=True, nslab=2, tc=1, ghost=None):
    """O3: the GPU's z-slab schedule emulated with plain loops (oracle.cpp run_slabs): nslab slabs,
    ghost planes (default radius*tc) refreshed every tc steps, shrinking redundant regions.
    fp32 only.  Equals O1 bit for bit when ghost >= radius*tc."""
    assert P.dtype == np.float32
    ghost = (order // 2) * tc if ghost is None else ghost
    dtype = P.dtype
    r = order // 2
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    h = np.ascontiguousarray(h, dtype=np.float64)
    src, rec = list(src or []), list(rec or [])
    src_a, rec_a = _pts(src), _pts(rec)
    if src:
        wavelet = np.ascontiguousarray(wavelet, dtype=dtype)
    trace = np.zeros((nt, max(len(rec), 1)), dtype=dtype)
    if time_order == 2:
        a = np.ascontiguousarray(a, dtype=dtype)
        c = np.ascontiguousarray(c, dtype=dtype)
    rc = _load().oracle_run_slabs_f32(ndim, n[0], n[1], n[2], r, _ptr(coeffs), _ptr(h), time_order,
                                      float(dt), _ptr(P), _ptr(C), _ptr(a) if time_order == 2 else None,
                                      _ptr(c) if time_order == 2 else None, nt, step0, len(src),
                                      _ptr(src_a), _ptr(wavelet) if src else None, len(rec), _ptr(rec_a),
                                      _ptr(trace), int(ftz), nslab, tc, ghost)
    if rc != 0:
        raise ValueError(f"oracle_run_slabs rejected its arguments (rc={rc})")
    return trace[:, :len(rec)]


def run_literal(ndim, n, order, coeffs, h, dt, P, C, vel, damp, nt=1, step0=0, src=(), wavelet=None,
                rec=(), ftz=True):
    """O1-literal: the wave update in the paper's printed expression and term order
    (oracle.cpp), from vel/damp instead of a/c.  Isotropic spacing only."""
    dtype = P.dtype
    r = order // 2
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    h = np.ascontiguousarray(h, dtype=np.float64)
    src, rec = list(src or []), list(rec or [])
    src_a, rec_a = _pts(src), _pts(rec)
    if src:
        wavelet = np.ascontiguousarray(wavelet, dtype=dtype)
    trace = np.zeros((nt, max(len(rec), 1)), dtype=dtype)
    vel = np.ascontiguousarray(vel, dtype=dtype)
    damp = np.ascontiguousarray(damp, dtype=dtype)
    fn = _load().oracle_run_literal_f32 if dtype == np.float32 else _load().oracle_run_literal_f64
    rc = fn(ndim, n[0], n[1], n[2], r, _ptr(coeffs), _ptr(h), float(dt), _ptr(P), _ptr(C), _ptr(vel),
            _ptr(damp), nt, step0, len(src), _ptr(src_a), _ptr(wavelet) if src else None, len(rec),
            _ptr(rec_a), _ptr(trace), int(ftz))
    if rc != 0:
        raise ValueError(f"oracle_run_literal rejected its arguments (rc={rc})")
    return trace[:, :len(rec)]


def run_problem(p, nt=None, dtype=np.float32, kind="untiled", ftz=True, **kw):
    """Convenience: run a workloads.Problem from its generated inputs; returns (P, C, trace)
    as interior arrays."""
    import workloads as W
    nt = p.nt if nt is None else nt
    r = p.radius
    up, uc = W.initial_fields(p)
    P = embed(up, p.ndim, r, dtype)
    C = embed(uc, p.ndim, r, dtype)
    a = c = None
    if p.time_order == 2:
        vel = embed(W.velocity(p), p.ndim, r, dtype)
        vel[vel == 0] = 1.0          # halo cells: any nonzero value, never used
        dmp = embed(W.damp(p), p.ndim, r, dtype)
        a, c = medium(vel, dmp, p.dt, dtype=dtype, ftz=ftz)
    wv = W.wavelet(p, nt).astype(dtype) if p.src else None
    if kind == "slabs":
        h = p.dx[:p.ndim] if p.ndim == 3 else p.dx[:2]
        tr = run_slabs(p.ndim, p.n, p.space_order, fd_weights(p.space_order), h, p.time_order, p.dt, P, C,
                       a, c, nt, 0, list(p.src), wv, list(p.rec), ftz, **kw)
        return extract(P, p.ndim, p.n, r), extract(C, p.ndim, p.n, r), tr
    if kind == "literal":
        assert p.time_order == 2
        vel = embed(W.velocity(p), p.ndim, r, dtype)
        vel[vel == 0] = 1.0
        dmp = embed(W.damp(p), p.ndim, r, dtype)
        del a, c
        h = p.dx[:p.ndim] if p.ndim == 3 else p.dx[:2]
        tr = run_literal(p.ndim, p.n, p.space_order, fd_weights(p.space_order), h, p.dt, P, C, vel, dmp,
                         nt, 0, list(p.src), wv, list(p.rec), ftz)
        return extract(P, p.ndim, p.n, r), extract(C, p.ndim, p.n, r), tr
    fn = run_untiled if kind == "untiled" else run_skewed
    tr = fn(p.ndim, p.n, p.space_order, fd_weights(p.space_order), p.dx[:p.ndim] if p.ndim == 3 else p.dx[:2],
            p.time_order, p.dt, P, C, a, c, nt, 0, list(p.src), wv, list(p.rec), ftz, **kw)
    return extract(P, p.ndim, p.n, r), extract(C, p.ndim, p.n, r), tr
