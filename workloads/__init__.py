"""Seeded synthetic inputs for the stencil hot path.

This module is the ONLY code shared by the CUDA product path and the CPU oracle
(tests/bench feed both from here).  It holds no arithmetic of the method itself:
no finite-difference weights, no medium precompute (m, a, c), no update rule.
It only produces the problem *inputs*: grid sizes, initial fields, velocity,
damping (sponge) field, time step, Ricker wavelet, source/receiver coordinates.

Every generated value is a pure function of (config, seed, GLOBAL interior
index), so any z-slab decomposition reproduces the same global arrays
(decomposition invariance).

Readings of the paper/BASELINE that fix these recipes are listed in DESIGN.md
(§"Readings"); the ids Q1..Q17 below refer to SURVEY.md §8(c).

Array convention: interior arrays are numpy float32 with shape (nz, ny, nx),
x fastest (build axis naming, SURVEY.md §8 conventions).  2-D problems have
nz == 1.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Problem", "problem", "splitmix64", "uniform01", "initial_fields",
    "velocity", "damp", "wavelet", "eigenmode_2d", "CONFIG_NAMES",
]

CONFIG_NAMES = ("C1", "C2", "C3", "C4", "C5", "P256", "P256L", "P384")

# Paper-replica workloads (SURVEY.md §8(f) NEXT-2 i): the paper's own source-free AWE SO8 runs
# (P:1787-1815): grid N^3 inside an (N+20)^3 array whose loops update indices
# 4..N+15, dt = 3.04 and h = 20 (the printed constants, P:1678-1708 =
# 2dt^2/h^2 x SO8 weights), Gaussian sigma = 0.4 on [-1, 1]^3 over the whole array.
PAPER_REPLICA = {"P256": (256, 33), "P256L": (256, 247), "P384": (384, 165)}

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser applied elementwise to uint64 (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + _GOLDEN
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniform01(seed: int, idx: np.ndarray) -> np.ndarray:
    """U[0,1) in float32, exactly 24-bit: (splitmix64(seed ^ idx) >> 40) * 2^-24 (Q16)."""
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed) ^ np.asarray(idx, dtype=np.uint64))
    return ((h >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)).astype(np.float32)


@dataclasses.dataclass(frozen=True)
class Problem:
    """One synthetic workload."""
    name: str
    ndim: int                      # 2 or 3
    n: Tuple[int, int, int]        # GLOBAL interior points (nx, ny, nz); nz == 1 for 2-D (Q1)
    space_order: int               # 2..16
    time_order: int                # 1 = heat, 2 = damped leapfrog wave
    dt: float
    dx: Tuple[float, float, float]
    nt: int
    init: str                      # "uniform" | "zero" | "eigenmode" | "gaussian"
    seed: int = 0
    layers: Optional[Tuple[float, ...]] = None   # velocity per equal-thickness z-layer (m/s)
    perturb: float = 0.0           # relative velocity perturbation amplitude (C4: 0.05)
    perturb_seed: int = 1234
    f_peak: Optional[float] = None # Ricker peak frequency (Hz)
    sponge: int = 0                # sponge width in points (Q14)
    src: Tuple[Tuple[int, int, int], ...] = ()
    rec: Tuple[Tuple[int, int, int], ...] = ()

    @property
    def radius(self) -> int:
        return self.space_order // 2

    @property
    def points(self) -> int:
        return self.n[0] * self.n[1] * self.n[2]

    @property
    def vmax(self) -> float:
        """Upper bound of the velocity field (used for CFL dt and sponge strength, Q10/Q11)."""
        return max(self.layers) * (1.0 + self.perturb) if self.layers else 0.0


def _cfl_dt(dx: float, vmax: float, cfl: float = 0.4) -> float:
    return cfl * dx / vmax


def _centre(n):
    return (n[0] // 2, n[1] // 2, n[2] // 2)


def _receiver_lattice(n, z: int, margin: int, count: int = 10):
    """count x count lattice on plane z (Q15): x_i = margin + floor((i+0.5)(N-2margin)/count)."""
    xs = [margin + int(math.floor((i + 0.5) * (n[0] - 2 * margin) / count)) for i in range(count)]
    ys = [margin + int(math.floor((j + 0.5) * (n[1] - 2 * margin) / count)) for j in range(count)]
    return tuple((x, y, z) for y in ys for x in xs)


def problem(name: str, n: Optional[Sequence[int]] = None, nt: Optional[int] = None,
            gpus: int = 1, sponge: Optional[int] = None) -> Problem:
    """Config C1..C5 (BASELINE.json configs); n/nt/sponge override for scaled tests.

    For C5 the global z extent is 768 * gpus (weak scaling)."""
    name = name.upper()
    if name == "C1":
        nn = tuple(n) if n is not None else (128, 128, 1)
        return Problem("C1", 2, (nn[0], nn[1], 1), 2, 1, 0.1, (1.0, 1.0, 1.0),
                       nt if nt is not None else 20, "uniform", seed=0)
    if name == "C2":
        nn = tuple(n) if n is not None else (256, 256, 256)
        return Problem("C2", 3, nn, 2, 1, 0.1, (1.0, 1.0, 1.0),
                       nt if nt is not None else 100, "uniform", seed=0)
    layers = (1500.0, 2500.0, 3500.0, 4500.0)
    if name == "C3":
        nn = tuple(n) if n is not None else (512, 512, 512)
        sp = 40 if sponge is None else sponge
        return Problem("C3", 3, nn, 8, 2, _cfl_dt(10.0, max(layers)), (10.0, 10.0, 10.0),
                       nt if nt is not None else 500, "zero", layers=layers, f_peak=15.0,
                       sponge=sp, src=(_centre(nn),))
    if name == "C4":
        nn = tuple(n) if n is not None else (1024, 1024, 1024)
        sp = 40 if sponge is None else sponge
        vmax = max(layers) * 1.05
        return Problem("C4", 3, nn, 16, 2, _cfl_dt(10.0, vmax), (10.0, 10.0, 10.0),
                       nt if nt is not None else 1000, "zero", layers=layers, perturb=0.05,
                       perturb_seed=1234, f_peak=10.0, sponge=sp, src=(_centre(nn),))
    if name == "C5":
        if n is not None:
            nn = tuple(n)
        else:
            nn = (768, 768, 768 * gpus)
        sp = 40 if sponge is None else sponge
        return Problem("C5", 3, nn, 12, 2, _cfl_dt(10.0, max(layers)), (10.0, 10.0, 10.0),
                       nt if nt is not None else 2000, "zero", layers=layers, f_peak=15.0,
                       sponge=sp, src=(_centre(nn),),
                       rec=_receiver_lattice(nn, z=min(sp, nn[2] - 1), margin=sp))
    if name in PAPER_REPLICA:
        N, steps = PAPER_REPLICA[name]
        nn = tuple(n) if n is not None else (N + 12, N + 12, N + 12)   # (N+20) - 2*4 updated
        sp = 6 if sponge is None else sponge   # Devito's 10-point layer minus the 4-point halo
        return Problem(name, 3, nn, 8, 2, 3.04, (20.0, 20.0, 20.0), nt if nt is not None else steps,
                       "gaussian", layers=(1.5, 2.5), sponge=sp)
    raise ValueError(f"unknown config {name!r}")


def _zrange(z0: int, z1: int) -> np.ndarray:
    return np.arange(z0, z1, dtype=np.int64)


def initial_fields(p: Problem, z0: int = 0, z1: Optional[int] = None):
    """(u_prev, u_cur) interior arrays for global planes [z0, z1) (planes outside [0,nz) are 0).

    heat: u_cur ~ U[0,1) from splitmix64(seed ^ global linear index) (Q16); u_prev = 0 (unused).
    wave: u^{-1} = u^0 = 0 (the source drives the field, Q12)."""
    z1 = p.n[2] if z1 is None else z1
    nx, ny, nz = p.n
    shape = (z1 - z0, ny, nx)
    u_prev = np.zeros(shape, np.float32)
    if p.init == "zero":
        return u_prev, np.zeros(shape, np.float32)
    if p.init == "eigenmode":
        assert p.ndim == 2
        return u_prev, eigenmode_2d(nx, ny)[None].copy()
    if p.init == "gaussian":
        g = gaussian_3d(p.n, z0, z1)
        return g.copy(), g
    u = np.zeros(shape, np.float32)
    plane = np.uint64(nx * ny)
    base = (np.arange(ny, dtype=np.uint64)[:, None] * np.uint64(nx)
            + np.arange(nx, dtype=np.uint64)[None, :])
    for k, z in enumerate(range(z0, z1)):
        if 0 <= z < nz:
            u[k] = uniform01(p.seed, np.uint64(z) * plane + base)
    return u_prev, u


def gaussian_3d(n, z0: int = 0, z1: Optional[int] = None, sigma: float = 0.4, halo: int = 4) -> np.ndarray:
    """The paper's initial field: multivariate normal pdf, mean 0, sigma 0.4 per axis,
    on np.mgrid[-1:1:A j] over the whole array of A = n + 2*halo points per axis; interior index i
    sits at array index i + halo.  fp64, rounded to fp32.  Planes outside [0, nz) are 0."""
    nx, ny, nz = n
    z1 = nz if z1 is None else z1

    def axis(m, idx):
        a = m + 2 * halo
        x = -1.0 + 2.0 * (np.asarray(idx, dtype=np.float64) + halo) / (a - 1)
        return np.exp(-x * x / (2.0 * sigma * sigma))
    gx = axis(nx, np.arange(nx))
    gy = axis(ny, np.arange(ny))
    zs = np.arange(z0, z1)
    gz = np.where((zs >= 0) & (zs < nz), axis(nz, zs), 0.0)
    norm = 1.0 / ((2.0 * np.pi) ** 1.5 * sigma ** 3)
    return (norm * gz[:, None, None] * gy[None, :, None] * gx[None, None, :]).astype(np.float32)


def eigenmode_2d(nx: int, ny: int, dtype=np.float32) -> np.ndarray:
    """sin(pi i h_x) sin(pi j h_y), i = 1..nx, h = 1/(n+1) (Q4), computed in fp64, returned as dtype."""
    i = np.arange(1, nx + 1, dtype=np.float64)
    j = np.arange(1, ny + 1, dtype=np.float64)
    return (np.sin(np.pi * j / (ny + 1))[:, None] * np.sin(np.pi * i / (nx + 1))[None, :]).astype(dtype)


def velocity(p: Problem, z0: int = 0, z1: Optional[int] = None) -> np.ndarray:
    """Layered velocity (4 equal-thickness layers by GLOBAL depth z), optional +-perturb
    relative perturbation from splitmix64(perturb_seed ^ global index) (Q11)."""
    z1 = p.n[2] if z1 is None else z1
    nx, ny, nz = p.n
    nl = len(p.layers)
    zc = np.clip(_zrange(z0, z1), 0, nz - 1)
    layer = np.minimum(nl - 1, (zc * nl) // nz)
    lv = np.asarray(p.layers, dtype=np.float64)[layer]
    if p.perturb == 0.0:
        v = np.broadcast_to(lv.astype(np.float32)[:, None, None], (z1 - z0, ny, nx))
        return np.ascontiguousarray(v)
    out = np.empty((z1 - z0, ny, nx), np.float32)
    plane = np.uint64(nx * ny)
    base = (np.arange(ny, dtype=np.uint64)[:, None] * np.uint64(nx)
            + np.arange(nx, dtype=np.uint64)[None, :])
    for k, z in enumerate(zc):
        u = uniform01(p.perturb_seed, np.uint64(z) * plane + base).astype(np.float64)
        out[k] = (lv[k] * (1.0 + p.perturb * (2.0 * u - 1.0))).astype(np.float32)
    return out


def _sponge_profile(n: int, width: int, coords: np.ndarray) -> np.ndarray:
    """(d/W)^2 with d = points into the layer on either side (Q14)."""
    d = np.maximum(0, width - coords) + np.maximum(0, coords - (n - 1 - width))
    return (d.astype(np.float64) / width) ** 2


def damp(p: Problem, z0: int = 0, z1: Optional[int] = None) -> np.ndarray:
    """Sponge damping field eta of m u_tt + eta u_t = lap u, Q14 reading:
    eta = d / v^2 with the damping RATE d = d_max * sum_axes (d_a/W)^2 [1/s],
    d_max = 3 vmax ln(1e3) / (2 W dx), so that the equation is u_tt + d u_t = v^2 lap u
    and dt*d_max ~ 0.1 at CFL 0.4 with W = 40."""
    z1 = p.n[2] if z1 is None else z1
    nx, ny, nz = p.n
    if p.sponge <= 0:
        return np.zeros((z1 - z0, ny, nx), np.float32)
    W = p.sponge
    d_max = 3.0 * p.vmax * math.log(1000.0) / (2.0 * W * p.dx[0])
    px = _sponge_profile(nx, W, np.arange(nx))
    py = _sponge_profile(ny, W, np.arange(ny))
    pxy = py[:, None] + px[None, :]
    v = velocity(p, z0, z1).astype(np.float64)
    if p.ndim == 2:
        return (d_max * pxy[None] / (v * v)).astype(np.float32)
    pz = _sponge_profile(nz, W, np.clip(_zrange(z0, z1), 0, nz - 1))
    return (d_max * (pz[:, None, None] + pxy[None]) / (v * v)).astype(np.float32)


def wavelet(p: Problem, nt_total: Optional[int] = None) -> np.ndarray:
    """Ricker w(t) = (1 - 2 pi^2 f^2 (t-t0)^2) exp(-pi^2 f^2 (t-t0)^2), t0 = 1/f, t = n dt,
    amplitude 1, fp64 rounded to fp32 (Q12).  Shape (nt_total, nsrc)."""
    nt_total = p.nt if nt_total is None else nt_total
    if not p.src:
        return np.zeros((nt_total, 0), np.float32)
    f = p.f_peak
    t = np.arange(nt_total, dtype=np.float64) * p.dt - 1.0 / f
    a = (np.pi * f * t) ** 2
    w = ((1.0 - 2.0 * a) * np.exp(-a)).astype(np.float32)
    return np.repeat(w[:, None], len(p.src), axis=1).copy()
