"""Schedule planner: the paper's legality reasoning plus a roofline choice
of the time-tile depths.  Host-side only; it decides parameters, the CUDA library computes.

* dependences()      distance vectors of the star stencil's reads (u[t-1] at +-k along
                     each axis gives (1, +-k e_axis); the leapfrog's u[t-2] centre gives (2, 0)).
* skew_factors()     per spatial dim, the smallest f >= 0 with d_k + f d_t >= 0 for every dependence
                     ("skewed relative to the outermost loop by a factor equal to the negated value
                     of greatest negative dependence").  P:2084-2086 words it as the
                     greatest *positive* distance; for the symmetric star stencils both are r.
* band_permutable()  a band of loops may be tiled rectangularly iff every (skewed) dependence is
                     non-negative in every band dim.
* plan()             T_k (on-chip levels per pass) and T_c (halo depth in steps between exchanges)
                     from the measured B200 behaviour and a halo-exchange cost model.

Axes are ordered (t, z, y, x), the build's naming (x contiguous, z streamed).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Sequence, Tuple

Vec = Tuple[int, ...]


def dependences(radius: int, time_order: int = 2, ndim: int = 3) -> List[Vec]:
    """Flow-dependence distance vectors (t, z, y, x) of u[t+1][p] = f(u[t][p +- k e], u[t-1][p])."""
    deps: List[Vec] = []
    nsp = 3
    axes = range(nsp - ndim, nsp)          # 2-D problems have no z dependences
    for k in range(1, radius + 1):
        for a in axes:
            for sgn in (1, -1):
                d = [1, 0, 0, 0]
                d[1 + a] = sgn * k
                deps.append(tuple(d))
    deps.append((1, 0, 0, 0))              # the centre term u[t][p]
    if time_order == 2:
        deps.append((2, 0, 0, 0))          # the leapfrog's u[t-1][p]
    return deps


def skew_factors(deps: Sequence[Vec], dims: Sequence[int]) -> Dict[int, int]:
    """Smallest non-negative f_k per spatial dim k (1..3 in (t, z, y, x)) with d_k + f_k d_t >= 0."""
    out = {}
    for k in dims:
        f = 0
        for d in deps:
            if d[0] <= 0:
                raise ValueError(f"dependence {d} has no positive time component")
            if d[k] < 0:
                f = max(f, -(d[k] // d[0]))      # ceil(-d_k / d_t)
        out[k] = f
    return out


def skew(deps: Sequence[Vec], factors: Dict[int, int]) -> List[Vec]:
    """Distances after x_k' = x_k + f_k t (the body index is un-skewed by the same amount)."""
    return [tuple(d[i] + factors.get(i, 0) * d[0] if i else d[0] for i in range(len(d))) for d in deps]


def band_permutable(deps: Sequence[Vec], band: Sequence[int]) -> bool:
    return all(d[k] >= 0 for d in deps for k in band)


@dataclasses.dataclass(frozen=True)
class Plan:
    t_kernel: int
    t_comm: int
    skew: int
    reason: str


# Measured on B200 (profiles/r02/study_tiling_vs_order.jsonl and
# profiles/r02/heat_tiling.txt: 512^3, wave 200 steps, heat 96 steps, one box): GPts/s per T_k of
# the instance build.py compiles for the shape (wave T_k = 2: r <= 2 overlapped tiles sweep2,
# r >= 3 the L1/L2 exchange pass sweepx; heat T_k = 2..4: the register-resident sweeph).
_MEASURED = {  # (time_order, radius): {T_k: GPts/s}
    (2, 1): {1: 334.5, 2: 424.8}, (2, 2): {1: 332.7, 2: 380.0}, (2, 3): {1: 321.7, 2: 264.1},
    (2, 4): {1: 319.6, 2: 250.4}, (2, 5): {1: 326.2, 2: 228.8}, (2, 6): {1: 318.7, 2: 205.9},
    (2, 7): {1: 264.8, 2: 178.4}, (2, 8): {1: 247.5, 2: 118.2},
    (1, 1): {1: 735.8, 2: 1176.3, 3: 1169.2, 4: 1204.7},
}
# grids whose own measurement differs from the 512^3 ranking (tile raggedness, L2 residency)
_MEASURED_GRID = {
    (1, 1, (256, 256, 256)): {1: 625.3, 2: 904.2, 3: 980.4, 4: 1017.4},   # C2
}
NVLINK_GBS = 770.0          # measured peer copy per direction (B200_PROFILING.md)
EXCHANGE_LATENCY_US = 25.0  # NCCL send/recv launch + sync per exchange (estimate)


def plan(time_order: int, radius: int, n: Sequence[int], nranks: int = 1, ndim: int = 3,
         supported=None) -> Plan:
    """Choose (t_kernel, t_comm).  supported(t_kernel) -> bool restricts to compiled instances."""
    deps = dependences(radius, time_order, ndim)
    f = skew_factors(deps, [1, 2, 3])
    skewed = skew(deps, f)
    assert band_permutable(skewed, [0, 1, 2, 3]) and f[3 if ndim == 2 else 1] == radius
    ok = supported or (lambda tk: True)
    rates = _MEASURED_GRID.get((time_order, radius, tuple(n)), _MEASURED.get((time_order, radius), {}))
    t1 = rates.get(1, 1.0)
    cands = [k for k in sorted(rates) if k > 1 and ndim == 3 and ok(k)]
    tk = max(cands, key=lambda k: rates[k], default=1)
    if tk > 1 and rates[tk] <= t1:
        tk = 1
    others = ", ".join(f"T_k={k} {rates[k]}" for k in sorted(rates) if k > 1)
    why = (f"T_k={tk} measured {rates[tk]} vs T=1 {t1} GPts/s" if tk > 1 else
           f"T=1 (measured {t1} vs {others} GPts/s)" if others else
           "T=1 (no T_k > 1 measurement for this shape)")
    tc = tk
    if nranks > 1:
        nx, ny, nz = n
        nzl = nz // nranks
        rate = 1e9 * max(t1, rates.get(tk, 0.0))
        step_s = nx * ny * nzl / rate
        best = None
        for cand in (1, 2, 4, 8, 16):
            if cand % tk or radius * cand > nzl:
                continue
            planes = radius * cand + radius * (cand - 1) * (time_order == 2)
            t_ex = EXCHANGE_LATENCY_US * 1e-6 + planes * nx * ny * 4 / (NVLINK_GBS * 1e9)
            redundant = radius * (cand - 1) / nzl            # extra planes computed per step
            per_step = step_s * (1 + redundant) + t_ex / cand   # exchange not overlapped (bound)
            if best is None or per_step < best[0] - 1e-12:
                best = (per_step, cand)
        tc = best[1] if best else tk
        why += f"; T_c={tc} minimises exchange latency + redundant ghost work"
    return Plan(tk, tc, f[1] if ndim == 3 else f[3], why)
