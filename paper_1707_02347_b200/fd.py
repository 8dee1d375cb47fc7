"""Finite-difference weights of the second derivative (product side).

Fornberg's recursive algorithm (Math. Comp. 51, 1988) run in exact rational arithmetic on the
symmetric stencil offsets 0, +-1, ..., +-m.  Returns c_0..c_m of
    u''(x) ~ (1/h^2) [c_0 u(x) + sum_k c_k (u(x+kh) + u(x-kh))]
which for space order 8 are the weights behind the paper's printed AWE constants
(P:1682-1707 = 0.046208 x these).  Independent of the oracle's closed
form (oracle/__init__.py); tests check the two agree exactly.
"""
from __future__ import annotations

from fractions import Fraction
from functools import lru_cache
from typing import List

import numpy as np


@lru_cache(maxsize=None)
def fornberg_weights(order: int) -> tuple:
    if order < 2 or order % 2:
        raise ValueError("space order must be even and >= 2")
    m = order // 2
    # nodes ordered 0, 1, -1, 2, -2, ...
    xs: List[Fraction] = [Fraction(0)]
    for k in range(1, m + 1):
        xs += [Fraction(k), Fraction(-k)]
    n = len(xs) - 1
    M = 2   # derivative order
    z = Fraction(0)
    # delta[mm][nn][nu]
    delta = [[[Fraction(0)] * (n + 1) for _ in range(n + 1)] for _ in range(M + 1)]
    delta[0][0][0] = Fraction(1)
    c1 = Fraction(1)
    for nn in range(1, n + 1):
        c2 = Fraction(1)
        for nu in range(nn):
            c3 = xs[nn] - xs[nu]
            c2 *= c3
            for mm in range(min(nn, M) + 1):
                prev = delta[mm - 1][nn - 1][nu] if mm > 0 else Fraction(0)
                delta[mm][nn][nu] = ((xs[nn] - z) * delta[mm][nn - 1][nu] - mm * prev) / c3
        for mm in range(min(nn, M) + 1):
            prev = delta[mm - 1][nn - 1][nn - 1] if mm > 0 else Fraction(0)
            delta[mm][nn][nn] = c1 / c2 * (mm * prev - (xs[nn - 1] - z) * delta[mm][nn - 1][nn - 1])
        c1 = c2
    w = delta[M][n]
    out = [w[0]]
    for k in range(1, m + 1):
        assert w[2 * k - 1] == w[2 * k]          # symmetric stencil
        out.append(w[2 * k - 1])
    return tuple(out)


def fd_weights(order: int) -> np.ndarray:
    """c_0..c_m as float64 (correctly rounded from the exact rationals)."""
    return np.array([float(c) for c in fornberg_weights(order)], dtype=np.float64)
