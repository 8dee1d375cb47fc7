"""Paper-replica workloads (SURVEY.md §8(f) NEXT-2 i): the paper's own source-free AWE SO8 runs
 with dt = 3.04, h = 20 and a Gaussian initial field."""
import numpy as np
import pytest

import oracle
import workloads as W


def test_replica_constants_are_the_papers():
    """The replica's dt and h turn the SO8 weights into the constants printed at P:1682-1707."""
    p = W.problem("P256")
    fac = 2.0 * p.dt ** 2 / p.dx[0] ** 2
    w = oracle.fd_weights(8)
    printed = [-3.94693333333333e-1, 7.39328e-2, -9.2416e-3, 1.17353650793651e-3, -8.25142857142857e-5]
    got = [3 * fac * w[0]] + [fac * w[k] for k in range(1, 5)]
    for g, e in zip(got, printed):
        assert abs(g - e) <= 5e-7 * abs(e)
    assert p.space_order == 8 and p.time_order == 2 and not p.src
    # CFL: v_max dt / h = 0.38 (Devito's critical-dt factor), below the SO8 limit 0.4529
    assert abs(p.vmax * p.dt / p.dx[0] - 0.38) < 1e-12


def test_replica_grid_sizes():
    """(N+20)^3 arrays with loops 4..size-5: N+12 updated points per axis."""
    assert W.problem("P256").n == (268,) * 3 and W.problem("P384").n == (396,) * 3
    assert (W.problem("P256").nt, W.problem("P256L").nt, W.problem("P384").nt) == (33, 247, 165)


def test_gaussian_matches_scipy_multivariate_normal():
    """gaussian_3d == scipy.stats.multivariate_normal.pdf on np.mgrid[-1:1:Aj]^3 (the paper's own
    set-up code), A = n + 8, at sampled interior points (fp32 rounding)."""
    from scipy.stats import multivariate_normal
    n = (36, 30, 26)
    g = W.gaussian_3d(n)
    rng = np.random.default_rng(5)
    cov = np.diag(np.array([0.4, 0.4, 0.4]) ** 2)
    for _ in range(50):
        i, j, k = (int(rng.integers(0, m)) for m in n)          # x, y, z interior indices
        coords = [-1.0 + 2.0 * (idx + 4) / (m + 8 - 1) for idx, m in zip((i, j, k), n)]
        want = multivariate_normal.pdf(coords, mean=[0, 0, 0], cov=cov)
        assert abs(float(g[k, j, i]) - want) <= 1e-6 * want + 1e-30


def test_replica_oracle_small_energy_decays():
    """Scaled replica (zero-flux interior, sponge): the Gaussian pulse spreads; the oracle stays finite
    and its discrete energy does not grow (pin of the source-free path, cf. test_wave_energy)."""
    p = W.problem("P256", n=(40, 36, 32), nt=30, sponge=4)
    P, C, _ = oracle.run_problem(p, dtype=np.float64)
    assert np.isfinite(C).all() and np.abs(C).max() < W.gaussian_3d(p.n).max()
