"""Planner: the paper's dependence / skew / legality reasoning, checked
against the paper's worked values and SPEC.md's examples, and the schedule choice."""
import itertools

from paper_1707_02347_b200 import planner as PL


def test_awe_so8_dependences_are_the_papers():
    """the outermost reads give (1,0,0,+-4), (1,0,+-4,0), (1,+-4,0,0)."""
    d = set(PL.dependences(4, 2, 3))
    for v in [(1, 0, 0, 4), (1, 0, 0, -4), (1, 0, 4, 0), (1, 0, -4, 0), (1, 4, 0, 0), (1, -4, 0, 0)]:
        assert v in d
    assert (2, 0, 0, 0) in d and len(d) == 6 * 4 + 2


def test_skew_factor_is_the_radius():
    """'int skew = 4*time' for SO8; r for every order."""
    for r in range(1, 9):
        f = PL.skew_factors(PL.dependences(r, 2, 3), [1, 2, 3])
        assert f == {1: r, 2: r, 3: r}


def test_skew_factor_spec_examples():
    """SPEC.md compute_skew_factors examples: {(1,1)} -> 0, {(2,-3)} -> 2."""
    assert PL.skew_factors([(1, 1)], [1]) == {1: 0}
    assert PL.skew_factors([(2, -3)], [1]) == {1: 2}


def test_legality_after_skew_and_negative_control():
    deps = PL.dependences(4, 2, 3)
    assert not PL.band_permutable(deps, [0, 1, 2, 3])                 # negative distances
    assert PL.band_permutable(PL.skew(deps, {1: 4, 2: 4, 3: 4}), [0, 1, 2, 3])
    assert not PL.band_permutable(PL.skew(deps, {1: 3, 2: 4, 3: 4}), [0, 1, 2, 3])


def test_brute_force_skew_minimal():
    """The factor is the smallest legal one, by brute force over small dependence sets."""
    for dt, dk in itertools.product(range(1, 4), range(-6, 4)):
        f = PL.skew_factors([(dt, dk)], [1])[1]
        assert dk + f * dt >= 0 and (f == 0 or dk + (f - 1) * dt < 0)


def test_plan_choices():
    assert PL.plan(2, 1, (512, 512, 512)).t_kernel == 2     # SO2 wave: time tiling wins on B200
    assert PL.plan(2, 4, (512, 512, 512)).t_kernel == 1     # SO8: untiled at the HBM roof
    assert PL.plan(1, 1, (256, 256, 256)).t_kernel == 4     # heat C2: register-resident sweeph
    assert PL.plan(1, 1, (512, 512, 512)).t_kernel == 4
    assert PL.plan(1, 1, (256, 256, 256), supported=lambda k: k <= 2).t_kernel == 2
    assert PL.plan(2, 6, (768, 768, 768)).t_kernel == 1
    p = PL.plan(2, 1, (768, 768, 768 * 8), nranks=8)
    assert p.t_comm % p.t_kernel == 0 and p.t_comm * 1 <= 768 and p.skew == 1
    p = PL.plan(2, 6, (768, 768, 768 * 8), nranks=8)
    assert p.t_comm >= 1 and 6 * p.t_comm <= 768
