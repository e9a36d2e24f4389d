"""GPU comparison-algorithm operators (baselines.hpp) against the unmodified
reference (oracle/_ref, baselines.cpp compiled from its own sources) on the
same inputs: ranks, kept indices exact; distances and fitness bit-equal."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cases(seed):
    """Random pools with duplicates, ties on an axis, exact zeros and
    infeasible rows with repeated cv values."""
    rng = np.random.default_rng(seed)
    out = []
    for n, m in ((1, 2), (2, 2), (7, 2), (60, 2), (300, 2), (257, 3), (900, 3)):
        F = np.round(rng.random((n, m)), 2 if seed % 2 else 6)
        if n > 4:
            F[1] = F[0]  # duplicate row
            F[3, 0] = F[2, 0]  # tie on an axis
        cv = np.where(rng.random(n) < 0.4, np.round(rng.random(n), 1), 0.0)
        out.append((F, cv))
    return out


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("cdp", [True, False])
def test_nondominated_sort_matches_reference(g, ref, seed, cdp):
    for F, cv in _cases(seed):
        assert np.array_equal(g.nondominated_sort(F, cv, cdp), ref.nondominated_sort(F, cv, cdp))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_crowding_distance_matches_reference(g, ref, seed):
    for F, cv in _cases(seed):
        n = F.shape[0]
        rng = np.random.default_rng(seed + n)
        for front in (np.arange(n), rng.permutation(n)[: max(1, n // 2)]):
            got, exp = g.crowding_distance(F, front), ref.crowding_distance(F, front)
            assert np.array_equal(got, exp), np.abs(got - exp).max()


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("cdp", [True, False])
def test_spea2_fitness_matches_reference(g, ref, seed, cdp):
    for F, cv in _cases(seed):
        assert np.array_equal(g.spea2_fitness(F, cv, cdp), ref.spea2_fitness(F, cv, cdp))


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("cdp", [True, False])
def test_spea2_select_matches_reference(g, ref, seed, cdp):
    for F, cv in _cases(seed):
        n = F.shape[0]
        if n > 300:  # the reference's serial truncation is cubic
            continue
        for cap in sorted({0, 1, max(1, n // 3), n // 2, n}):
            assert np.array_equal(g.spea2_select(F, cv, cdp, cap), ref.spea2_select(F, cv, cdp, cap)), (n, cap)


def test_cdp_rejects_negative_cv(g):
    F = np.zeros((3, 2))
    with pytest.raises(ValueError, match="negative constraint violation"):
        g.nondominated_sort(F, np.array([0.0, -1.0, 0.0]), True)
    with pytest.raises(ValueError, match="negative constraint violation"):
        g.spea2_fitness(F, np.array([0.0, -1.0, 0.0]), True)
