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


# ------------------------------------------------------------ baseline runs
@pytest.mark.parametrize("algo,per", [("cnsga2", 1), ("ccmo", 2)])
def test_baseline_run_semantics(g, algo, per):
    """RunDriver (baselines.cpp:282-316): evals = per * n * (gen + 1), k_max
    generations, eval budget, determinism, bounds, feasible ratio of pop1."""
    p = g.make_problem("LIRCMOP1")
    r = g.run_baseline(p, algo, g.RunConfig(n=40, k_max=6, seed=3, record_walltime=False))
    assert [h.evals for h in r.history] == [per * 40 * (k + 1) for k in range(7)]
    again = g.run_baseline(p, algo, g.RunConfig(n=40, k_max=6, seed=3, record_walltime=False))
    assert np.array_equal(r.pop1.X, again.pop1.X)
    lo, hi = np.array(p.bounds).T
    assert np.all(r.pop1.X >= lo) and np.all(r.pop1.X <= hi)
    assert r.history[-1].feasible_ratio == np.mean(r.pop1.cv == 0.0)
    b = g.run_baseline(p, algo, g.RunConfig(n=40, k_max=0, eval_budget=per * 40 * 4 + 1, seed=3))
    assert b.history[-1].evals == per * 40 * 4
    re = g.evaluate_population(p, r.pop1.X)
    assert np.allclose(re.F, r.pop1.F, rtol=1e-6)


def test_baseline_igd_hook(g):
    from conftest import golden

    p = g.make_problem("LIRCMOP1")
    front = golden("fronts.npz")["LIRCMOP1"]
    r = g.run_baseline(p, "cnsga2", g.RunConfig(n=50, k_max=5, seed=1), igd_front=front)
    assert all(h.igd is not None for h in r.history)
    fr = g.metric_front(r.pop1)
    assert r.history[-1].igd == (g.igd(fr, front) if len(fr) else np.inf)


@pytest.mark.parametrize("key", ["cnsga2/LIRCMOP1", "cnsga2/C1-DTLZ1", "ccmo/LIRCMOP1"])
def test_baseline_statistical_parity_with_reference_runs(g, key):
    """Final IGD over the seeds of the reference's own runs (golden) vs the
    device runs: not significantly worse (Mann-Whitney U, p < 0.01)."""
    from scipy.stats import mannwhitneyu

    from conftest import golden

    gd = golden("baseline_runs.npz")
    algo, name = key.split("/")
    n, gens = (int(v) for v in gd[f"{key}/cfg"])
    ref_igd = gd[f"{key}/igd"]
    front = golden("fronts.npz")[name]
    p = g.make_problem(name)
    vals = []
    for seed in range(1, len(ref_igd) + 1):
        r = g.run_baseline(p, algo, g.RunConfig(n=n, k_max=gens, seed=seed, record_walltime=False))
        fr = g.metric_front(r.pop1)
        vals.append(g.igd(fr, front) if len(fr) else np.inf)
    vals = np.array(vals)
    worse = mannwhitneyu(vals, ref_igd, alternative="greater").pvalue
    assert worse >= 0.01, (np.median(vals), np.median(ref_igd), worse)
