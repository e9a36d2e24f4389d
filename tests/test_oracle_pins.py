"""CPU: pins the oracle restatement (oracle/gmpea_oracle.cpp) before it is
trusted as the GPU checker — against published known-answer vectors, the
committed golden fixtures (made by the unmodified reference) and, where the
reference build is present, against the reference itself."""
import os
import numpy as np
import pytest

from conftest import GOLDEN, MW_PROBLEMS, REF_PROBLEMS, golden


def test_philox_random123_kat(orc):
    # Random123 kat_vectors, philox4x32_10
    assert list(orc.philox([0, 0, 0, 0], [0, 0])) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert list(orc.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6,
                                                                     0x6D5451FD]
    assert list(orc.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0])) == [
        0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


@pytest.mark.parametrize("name", REF_PROBLEMS + MW_PROBLEMS)
def test_eval_matches_golden(orc, name):
    gd = golden("eval.npz")
    F, G, cv = orc.evaluate(name, gd[f"{name}/X"])
    # bit-identical: same formulas, same operation order, same libm
    assert np.array_equal(F, gd[f"{name}/F"])
    assert np.array_equal(G, gd[f"{name}/G"])
    assert np.array_equal(cv, gd[f"{name}/cv"])


def test_known_answers(orc):
    # tests/test_problems.cpp:70-80: C1-DTLZ1 at x = (0.5, 0.5, 0.5...) -> f = (0.125, 0.125, 0.25)
    F, G, cv = orc.evaluate("C1-DTLZ1", np.full((1, 7), 0.5))
    assert np.allclose(F[0], [0.125, 0.125, 0.25])
    # tests/test_scalarize.cpp:138-153: PBI along / at / perpendicular to the axis
    assert orc.pbi([1.0, 0.0], [1.0, 0.0], [0.0, 0.0]) == 1.0
    assert orc.pbi([0.0, 0.0], [1.0, 0.0], [0.0, 0.0]) == 0.0
    assert orc.pbi([0.0, 1.0], [1.0, 0.0], [0.0, 0.0]) == 5.0
    # tests/test_metrics.cpp:32-41 IGD example
    assert orc.igd(np.array([[0.0, 0.0]]), np.array([[3.0, 4.0], [0.0, 0.0]])) == 2.5
    # tests/test_metrics.cpp:66-85 HV examples
    assert orc.hypervolume(np.array([[0.0, 0.0]]), [1.0, 1.0]) == 1.0
    assert orc.hypervolume(np.array([[0.0, 1.0], [1.0, 0.0]]), [2.0, 2.0]) == 3.0


def test_lattice_and_knn_match_golden(orc):
    gd = golden("knn.npz")
    keys = sorted({k.split("/")[0] for k in gd.files})
    for key in keys:
        W = gd[key + "/W"]
        if key.startswith("lat_"):
            _, m, n, t1, t2 = key.split("_")
            assert np.array_equal(orc.reference_vectors(int(m), int(n)), W)
        if W.shape[0] <= 1100:
            assert np.array_equal(orc.knn(W, gd[key + "/B1"].shape[1]), gd[key + "/B1"]), key
            assert np.array_equal(orc.knn(W, gd[key + "/B2"].shape[1]), gd[key + "/B2"]), key
        if key.startswith("lat_"):
            # the windowed lattice KNN (CPU-baseline topology) == build_neighborhoods
            B1, B2 = orc.lattice_knn(int(m), int(n), int(t1), int(t2), threads=2)
            assert np.array_equal(B1, gd[key + "/B1"]) and np.array_equal(B2, gd[key + "/B2"]), key


def test_selection_matches_golden(orc):
    gd = golden("selection.npz")
    for k in range(int(gd["count"])):
        pre = f"{k}/"
        pops = [dict(F=gd[pre + f"{i}F"], cv=gd[pre + f"{i}cv"]) for i in range(4)]
        s1, s2 = orc.selection(pops, gd[pre + "W"], gd[pre + "z"], 5.0, gd[pre + "B1"], gd[pre + "B2"])
        assert np.array_equal(s1, gd[pre + "src1"]) and np.array_equal(s2, gd[pre + "src2"]), k


def test_metrics_match_golden(orc):
    gd = golden("metrics.npz")
    for k in range(24):
        pre = f"{k}/"
        F, cv = gd[pre + "F"], gd[pre + "cv"]
        idx = orc.metric_front(F, cv)
        assert np.array_equal(F[idx], gd[pre + "front"])
        assert orc.igd(F, gd[pre + "R"]) == float(gd[pre + "igd"])
        m = F.shape[1]
        assert orc.hypervolume(gd[pre + "P"], np.full(m, 1.1)) == float(gd[pre + "hv"])


def test_many_objective_operators_match_golden(orc):
    """m > 3 (lattice, KNN, metric_front, IGD, Monte-Carlo HV) against the
    reference's own outputs (make_golden.py many_obj_fixture)."""
    gd = golden("many_obj.npz")
    for key in sorted({k.split("/")[0] for k in gd.files}):
        if key.startswith("lat_"):
            _, m, n, t1, t2 = key.split("_")
            W = gd[key + "/W"]
            assert np.array_equal(orc.reference_vectors(int(m), int(n)), W), key
            assert np.array_equal(orc.knn(W, int(t1)), gd[key + "/B1"]), key
            assert np.array_equal(orc.knn(W, int(t2)), gd[key + "/B2"]), key
        else:
            pre = key + "/"
            F, cv = gd[pre + "F"], gd[pre + "cv"]
            assert np.array_equal(F[orc.metric_front(F, cv)], gd[pre + "front"]), key
            assert orc.igd(F, gd[pre + "R"]) == float(gd[pre + "igd"]), key
            m = F.shape[1]
            assert orc.hypervolume(gd[pre + "P"], np.full(m, 1.1)) == float(gd[pre + "hv"]), key


def test_wta_scenarios_match_reference(orc, ref):
    for num in range(1, 11):
        a, b = orc.wta_scenario(num), ref.wta_scenario(num)
        for k in a:
            assert np.array_equal(a[k], b[k]), (num, k)


def test_oracle_selection_equals_reference_live(orc, ref):
    """Acceptance criterion 1 protocol (tests/acceptance.cpp:78-119) on fresh instances."""
    rng = np.random.default_rng(9001)
    for _ in range(100):
        n = int(rng.integers(4, 33))
        m = int(rng.integers(2, 4))
        nc = int(rng.integers(1, 4))
        pops = []
        for _ in range(4):
            Cm = rng.uniform(-1, 1, (n, nc))
            feas = rng.random(n) < 0.35
            Cm[feas] = -np.abs(Cm[feas])
            pops.append(dict(X=rng.random((n, 2)), F=rng.uniform(0, 5, (n, m)), C=Cm,
                             cv=np.array([orc.cv(c, nc) for c in Cm])))
        W = 0.05 + rng.random((n, m))
        W /= W.sum(1, keepdims=True)
        z = rng.uniform(-0.5, 0.5, m)
        t1 = 1 + int(rng.integers(0, min(n, 5)))
        t2 = t1 + int(rng.integers(0, n - t1 + 1))
        B1, B2 = ref.build_neighborhoods(W, t1, t2)
        outs = ref.environmental_selection(pops, W, z, 5.0, B1, B2)
        s1, s2, mk1, mk2 = orc.selection(pops, W, z, 5.0, B1, B2, want_marks=True)
        rm1, rm2 = ref.op2_marks(pops, W, z, 5.0, B1, B2)
        assert np.array_equal(mk1, rm1) and np.array_equal(mk2, rm2)
        for s, o, par in ((s1, outs[0], pops[0]), (s2, outs[1], pops[1])):
            exp = par["F"].copy()
            for j in range(n):
                if s[j] >= 0:
                    exp[j] = (pops[2] if s[j] < n else pops[3])["F"][s[j] % n]
            assert np.array_equal(exp, o["F"])


def test_oracle_eval_equals_reference_live(orc, ref):
    rng = np.random.default_rng(46)
    for name in REF_PROBLEMS:
        X = rng.random((200, ref.problem_info(name)["d"]))
        for a, b in zip(orc.evaluate(name, X), ref.evaluate(name, X)):
            assert np.array_equal(a, b), name


def test_oracle_reproduce_identities(orc):
    """tests/test_gmpea.cpp:141-188 identities on the Philox restatement."""
    rng = np.random.default_rng(503)
    X = rng.random((40, 30))
    W = orc.reference_vectors(2, 40)
    nb = orc.knn(W, 5)
    # bounds
    for op in (0, 1):
        off, _ = orc.reproduce("LIRCMOP1", X, nb, op, seed=5, gen=1, pop=1)
        assert off.min() >= 0.0 and off.max() <= 1.0
    # SBX prob 0, no mutation: the child is parent a
    same = np.full((10, 30), 0.5)
    nb10 = orc.knn(orc.reference_vectors(2, 10), 3)
    off, _ = orc.reproduce("LIRCMOP1", same, nb10, 0, 1, 1, 1, params=(0.0, 20, 20, 1.0, 0.5), pm_prob=0.0)
    assert np.array_equal(off, same)
    # DE with F = 0, CR = 1, no mutation: the trial equals the base vector
    off, _ = orc.reproduce("LIRCMOP1", X[:10], nb10, 1, 1, 1, 1, params=(1.0, 20, 20, 1.0, 0.0), pm_prob=0.0)
    assert np.array_equal(off, X[:10])


# ------------------------------------------------------------------ DAS-CMOP
# DAS-CMOP1-9 have no reference counterpart: "parity unpinned".
# The oracle's restatement is cross-checked against a second, independent
# vectorised restatement of the published definitions (Fan et al., Evol.
# Comput. 28(3), 2020; difficulty triplet (0.5, 0.5, 0.5)) and against closed
# forms on the Pareto set.
def das_numpy(k, X):
    a, b, d, r = 20.0, 0.0, 0.5, 0.25
    e = d - np.log(0.5)
    x1 = X[:, 0]
    m = 3 if k >= 7 else 2
    y = X[:, m - 1:] - (np.sin(0.5 * np.pi * x1)[:, None] if m == 2 else 0.5)
    if k in (4, 5, 6, 9):
        g = (X.shape[1] - m + 1) + np.sum(y * y - np.cos(20.0 * np.pi * y), axis=1)
    else:
        g = np.sum(y * y, axis=1)
    cons = [b - np.sin(a * np.pi * x1)]
    if m == 2:
        h = {0: 1 - x1 ** 2, 1: 1 - np.sqrt(x1), 2: 1 - np.sqrt(x1) + 0.5 * np.abs(np.sin(5 * np.pi * x1))}[(k - 1) % 3]
        F = np.stack([x1 + g, h + g], 1)
        cons.append(-(e - g) * (g - d))
        th = -0.25 * np.pi
        for p, q in zip([0, 1, 0, 1, 2, 0, 1, 2, 3], [1.5, 0.5, 2.5, 1.5, 0.5, 3.5, 2.5, 1.5, 0.5]):
            u = (F[:, 0] - p) * np.cos(th) - (F[:, 1] - q) * np.sin(th)
            v = (F[:, 0] - p) * np.sin(th) + (F[:, 1] - q) * np.cos(th)
            cons.append(r - (u ** 2 / 0.09 + v ** 2 / 1.44))
    else:
        x2 = X[:, 1]
        if k == 7:
            F = np.stack([x1 * x2, x2 * (1 - x1), 1 - x2], 1) + g[:, None]
        else:
            c0, s0 = np.cos(0.5 * np.pi * x1), np.sin(0.5 * np.pi * x1)
            F = np.stack([c0 * np.cos(0.5 * np.pi * x2), c0 * np.sin(0.5 * np.pi * x2), s0], 1) + g[:, None]
        cons.append(b - np.cos(a * np.pi * x2))
        cons.append(-(e - g) * (g - d))
        t = 1 / np.sqrt(3)
        for P in ([1, 0, 0], [0, 1, 0], [0, 0, 1], [t, t, t]):
            cons.append(r * r - np.sum((F - np.array(P)) ** 2, 1))
    G = np.stack(cons, 1)
    return F, G, np.maximum(G, 0).sum(1)


@pytest.mark.parametrize("k", range(1, 10))
def test_dascmop_oracle_vs_independent_restatement(orc, k):
    rng = np.random.default_rng(k)
    X = rng.random((300, 30))
    # half the rows on / near the Pareto set (distance genes at their optimum)
    m = 3 if k >= 7 else 2
    opt = np.sin(0.5 * np.pi * X[:150, :1]) if m == 2 else np.full((150, 1), 0.5)
    # noise 0.02: g near 0 (type II violated); 0.15: g near the feasible band [d, e]
    sd = np.where(np.arange(150) < 75, 0.02, 0.15)[:, None]
    X[:150, m - 1:] = np.clip(opt + sd * rng.normal(0, 1, (150, 30 - m + 1)), 0, 1)
    F, G, cv = orc.evaluate(f"DASCMOP{k}", X)
    Fn, Gn, cvn = das_numpy(k, X)
    assert np.allclose(F, Fn, rtol=1e-12, atol=1e-12)
    assert np.allclose(G, Gn, rtol=1e-12, atol=1e-12)
    assert np.allclose(cv, cvn, rtol=1e-12, atol=1e-12)
    assert G.shape[1] == (7 if k >= 7 else 11)
    # both feasible and infeasible rows are exercised
    assert (cv == 0).any() or k in (4, 5, 6, 9)


def test_dascmop_known_answers(orc):
    # DAS-CMOP1 on its unconstrained Pareto set (g = 0): f = (x1, 1 - x1^2)
    x = np.zeros((1, 30))
    x[0, 0] = 0.25
    x[0, 1:] = np.sin(0.5 * np.pi * 0.25)
    F, G, cv = orc.evaluate("DASCMOP1", x)
    assert np.allclose(F[0], [0.25, 1 - 0.0625], atol=1e-15)
    # type II with g = 0: -(e - 0)(0 - d) = e d > 0 (the unconstrained set is infeasible)
    assert np.isclose(G[0, 1], 0.5 * (0.5 - np.log(0.5)))
    # type I: b - sin(20 pi x1) = -sin(5 pi) = 0 at x1 = 0.25
    assert abs(G[0, 0]) < 1e-14
    # DAS-CMOP7 at x3.. = 0.5 (g = 0): f = (x1 x2, x2 (1 - x1), 1 - x2), sum 1
    x = np.full((1, 30), 0.5)
    x[0, :2] = [0.2, 0.6]
    F, G, cv = orc.evaluate("DASCMOP7", x)
    assert np.allclose(F[0], [0.12, 0.48, 0.4], atol=1e-15)
    # DAS-CMOP9's Rastrigin distance vanishes at the same point: unit-sphere objectives
    F, _, _ = orc.evaluate("DASCMOP9", x)
    assert np.isclose(np.sum(F[0] ** 2), 1.0)


@pytest.mark.parametrize("name", MW_PROBLEMS + [f"DASCMOP{k}" for k in range(1, 10)])
def test_restated_front_candidates_are_feasible_and_in_bounds(orc, name):
    """Restated MW / DAS-CMOP front candidates (no reference counterpart):
    every row lies in the box, and the rows realise a feasible distance —
    positions that have one (the level scan found it; MW10 has few) give rows that
    evaluate feasible through the ordinary evaluator."""
    info = orc.problem_info(name)
    X = orc.front_candidates(name, 400)
    assert X.shape[1] == info["d"]
    assert np.all(X >= info["lo"]) and np.all(X <= info["hi"])
    F, G, cv = orc.evaluate(name, X)
    assert np.isfinite(F).all()
    assert (cv == 0.0).mean() >= 0.05, (cv == 0.0).mean()  # MW10: 8.5 % of positions


def test_wta_large_files_oracle_pinned_to_reference(orc):
    """The oracle's WTA restatement on the large scenario files (>= 24
    vehicles, up to 316 strike slots, capacities up to 12) equals the
    reference's own load_wta + make_wta_problem + evaluate bit for bit
    (tests/golden/wta_large.npz, made by the reference)."""
    from paper_2509_19821_b200.wta import load_wta

    gd = golden("wta_large.npz")
    for key in ("wta_P65", "wta_custom40", "wta_custom24"):
        inst = load_wta(os.path.join(GOLDEN, key + ".txt"))
        orc.wta_register(inst.scenario, inst.n_targets, inst.n_vehicles, inst.max_strikes, inst.capacity,
                         [v for row in inst.p for v in row])
        F, G, cv = orc.evaluate("WTA-" + inst.scenario, gd[key + "/X"].astype(np.float64))
        assert np.array_equal(F, gd[key + "/F"]) and np.array_equal(G, gd[key + "/G"])
        assert np.array_equal(cv, gd[key + "/cv"])


def test_wta_synthetic_scenarios_continue_the_reference_formula(orc):
    """wta_synthetic(num): the reference's scenario generator (wta.cpp:31-46)
    continued past P10 -- equal to wta_scenario for P1..P10, and to the
    oracle's restatement of the same formula up to P123 (64 vehicles)."""
    from paper_2509_19821_b200.wta import wta_scenario, wta_synthetic

    for num in range(1, 11):
        assert wta_synthetic(num) == wta_scenario(f"P{num}")
    for num in (11, 40, 65, 123):
        w, o = wta_synthetic(num), orc.wta_scenario(num)
        assert w.n_targets == 4 + 2 * (num - 1) and w.n_vehicles == 3 + (num - 1) // 2
        assert w.max_strikes == o["strikes"].tolist() and w.capacity == o["capacity"].tolist()
        assert [v for row in w.p for v in row] == o["p"].tolist()
    with pytest.raises(ValueError):
        wta_synthetic(124)
