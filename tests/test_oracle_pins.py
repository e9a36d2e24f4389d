"""CPU: pins the oracle restatement (oracle/gmpea_oracle.cpp) before it is
trusted as the GPU checker — against published known-answer vectors, the
committed golden fixtures (made by the unmodified reference) and, where the
reference build is present, against the reference itself."""
import numpy as np
import pytest

from conftest import MW_PROBLEMS, REF_PROBLEMS, golden


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
