"""Generates the committed golden fixtures of tests/golden/ from the
UNMODIFIED reference (oracle/_ref/libgmpea_ref.so, built by oracle/Makefile
from /root/reference/proj/src).  Run here, where /root/reference exists:

    python tests/golden/make_golden.py

The GPU box has no /root/reference; the GPU parity tests read these files.
Inputs are fp32-representable so the fp32 engine sees exactly what the f64
reference saw.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import Oracle, Reference, build_ref  # noqa: E402

from conftest import DAS_PROBLEMS, MW_PROBLEMS, REF_PROBLEMS, f32  # noqa: E402


def eval_fixture(ref, orc, rng):
    out = {}
    for name in REF_PROBLEMS:
        d = ref.problem_info(name)["d"]
        X = f32(rng.random((64, d)))
        if name.startswith("WTA"):
            # exercise the 0.5 threshold and ties of the decode
            X[:8] = f32(np.round(X[:8] * 4) / 4)
        F, G, cv = ref.evaluate(name, X)
        out[f"{name}/X"], out[f"{name}/F"], out[f"{name}/G"], out[f"{name}/cv"] = X, F, G, cv
    for name in MW_PROBLEMS:  # unpinned: oracle restatement, recorded for regression only
        info = orc.problem_info(name)
        X = f32(info["lo"] + (info["hi"] - info["lo"]) * rng.random((64, info["d"])))
        F, G, cv = orc.evaluate(name, X)
        out[f"{name}/X"], out[f"{name}/F"], out[f"{name}/G"], out[f"{name}/cv"] = X, F, G, cv
    np.savez_compressed(os.path.join(HERE, "eval.npz"), **out)


def random_pop(rng, n, m, nc):
    """tests/oracles.cpp:545-565 shape: F ~ U(0,5), C ~ U(-1,1), ~35% feasible."""
    X = f32(rng.random((n, 2)))
    F = f32(rng.uniform(0.0, 5.0, (n, m)))
    Cm = f32(rng.uniform(-1.0, 1.0, (n, nc)))
    feas = rng.random(n) < 0.35
    Cm[feas] = -np.abs(Cm[feas])
    cv = f32(np.maximum(Cm, 0.0).sum(1))
    return dict(X=X, F=F, C=Cm, cv=cv)


def selection_fixture(ref, orc, rng, count=200):
    out = {"count": np.array(count)}
    for k in range(count):
        n = int(rng.integers(4, 33))
        m = int(rng.integers(2, 4))
        nc = int(rng.integers(1, 4))
        pops = [random_pop(rng, n, m, nc) for _ in range(4)]
        if k % 4 == 0:  # lattice weights (tests/test_gmpea.cpp:29-41)
            W = ref.reference_vectors(m, n)
        else:  # random positive weights (tests/acceptance.cpp:92-101)
            W = 0.05 + rng.random((n, m))
            W /= W.sum(1, keepdims=True)
        z = f32(rng.uniform(-0.5, 0.5, m))
        t1 = 1 + int(rng.integers(0, min(n, 5)))
        t2 = t1 + int(rng.integers(0, n - t1 + 1))
        B1, B2 = ref.build_neighborhoods(W, t1, t2)
        outs = ref.environmental_selection(pops, W, z, 5.0, B1, B2)
        s1, s2 = orc.selection(pops, W, z, 5.0, B1, B2)
        # the oracle's winner codes reproduce the reference's output rows exactly
        for s, o, par in ((s1, outs[0], pops[0]), (s2, outs[1], pops[1])):
            for key in ("X", "F", "C", "cv"):
                exp = par[key].copy()
                for j in range(n):
                    if s[j] >= 0:
                        exp[j] = (pops[2] if s[j] < n else pops[3])[key][s[j] % n]
                assert np.array_equal(exp, o[key])
        pre = f"{k}/"
        for i, p in enumerate(pops):
            for key in ("X", "F", "C", "cv"):
                out[pre + f"{i}{key}"] = p[key]
        out[pre + "W"], out[pre + "z"], out[pre + "B1"], out[pre + "B2"] = W, z, B1, B2
        out[pre + "src1"], out[pre + "src2"] = s1, s2
        for i in range(2):
            for key in ("X", "F", "C", "cv"):
                out[pre + f"out{i}{key}"] = outs[i][key]
    np.savez_compressed(os.path.join(HERE, "selection.npz"), **out)


def knn_fixture(ref, rng):
    out = {}
    cases = [(2, 5, 2, 5), (2, 100, 5, 20), (2, 1001, 5, 20), (3, 105, 5, 20), (3, 300, 5, 20),
             (3, 1000, 5, 20), (3, 3000, 5, 20), (2, 40, 20, 40), (3, 33, 33, 33)]
    for (m, n, t1, t2) in cases:
        W = ref.reference_vectors(m, n)
        B1, B2 = ref.build_neighborhoods(W, t1, t2)
        key = f"lat_{m}_{n}_{t1}_{t2}"
        out[key + "/W"], out[key + "/B1"], out[key + "/B2"] = W, B1, B2
    for k in range(10):
        n = int(rng.integers(4, 200))
        m = int(rng.integers(2, 4))
        W = 0.05 + rng.random((n, m))
        W /= W.sum(1, keepdims=True)
        t1 = int(rng.integers(1, min(n, 8) + 1))
        t2 = int(rng.integers(t1, min(n, 40) + 1))
        B1, B2 = ref.build_neighborhoods(W, t1, t2)
        key = f"rnd_{k}"
        out[key + "/W"], out[key + "/B1"], out[key + "/B2"] = W, B1, B2
    np.savez_compressed(os.path.join(HERE, "knn.npz"), **out)


def metrics_fixture(ref, rng):
    out = {}
    for k in range(24):
        m = 2 + k % 2
        n = int(rng.integers(1, 400))
        F = f32(rng.random((n, m)))
        F[rng.random(n) < 0.15] = F[0]  # duplicates
        cv = np.where(rng.random(n) < 0.3, rng.random(n), 0.0)
        R = rng.random((50, m))
        key = f"{k}/"
        out[key + "F"], out[key + "cv"], out[key + "R"] = F, cv, R
        out[key + "front"] = ref.metric_front(F, cv)
        out[key + "igd"] = np.array(ref.igd(F, R))
        P = f32(rng.random((n, m)) * 1.2)
        out[key + "P"] = P
        out[key + "hv"] = np.array(ref.hypervolume(P, np.full(m, 1.1)))
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)


def fronts_fixture(ref):
    out = {}
    for name in REF_PROBLEMS:
        if name.startswith("WTA"):
            continue
        out[name] = ref.pf_reference(name, 1000)
    np.savez_compressed(os.path.join(HERE, "fronts.npz"), **out)


def pf_fixture(ref):
    """pf_reference at sizes other than 1000 (small, and large enough to need
    the oversampling retries for some problems)."""
    out = {}
    for name in REF_PROBLEMS:
        if name.startswith("WTA"):
            continue
        for npts in (64, 2500):
            out[f"{name}/{npts}"] = ref.pf_reference(name, npts)
    np.savez_compressed(os.path.join(HERE, "pf_ref.npz"), **out)


def nondominated_rows(F):
    """fronts.cpp:15-42 (m = 2: lexicographic sweep, duplicates dropped; m = 3:
    pairwise Pareto dominance, duplicates kept)."""
    n = len(F)
    if F.shape[1] == 2:
        order = sorted(range(n), key=lambda i: (F[i, 0], F[i, 1]))  # stable
        keep, best = [], np.inf
        for i in order:
            if F[i, 1] < best:
                keep.append(i)
                best = F[i, 1]
        return np.array(sorted(keep), dtype=np.int64)
    keep = []
    for i in range(n):
        le = np.all(F <= F[i], axis=1) & np.any(F < F[i], axis=1)
        if not le.any():
            keep.append(i)
    return np.array(keep, dtype=np.int64)


def restated_nd_set(orc, name, n_points):
    """The nondominated candidate set pf_reference (fronts.cpp:54-79) subsamples
    for n_points, from the oracle's restated candidates."""
    m = orc.problem_info(name)["m"]
    over = max(8 * n_points, 2000)
    if m >= 3:
        over = min(over, 12000)
    for attempt in range(4):
        X = orc.front_candidates(name, over)
        F, G, cv = orc.evaluate(name, X)
        Ff = F[cv == 0.0]
        if len(Ff) >= max(n_points, 1):
            nd = Ff[nondominated_rows(Ff)]
            if len(nd) >= n_points or attempt == 3:
                return nd
        over *= 4
        if m >= 3:
            over = min(over, 50000)
    raise RuntimeError("no feasible front")


def restated_fronts_fixture(ref, orc):
    """MW / DAS-CMOP fronts: the reference's own pf_reference pipeline
    (fronts.cpp:54-103: evaluate, feasible filter, nondominated filter,
    subsample) over the oracle's restated front candidates (these suites have
    no reference counterpart; the candidates are wired in by oracle/ref_shim.cpp)."""
    out = {}
    for name in MW_PROBLEMS + DAS_PROBLEMS:
        for npts in (64, 1000):
            out[f"{name}/{npts}"] = ref.pf_reference(name, npts)
        out[f"{name}/nd64"] = restated_nd_set(orc, name, 64)
    np.savez_compressed(os.path.join(HERE, "pf_restated.npz"), **out)


def runs_fixture(ref):
    """Final IGD of the reference's own run_gmpea over 30 seeds (statistical parity)."""
    fronts = np.load(os.path.join(HERE, "fronts.npz"))
    out = {}
    for name, op, n, gens in (("LIRCMOP1", 1, 100, 200), ("LIRCMOP13", 1, 105, 200),
                              ("C1-DTLZ1", 0, 105, 300), ("LIRCMOP9", 1, 100, 200)):
        vals = []
        for seed in range(1, 31):
            pop, hist = ref.run_gmpea(name, n, k_max=gens, seed=seed, op=op, record_walltime=False)
            front = ref.metric_front(pop["F"], pop["cv"])
            vals.append(ref.igd(front, fronts[name]) if len(front) else np.inf)
        out[f"{name}/igd"] = np.array(vals)
        out[f"{name}/cfg"] = np.array([op, n, gens])
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **out)


def baseline_runs_fixture(ref):
    """Final IGD of the reference's own run_cnsga2 / run_ccmo (statistical parity)."""
    fronts = np.load(os.path.join(HERE, "fronts.npz"))
    out = {}
    for algo, name, n, gens, seeds in (("cnsga2", "LIRCMOP1", 100, 100, 30), ("cnsga2", "C1-DTLZ1", 91, 100, 30),
                                       ("ccmo", "LIRCMOP1", 60, 40, 30)):
        vals = []
        for seed in range(1, seeds + 1):
            pop, hist = ref.run_baseline(algo, name, n, gens, seed)
            front = ref.metric_front(pop["F"], pop["cv"])
            vals.append(ref.igd(front, fronts[name]) if len(front) else np.inf)
        out[f"{algo}/{name}/igd"] = np.array(vals)
        out[f"{algo}/{name}/cfg"] = np.array([n, gens])
    np.savez_compressed(os.path.join(HERE, "baseline_runs.npz"), **out)


WTA_LARGE = ("wta_P65.txt", "wta_custom40.txt", "wta_custom24.txt")


def wta_file_evaluate(path, X, nc):
    """The reference's load_wta + evaluate in a numpy-free subprocess
    (tests/golden/wta_file_eval.py says why)."""
    import subprocess
    import tempfile

    n, d = X.shape
    with tempfile.TemporaryDirectory() as tmp:
        xin, out = os.path.join(tmp, "x.f64"), os.path.join(tmp, "out.f64")
        np.ascontiguousarray(X, np.float64).tofile(xin)
        subprocess.run([sys.executable, os.path.join(HERE, "wta_file_eval.py"), path, xin, str(n), str(d), str(nc),
                        out], check=True)
        r = np.fromfile(out, np.float64)
    F = r[:2 * n].reshape(n, 2)
    G = r[2 * n:2 * n + n * nc].reshape(n, nc)
    return F, G, r[2 * n + n * nc:]


def wta_large_fixture(ref):
    """Large WTA scenarios in the reference's file
    format, evaluated by the reference's own load_wta + make_wta_problem:
    the synthetic P65 (35 vehicles, 277 slots), a 40-vehicle file with
    capacities up to 12 (> 256 slots: 64-bit decode keys) and a 24-vehicle
    file with <= 256 slots (narrow keys past the former 16-vehicle cap)."""
    sys.path.insert(0, ROOT)
    from paper_2509_19821_b200.wta import WTAInstance, save_wta, wta_synthetic

    rng = np.random.default_rng(64)
    insts = [wta_synthetic(65)]
    for name, nt, nv, cap_hi in (("custom40", 150, 40, 12), ("custom24", 60, 24, 9)):
        strikes = [int(v) for v in rng.integers(1, 4, nt)]
        if name == "custom24":  # at most 256 slots
            while sum(strikes) > 250:
                strikes[int(np.argmax(strikes))] -= 1
        p = [[float(v) for v in np.round(rng.uniform(0.3, 0.95, k), 6)] for k in strikes]
        cap = [int(v) for v in rng.integers(1, cap_hi + 1, nv)]
        insts.append(WTAInstance(name, nt, nv, strikes, p, cap))
    out = {}
    for inst, fname in zip(insts, WTA_LARGE):
        path = os.path.join(HERE, fname)
        save_wta(inst, path)
        d = inst.gene_count()
        X = f32(rng.random((24, d)))
        X[16:] = f32(np.round(X[16:] * 4) / 4)  # value ties across the decode order
        X[20:22] = f32(0.5 + 0.5 * rng.random((2, d)))  # every gene a candidate: capacity binds
        sparse = rng.random((2, d)) < 0.15 / inst.n_vehicles  # few candidates: feasible rows
        X[22:] = f32(np.where(sparse, 0.5 + 0.5 * rng.random((2, d)), 0.5 * rng.random((2, d))))
        nc = inst.n_vehicles + inst.n_targets
        F, G, cv = wta_file_evaluate(path, X, nc)
        key = fname[:-4]
        out[f"{key}/X"] = X.astype(np.float32)
        out[f"{key}/F"], out[f"{key}/G"], out[f"{key}/cv"] = F, G, cv
    np.savez_compressed(os.path.join(HERE, "wta_large.npz"), **out)


def many_obj_fixture(ref):
    """m > 3 operators: the reference's own
    reference_vectors + build_neighborhoods on m = 4..6 lattices, and
    metric_front / igd / hypervolume (the Monte-Carlo hv_mc branch,
    metrics.cpp:95-121) on random m = 4, 5 sets."""
    rng = np.random.default_rng(4567)
    out = {}
    for (m, n, t1, t2) in ((4, 120, 5, 20), (4, 300, 8, 30), (5, 210, 5, 20), (6, 462, 5, 20), (6, 100, 3, 10)):
        W = ref.reference_vectors(m, n)
        B1, B2 = ref.build_neighborhoods(W, t1, t2)
        key = f"lat_{m}_{n}_{t1}_{t2}"
        out[key + "/W"], out[key + "/B1"], out[key + "/B2"] = W, B1, B2
    for k in range(6):
        m = 4 + k % 2
        n = int(rng.integers(20, 300))
        F = f32(rng.random((n, m)))
        F[rng.random(n) < 0.1] = F[0]
        cv = np.where(rng.random(n) < 0.3, rng.random(n), 0.0)
        R = rng.random((40, m))
        key = f"met_{k}/"
        out[key + "F"], out[key + "cv"], out[key + "R"] = F, cv, R
        out[key + "front"] = ref.metric_front(F, cv)
        out[key + "igd"] = np.array(ref.igd(F, R))
        P = f32(rng.random((min(n, 60), m)) * 1.2)
        out[key + "P"] = P
        out[key + "hv"] = np.array(ref.hypervolume(P, np.full(m, 1.1)))
    np.savez_compressed(os.path.join(HERE, "many_obj.npz"), **out)


def main():
    if not build_ref():
        raise SystemExit("reference sources not available")
    ref, orc = Reference(), Oracle()
    if "--restated-fronts" in sys.argv:  # only the MW / DAS-CMOP front fixture
        restated_fronts_fixture(ref, orc)
        return
    if "--many-obj" in sys.argv:  # only the m > 3 operator fixture
        many_obj_fixture(ref)
        return
    if "--wta-large" in sys.argv:  # only the large WTA scenario fixture
        wta_large_fixture(ref)
        return
    rng = np.random.default_rng(20250919)
    eval_fixture(ref, orc, rng)
    selection_fixture(ref, orc, rng)
    knn_fixture(ref, rng)
    metrics_fixture(ref, rng)
    fronts_fixture(ref)
    pf_fixture(ref)
    restated_fronts_fixture(ref, orc)
    runs_fixture(ref)
    baseline_runs_fixture(ref)
    wta_large_fixture(ref)
    many_obj_fixture(ref)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
