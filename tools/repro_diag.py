"""Diagnostic: where do engine offspring genes differ from the f64 oracle's
by more than 1e-5 * span?  Prints the worst genes with their parents."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2509_19821_b200 as g  # noqa: E402
from oracle import Oracle  # noqa: E402

orc = Oracle()


def f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


for name, op in [("LIRCMOP13", 1), ("LIRCMOP1", 0), ("MW1", 0), ("MW7", 0), ("C1-DTLZ1", 0), ("WTA-P3", 0),
                 ("MW14", 1), ("DASCMOP7", 1), ("DASCMOP4", 0)]:
    info = orc.problem_info(name)
    n = 20000
    rng = np.random.default_rng(5)
    X = f32(info["lo"] + (info["hi"] - info["lo"]) * rng.random((n, info["d"])))
    # a share of genes sitting exactly at the bounds (as clipped parents do)
    mask = rng.random(X.shape) < 0.05
    X[mask] = np.where(rng.random(mask.sum()) < 0.5, info["lo"][np.nonzero(mask)[1]], info["hi"][np.nonzero(mask)[1]])
    nb = orc.knn(orc.reference_vectors(2, 2000), 20)
    nb = np.concatenate([nb + 2000 * k for k in range(n // 2000)]).astype(np.uint32)
    p = g.make_problem(name)
    span = info["hi"] - info["lo"]
    for gen in (1, 7):
        off = g.reproduce(g.Population(X, None, None, None), nb, p, op, seed=99, gen=gen, pop_id=2)
        want, picks = orc.reproduce(name, X, nb, op, 99, gen, 2)
        err = np.abs(off - want) / span
        bad = np.argwhere(err > 1e-5)
        print(f"{name} op={op} gen={gen}: max err/span {err.max():.3e}, genes > 1e-5: {len(bad)} of {err.size}",
              flush=True)
        for i, j in bad[np.argsort(-err[bad[:, 0], bad[:, 1]])][:6]:
            a, b, c = picks[i]
            pa, pb = nb[i, a], nb[i, b]
            print(f"   row {i} gene {j}: eng {off[i, j]:.9g} orc {want[i, j]:.9g} | x_i {X[i, j]:.9g} "
                  f"x_a {X[pa, j]:.9g} x_b {X[pb, j]:.9g} (pick3 {c})")
