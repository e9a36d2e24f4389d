"""One engine generation against the oracle's operator chain, with every
disagreement proved to be a tie (north_star: values within 1e-5 relative;
selection and replacement indices bit-exact wherever the deciding keys are
not tied within that tolerance).

The chain of run_gmpea's loop body (proj/src/gmpea.cpp:463-478):

  (a) reproduce     engine offspring X  vs  oracle reproduce (f64, the same
                    Philox draws) on the engine's parent rows
  (b) evaluate      engine offspring F, C, cv  vs  oracle evaluate of the
                    engine's offspring rows
  (c) update_ideal  engine z  ==  min(z0, offspring F)  (fp32 min, exact)
  (d) selection     engine survivors  vs  oracle OP1/OP2/OP3 (f64) on the
                    engine's own keys; each slot whose survivor differs must
                    be a tie: the two survivors' keys at that slot tie within
                    1e-5 (lexicographically (cv, g) for pop1: FPR, gmpea.cpp:296;
                    g for pop2), or the difference cascades from an OP1 tie of
                    one of the slot's claimants (gmpea.cpp:248-279).

Test infrastructure only (imports the oracle).
"""
from __future__ import annotations

import numpy as np

TOL = 1e-5


def close(a, b, tol=TOL):
    return abs(a - b) <= tol * max(1.0, abs(b))


def agg_keys(F, W, z, theta, agg):
    """PBI (scalarize.cpp:72-89) or Tchebycheff of rows F at weights W, f64."""
    F, W = np.atleast_2d(F), np.atleast_2d(W)
    D = F - z
    if agg == 1:
        return (np.maximum(W, 1e-6) * np.abs(D)).max(1)
    wn = np.sqrt((W * W).sum(1))
    d1 = np.abs((D * W).sum(1)) / wn
    R = D - d1[:, None] * (W / wn[:, None])
    return d1 + theta * np.sqrt((R * R).sum(1))


def reverse_lists(B):
    """claimants c of slot j (j in B[c]), ascending, as CSR (start, ids)."""
    n, t = B.shape
    j = B.reshape(-1).astype(np.int64)
    c = np.repeat(np.arange(n, dtype=np.int64), t)
    order = np.lexsort((c, j))
    start = np.searchsorted(j[order], np.arange(n + 1))
    return start, c[order]


def keys_tie(cva, ga, cvb, gb, lex):
    if not lex:
        return close(ga, gb)
    # FPR: cv first; a within-tolerance cv difference decides either way
    if not close(cva, cvb):
        return False
    return cva != cvb or close(ga, gb)


def check_generation(g, orc, name, op, n, seed=5, agg=0, theta=5.0, gene_tol=TOL, log=None, problem=None):
    """Runs one generation and checks (a)-(d); returns a summary dict.
    problem: an engine problem object for `name` (custom scenarios)."""
    p = problem if problem is not None else g.make_problem(name)
    eng = g.Engine(p, g.RunConfig(n=n, k_max=1, seed=seed, op=g.VariationOp(op), aggregation=agg,
                                  record_walltime=False))
    P = [eng.population(1), eng.population(2)]
    topo = eng.neighborhoods()
    B = [topo.b1, topo.b2]
    z0 = eng.ideal()
    eng.run()
    N = [eng.population(1), eng.population(2)]
    O = [eng.offspring(1), eng.offspring(2)]
    z = eng.ideal()
    rr = eng.replacement_rates()
    eng.close()
    info = orc.problem_info(name)
    span = info["hi"] - info["lo"]
    out = {"name": name, "n": n, "op": op}
    # (a) variation, draw for draw
    worst = 0.0
    for q in range(2):
        want, _ = orc.reproduce(name, P[q].X, B[q], op, seed, 1, q + 1)
        err = np.abs(O[q].X - want) / span
        worst = max(worst, float(err.max()))
        assert err.max() <= gene_tol, (name, q, float(err.max()), np.unravel_index(err.argmax(), err.shape))
    out["gene_err_max"] = worst
    # (b) evaluation of the engine's own offspring rows
    for q in range(2):
        F, G, cv = orc.evaluate(name, O[q].X)
        for a, b, what in ((O[q].F, F, "F"), (O[q].C, G, "C"), (O[q].cv, cv, "cv")):
            bad = np.abs(a - b) > TOL * np.maximum(1.0, np.abs(b))
            assert not bad.any(), (name, q, what, int(bad.sum()), float(np.abs(a - b).max()))
    # (c) ideal point
    zexp = np.minimum(z0, np.minimum(O[0].F.min(0), O[1].F.min(0)))
    assert np.array_equal(z, zexp), (z, zexp)
    # (d) selection on the engine's keys
    m = p.m
    W = orc.reference_vectors(m, n)
    keys = [dict(F=x.F, cv=x.cv) for x in (P[0], P[1], O[0], O[1])]
    src = orc.selection(keys, W, z, theta, B[0], B[1], agg=agg)
    g_off = [agg_keys(O[k].F, W, z, theta, agg) for k in range(2)]  # offspring keys at their own slot
    ties = {"op3": 0, "op1": 0, "op3_gap_max": 0.0}
    for q in range(2):
        s = src[q]
        kept = s < 0
        c = np.where(kept, 0, s % n)
        from_o2 = s >= n
        exp = {}
        for key in ("X", "F", "C", "cv"):
            par = getattr(P[q], key)
            o1, o2 = getattr(O[0], key), getattr(O[1], key)
            cand = np.where((from_o2.reshape(-1, *([1] * (par.ndim - 1)))), o2[c], o1[c])
            exp[key] = np.where(kept.reshape(-1, *([1] * (par.ndim - 1))), par, cand)
        same = np.ones(n, bool)
        for key in ("X", "F", "C", "cv"):
            a, b = getattr(N[q], key), exp[key]
            same &= (a == b).reshape(n, -1).all(1) if a.ndim > 1 else (a == b)
        bad = np.nonzero(~same)[0]
        if len(bad) == 0:
            continue
        start, ids = reverse_lists(B[q])
        for j in bad:
            cl = ids[start[j]:start[j + 1]]
            # the engine's survivor: the first candidate whose row it holds
            cands = [(-1, P[q])] + [(int(cc), O[0]) for cc in cl] + [(n + int(cc), O[1]) for cc in cl]
            ecode = None
            for code, pop in cands:
                r = j if code < 0 else code % n
                if np.array_equal(pop.X[r], N[q].X[j]) and pop.cv[r] == N[q].cv[j] and \
                        np.array_equal(pop.F[r], N[q].F[j]):
                    ecode = code
                    break
            assert ecode is not None, (name, q, j, "survivor is no candidate of the slot")

            def key_of(code):
                pop = P[q] if code < 0 else O[code // n]
                r = j if code < 0 else code % n
                return float(pop.cv[r]), float(agg_keys(pop.F[r], W[j], z, theta, agg)[0])

            ca, ga = key_of(ecode)
            cb, gb = key_of(int(s[j]))
            if keys_tie(ca, ga, cb, gb, q == 0):
                ties["op3"] += 1
                ties["op3_gap_max"] = max(ties["op3_gap_max"], abs(ga - gb) / max(1.0, abs(gb)))
                continue
            # cascade from an OP1 tie of a claimant (or of the survivors' own slots)
            slots = set(int(x) for x in cl)
            op1_tie = False
            for cc in slots:
                c1, c2 = float(O[0].cv[cc]), float(O[1].cv[cc])
                g1, g2 = float(g_off[0][cc]), float(g_off[1][cc])
                if keys_tie(c1, g1, c2, g2, True) or close(g1, g2):
                    op1_tie = True
                    break
            assert op1_tie, (name, q, j, ecode, int(s[j]), (ca, ga), (cb, gb))
            ties["op1"] += 1
    out.update(ties)
    out["replaced"] = int((src[0] >= 0).sum() + (src[1] >= 0).sum())
    # the engine's replacement diagnostic counts the same winners (up to ties)
    n_eng = int(round(rr[1] * 2 * n))
    assert abs(n_eng - out["replaced"]) <= ties["op3"] + ties["op1"], (n_eng, out)
    out["engine_replaced"] = n_eng
    if log is not None:
        log.append(out)
    return out
