"""Root cause of the LIRCMOP1 statistics: where does the
engine's final-quality shift against the reference come from?

Four arms, 90 seeds each, LIRCMOP1 at N = 10^4, 100 generations, DE (the suite
default), every final front scored by the same IGD (the reference's own
pf_reference front, tests/golden/fronts.npz) and normalised HV (the bounds of
the reference runs, tests/golden/lircmop1_90seeds_ref.json):

  reference   the reference's own run_gmpea (mt19937_64 stream, f64)    [golden]
  b200        the engine (Philox draws, fp32 state)                     [r01 profile]
  philox-f64  the oracle's loop with the engine's Philox draws, all f64
  philox-f32  the same with the state rounded to fp32 after every step

philox-f64 vs reference isolates the draw schema; philox-f32 vs philox-f64
isolates fp32 storage; b200 vs philox-f32 what remains (fp32 arithmetic).

    python tools/lircmop1_arms.py [--procs 8] -> profiles/r02_lircmop1_arms.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def _run(job):
    from oracle import Oracle

    seed, fp32, n, gens = job
    o = Oracle()
    _, F, cv = o.run_gmpea("LIRCMOP1", n, gens, seed=seed, op=1, fp32=fp32)
    idx = o.metric_front(F, cv)
    return seed, fp32, F[idx]


def _run_ref(job):
    """the reference's own run_gmpea (mt19937_64, f64), another batch of seeds"""
    from oracle import Reference

    seed, n, gens = job
    r = Reference()
    pop, _ = r.run_gmpea("LIRCMOP1", n, k_max=gens, seed=seed, op=1, record_walltime=False)
    return seed, r.metric_front(pop["F"], pop["cv"])


def main():
    from scipy.stats import mannwhitneyu
    from oracle import Oracle

    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--seeds", type=int, default=90)
    ap.add_argument("--noise", action="store_true",
                    help="also a second batch of seeds (91-180) of the reference and philox-f64 arms: how far two "
                         "batches of the SAME arm drift apart")
    args = ap.parse_args()
    refj = json.load(open(os.path.join(ROOT, "tests", "golden", "lircmop1_90seeds_ref.json")))
    n, gens = refj["n"], refj["gens"]
    rp = refj["problems"]["LIRCMOP1"]
    lo, hi = np.array(rp["ideal"]), np.array(rp["nadir"])
    front = np.load(os.path.join(ROOT, "tests", "golden", "fronts.npz"))["LIRCMOP1"]
    eng = json.load(open(os.path.join(ROOT, "profiles", "r01_lircmop1_90seeds_parity.json")))["results"]["LIRCMOP1"]
    o = Oracle()
    span = np.where(hi > lo, hi - lo, 1.0)

    def score(fr):
        if len(fr) == 0:
            return np.inf, 0.0
        return o.igd(fr, front), o.hypervolume((fr - lo) / span, np.full(fr.shape[1], 1.1))

    jobs = [(s, fp32, n, gens) for s in range(1, args.seeds + 1) for fp32 in (False, True)]
    arms = {"philox-f64": {}, "philox-f32": {}}
    with ProcessPoolExecutor(args.procs) as ex:
        for seed, fp32, fr in ex.map(_run, jobs):
            arms["philox-f32" if fp32 else "philox-f64"][seed] = score(fr)
    res = {"config": {"problem": "LIRCMOP1", "n": n, "gens": gens, "seeds": args.seeds, "op": "de"},
           "arms": {"reference": {"igd": rp["igd"], "hv": rp["hv"]},
                    "b200": {"igd": eng["b200_igd"], "hv": eng["b200_hv"]}}}
    for k, v in arms.items():
        res["arms"][k] = {"igd": [v[s][0] for s in sorted(v)], "hv": [v[s][1] for s in sorted(v)]}
    pairs = [("philox-f64", "reference"), ("philox-f32", "philox-f64"), ("b200", "philox-f32"),
             ("b200", "reference"), ("philox-f32", "reference")]
    if args.noise:
        s2 = range(args.seeds + 1, 2 * args.seeds + 1)
        with ProcessPoolExecutor(args.procs) as ex:
            ref2 = {sd: score(fr) for sd, fr in ex.map(_run_ref, [(sd, n, gens) for sd in s2])}
            ph2 = {sd: score(fr) for sd, _, fr in ex.map(_run, [(sd, False, n, gens) for sd in s2])}
        res["arms"]["reference-b2"] = {"igd": [ref2[k][0] for k in sorted(ref2)], "hv": [ref2[k][1] for k in sorted(ref2)]}
        res["arms"]["philox-f64-b2"] = {"igd": [ph2[k][0] for k in sorted(ph2)], "hv": [ph2[k][1] for k in sorted(ph2)]}
        pairs += [("reference-b2", "reference"), ("philox-f64-b2", "philox-f64"), ("philox-f64-b2", "reference-b2")]
    res["median"] = {k: {"igd": float(np.median(a["igd"])), "hv": float(np.median(a["hv"]))}
                     for k, a in res["arms"].items()}
    res["mann_whitney_p"] = {f"{a} vs {b}": {m: float(mannwhitneyu(res["arms"][a][m], res["arms"][b][m],
                                                                    alternative="two-sided").pvalue)
                                             for m in ("igd", "hv")} for a, b in pairs}
    out = os.path.join(ROOT, "profiles", "r02_lircmop1_arms.json")
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({"median": res["median"], "p": res["mann_whitney_p"]}, indent=1))


if __name__ == "__main__":
    main()
