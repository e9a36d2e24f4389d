"""BASELINE.json configs[1]: MW1-MW14 (and DAS-CMOP1-9), N = 10,000, 30 seeds —
final-population quality of the engine vs the reference's own run_gmpea on the
same problems.

The reference has no MW problems, so its loop runs the oracle's
restated MW evaluators wrapped as reference ProblemDefs (oracle/ref_shim.cpp,
problem_for) — "reference loop + restated evaluator".  Neither side has an
analytic MW front, so the metric is the reference harness's normalised
hypervolume (experiment.cpp:240-281: ideal/nadir over the runs' fronts,
reference point 1.1): here the bounds come from the reference runs and are
applied to both arms.  Since the restated fronts exist
(tests/golden/pf_restated.npz, the reference's pf_reference over the restated
candidates), the final IGD against them is compared as well.

    python tools/mw_parity.py ref   [--seeds 30 --n 10000 --gens 200 --procs 8]
        runs the reference here (CPU) -> tests/golden/mw_ref_hv.json
    python tools/mw_parity.py gpu   -> profiles/r01_mw_parity.json (needs a B200)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
REF_JSON = os.path.join(ROOT, "tests", "golden", "mw_ref_hv.json")
PROBLEMS = [f"MW{i}" for i in range(1, 15)]


def _ref_run(job):
    name, n, gens, seed = job
    from oracle import Reference

    r = Reference()
    pop, _ = r.run_gmpea(name, n, k_max=gens, seed=seed, op=suite_op(name), record_walltime=False)
    return name, seed, r.metric_front(pop["F"], pop["cv"])


def hv_of(front, lo, hi, hv_fn):
    if len(front) == 0:
        return 0.0
    span = np.where(hi > lo, hi - lo, 1.0)
    return float(hv_fn((front - lo) / span, np.full(front.shape[1], 1.1)))


def restated_front(name):
    """IGD reference front: the reference's own pf_reference (fronts.npz) for
    its suites, the restated fronts (pf_restated.npz) for MW / DAS-CMOP."""
    ref = np.load(os.path.join(ROOT, "tests", "golden", "fronts.npz"))
    if name in ref.files:
        return ref[name]
    fx = np.load(os.path.join(ROOT, "tests", "golden", "pf_restated.npz"))
    return fx[f"{name}/1000"]


def suite_op(name):
    return 1 if name.startswith("LIRCMOP") else 0  # experiment.cpp:117-123


def igd_of(front, ref_front, igd_fn):
    return float(igd_fn(front, ref_front)) if len(front) else float("inf")


def cmd_ref(args):
    from oracle import Reference

    probs = args.problems.split(",") if args.problems else PROBLEMS
    jobs = [(p, args.n, args.gens, s) for p in probs for s in range(1, args.seeds + 1)]
    fronts = {}
    with ProcessPoolExecutor(args.procs) as ex:
        for name, seed, fr in ex.map(_ref_run, jobs):
            fronts.setdefault(name, {})[seed] = fr
            print(name, seed, len(fr), flush=True)
    ref = Reference()
    out = {"n": args.n, "gens": args.gens, "seeds": args.seeds, "problems": {}}
    for name in probs:
        allf = [f for f in fronts[name].values() if len(f)]
        if not allf:
            out["problems"][name] = {"ideal": None, "nadir": None, "hv": [0.0] * args.seeds,
                                     "igd": [float("inf")] * args.seeds}
            continue
        cat = np.concatenate(allf)
        lo, hi = cat.min(0), cat.max(0)
        hvs = [hv_of(fronts[name][s], lo, hi, ref.hypervolume) for s in range(1, args.seeds + 1)]
        pf = restated_front(name)
        igds = [igd_of(fronts[name][s], pf, ref.igd) for s in range(1, args.seeds + 1)]
        out["problems"][name] = {"ideal": lo.tolist(), "nadir": hi.tolist(), "hv": hvs, "igd": igds}
    with open(args.ref_json, "w") as f:
        json.dump(out, f, indent=1)


def cmd_gpu(args):
    from scipy.stats import mannwhitneyu

    import paper_2509_19821_b200 as g

    ref = json.load(open(args.ref_json))
    res = {}
    for name in ref["problems"]:
        rp = ref["problems"][name]
        p = g.make_problem(name)
        hvs, igds = [], []
        pf = restated_front(name)
        for seed in range(1, ref["seeds"] + 1):
            r = g.run_gmpea(p, g.RunConfig(n=ref["n"], k_max=ref["gens"], seed=seed,
                                           op=g.VariationOp(suite_op(name))))
            fr = g.metric_front(r.pop1)
            if rp["ideal"] is None:
                hvs.append(0.0)
            else:
                hvs.append(hv_of(fr, np.array(rp["ideal"]), np.array(rp["nadir"]), g.hypervolume))
            igds.append(igd_of(fr, pf, g.igd))

        def compare(a, b, higher_better):
            a, b = np.asarray(a, float), np.asarray(b, float)
            if np.array_equal(np.unique(a), np.unique(b)) and len(np.unique(a)) == 1:
                return 1.0, "="
            # infinite IGD (no feasible point) ranks last: map it to a large finite value
            fin = np.concatenate([a, b])[np.isfinite(np.concatenate([a, b]))]
            big = (fin.max() * 10 + 1) if len(fin) else 1.0
            a2, b2 = np.where(np.isfinite(a), a, big), np.where(np.isfinite(b), b, big)
            pv = float(mannwhitneyu(a2, b2, alternative="two-sided").pvalue)
            better = np.median(a2) > np.median(b2) if higher_better else np.median(a2) < np.median(b2)
            return pv, "=" if pv >= 0.05 else ("+" if better else "-")

        pval, verdict = compare(hvs, rp["hv"], True)
        res[name] = {"b200_median_hv": float(np.median(hvs)), "ref_median_hv": float(np.median(rp["hv"])),
                     "p_value": pval, "verdict": verdict,
                     "b200_feasible_runs": int((np.array(hvs) > 0).sum()),
                     "ref_feasible_runs": int((np.array(rp["hv"]) > 0).sum()),
                     "b200_hv": [float(x) for x in hvs]}
        if "igd" in rp:
            pi, vi = compare(igds, rp["igd"], False)
            res[name].update({"b200_median_igd": float(np.median(igds)), "ref_median_igd": float(np.median(rp["igd"])),
                              "igd_p_value": pi, "igd_verdict": vi, "b200_igd": igds})
        print(name, res[name], flush=True)
    with open(args.out, "w") as f:
        json.dump({"config": {k: ref[k] for k in ("n", "gens", "seeds")}, "results": res}, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["ref", "gpu"])
    ap.add_argument("--seeds", type=int, default=30)
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--gens", type=int, default=200)
    ap.add_argument("--procs", type=int, default=6)
    ap.add_argument("--problems", default="")
    ap.add_argument("--ref-json", default=REF_JSON)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_mw_parity.json"))
    args = ap.parse_args()
    cmd_ref(args) if args.cmd == "ref" else cmd_gpu(args)


if __name__ == "__main__":
    main()
