"""The reference's experiment harness (proj/src/experiment.cpp, record.cpp)
driven by the B200 engine: the same JSON config schema, the same per-run JSONL
records, summary.jsonl and results.csv (Wilcoxon marks), and scaling_study —
so an existing experiment matrix switches to the engine by pointing at this
module.

Algorithms: "gmpea", "gmpea-s" (t1 = t2 = 5), "gmpea-l" (t1 = t2 = 20) on the
engine, and the reference's comparison baselines "cnsga2" and "ccmo"
(experiment.cpp:125-138) on the device operators of baselines.cuh.

IGD problems use the reference's own 1000-point pf_reference fronts
(data/fronts_1000.npz, generated from the unmodified reference); per-generation
IGD is recorded as the reference's hook does (experiment.cpp:200-205).
"""
from __future__ import annotations

import dataclasses
import json
import math
import os
import time
from typing import Dict, List, Optional

import numpy as np

from . import _lib as g

HERE = os.path.dirname(os.path.abspath(__file__))
ALGORITHMS = ("gmpea", "gmpea-s", "gmpea-l", "cnsga2", "ccmo")


@dataclasses.dataclass
class ExperimentConfig:
    """experiment.hpp:18-33."""

    algorithms: List[str]
    problems: List[str]
    seeds: List[int]
    eval_budget: Optional[int] = None
    time_budget_s: Optional[float] = None
    k_max: int = 0
    n: int = 100
    operators: Dict[str, str] = dataclasses.field(default_factory=dict)
    reference_algorithm: str = ""
    output_dir: str = "out"
    workers: int = 1
    record_walltime: bool = True
    igd_reference_points: int = 1000


def load_experiment_config(path: str) -> ExperimentConfig:
    """experiment.cpp:46-77."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise RuntimeError(f"cannot open config {path}")
    except ValueError as e:
        raise RuntimeError(f"config {path} is not valid JSON: {e}")
    b = j.get("budget", {})
    return ExperimentConfig(
        algorithms=list(j["algorithms"]), problems=list(j["problems"]), seeds=[int(s) for s in j["seeds"]],
        eval_budget=int(b["evals"]) if "evals" in b else None,
        time_budget_s=float(b["seconds"]) if "seconds" in b else None,
        k_max=int(j.get("k_max", 0)), n=int(j.get("n", 100)), operators=dict(j.get("operators", {})),
        reference_algorithm=j.get("reference_algorithm", ""), output_dir=j.get("output_dir", "out"),
        workers=int(j.get("workers", 1)), record_walltime=bool(j.get("record_walltime", True)),
        igd_reference_points=int(j.get("igd_reference_points", 1000)))


def validate_config(cfg: ExperimentConfig) -> None:
    """experiment.cpp:79-115: lists every error at once."""
    errors = []
    if not cfg.algorithms:
        errors.append("empty algorithm list")
    if not cfg.problems:
        errors.append("empty problem list")
    if not cfg.seeds:
        errors.append("empty seed list")
    if cfg.eval_budget is not None and cfg.time_budget_s is not None:
        errors.append("both evals and seconds budgets set; pick one")
    if cfg.eval_budget is None and cfg.time_budget_s is None and cfg.k_max == 0:
        errors.append("no budget configured (evals, seconds or k_max)")
    if cfg.eval_budget is not None and cfg.eval_budget == 0:
        errors.append("evals budget must be positive")
    if cfg.time_budget_s is not None and cfg.time_budget_s <= 0.0:
        errors.append("seconds budget must be positive")
    if cfg.n == 0:
        errors.append("population size must be positive")
    for a in cfg.algorithms:
        if a not in ALGORITHMS:
            errors.append("unknown algorithm: " + a)
    if cfg.reference_algorithm and cfg.reference_algorithm not in cfg.algorithms:
        errors.append("reference algorithm not in algorithm list: " + cfg.reference_algorithm)
    names = set(g.problem_names())
    for p in cfg.problems:
        if p not in names:
            errors.append("unknown problem: " + p)
    for suite, op in cfg.operators.items():
        if op not in ("sbx", "de"):
            errors.append(f"unknown operator '{op}' for suite {suite}")
    if cfg.igd_reference_points < 1:
        errors.append("igd_reference_points must be positive")
    if errors:
        raise ValueError("invalid experiment config:" + "".join("\n  - " + e for e in errors))


def suite_of(problem: str) -> str:
    if problem.startswith("LIRCMOP"):
        return "lircmop"
    if problem.startswith("WTA"):
        return "wta"
    if problem.startswith("MW"):
        return "mw"
    if problem.startswith("DASCMOP") or problem.startswith("DAS-CMOP"):
        return "dascmop"
    return "dtlz"


def operator_for(cfg: ExperimentConfig, problem: str) -> g.VariationOp:
    """experiment.cpp:117-123: DE for LIRCMOP, SBX elsewhere unless configured."""
    s = suite_of(problem)
    if s in cfg.operators:
        return g.VariationOp.de if cfg.operators[s] == "de" else g.VariationOp.sbx_pm
    return g.VariationOp.de if s == "lircmop" else g.VariationOp.sbx_pm


_FRONTS = None


def reference_front(problem: str, n_points: int = 1000) -> Optional[np.ndarray]:
    """pf_reference(p, n_points) (experiment.cpp:170-172), or None for the
    problems without an analytic front (HV problems).  1000 points: the
    unmodified reference's own front (data/fronts_1000.npz); other sizes are
    built on the device (gmpea_pf_reference, tests/test_gpu_parity.py)."""
    global _FRONTS
    if _FRONTS is None:
        _FRONTS = dict(np.load(os.path.join(HERE, "data", "fronts_1000.npz")))
    if n_points == 1000 or problem not in _FRONTS:
        return _FRONTS.get(problem)
    key = f"{problem}/{n_points}"
    if key not in _FRONTS:
        _FRONTS[key] = g.pf_reference(g.make_problem(problem), n_points)
    return _FRONTS[key]


def run_algorithm(algorithm: str, problem: g.Problem, cfg: g.RunConfig,
                  igd_front: Optional[np.ndarray] = None) -> g.RunResult:
    """experiment.cpp:125-138 on the engine; with igd_front the IGD hook runs
    on pop1 after every generation, outside the loop clock."""
    if algorithm not in ALGORITHMS:
        raise ValueError("unknown algorithm: " + algorithm)
    if algorithm in g.BASELINE_ALGORITHMS:
        return g.run_baseline(problem, algorithm, cfg, igd_front)
    c = dataclasses.replace(cfg)
    if algorithm == "gmpea-s":
        c.t1 = c.t2 = 5
    elif algorithm == "gmpea-l":
        c.t1 = c.t2 = 20
    # the IGD hook on the device (RunConfig.igd_reference), outside the loop clock
    c.igd_reference = igd_front
    return g.run_gmpea(problem, c)


def _num(v) -> str:
    """nlohmann::json dump of a double (shortest round trip, 0.0 keeps its point)."""
    return json.dumps(float(v))


def record_to_jsonl(history: List[g.GenRecord]) -> str:
    """record.cpp:15-31 (key order, +inf IGD as null)."""
    out = []
    for r in history:
        parts = [f'"gen":{int(r.gen)}', f'"evals":{int(r.evals)}', f'"wall_ms":{_num(r.wall_ms)}',
                 f'"feasible_ratio":{_num(r.feasible_ratio)}']
        if r.igd is not None:
            parts.append('"igd":' + (_num(r.igd) if math.isfinite(r.igd) else "null"))
        if r.hv is not None:
            parts.append(f'"hv":{_num(r.hv)}')
        out.append("{" + ",".join(parts) + "}\n")
    return "".join(out)


def parse_jsonl(text: str) -> List[g.GenRecord]:
    """record.cpp:33-61."""
    out = []
    for lineno, line in enumerate(text.splitlines(), 1):
        if not line:
            continue
        try:
            j = json.loads(line)
        except ValueError as e:
            raise RuntimeError(f"parse_jsonl: bad JSON on line {lineno}: {e}")
        igd = j.get("igd", None) if "igd" in j else None
        if "igd" in j and igd is None:
            igd = math.inf
        out.append(g.GenRecord(int(j["gen"]), int(j["evals"]), float(j["wall_ms"]), float(j["feasible_ratio"]),
                               igd, j.get("hv")))
    return out


def fmt(v: float) -> str:
    """experiment.cpp:31-37: setprecision(12)."""
    if math.isnan(v):
        return "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%.12g" % v


def wilcoxon_rank_sum(a, b, alpha=0.05):
    """metrics.cpp:216-255: two-sided rank-sum with tie correction; direction
    -1 when a's median is lower, +1 higher, 0 without a significant call."""
    n1, n2 = len(a), len(b)
    if n1 == 0 or n2 == 0:
        raise ValueError("wilcoxon_rank_sum: empty sample")
    allv = sorted([(v, 0) for v in a] + [(v, 1) for v in b])
    N = n1 + n2
    rank = [0.0] * N
    tie = 0.0
    i = 0
    while i < N:
        j = i
        while j < N and allv[j][0] == allv[i][0]:
            j += 1
        avg = 0.5 * (i + j - 1) + 1.0
        for k in range(i, j):
            rank[k] = avg
        t = float(j - i)
        tie += t * t * t - t
        i = j
    w = sum(rank[k] for k in range(N) if allv[k][1] == 0)
    mean = n1 * (N + 1.0) / 2.0
    var = n1 * n2 / 12.0 * (N + 1.0 - tie / (N * (N - 1.0)))
    if var <= 0.0:
        return 1.0, 0
    diff = w - mean
    cc = -0.5 if diff > 0.5 else (0.5 if diff < -0.5 else -diff)
    z = (diff + cc) / math.sqrt(var)
    p = 2.0 * (1.0 - 0.5 * math.erfc(-abs(z) / math.sqrt(2.0)))
    direction = 0
    if p < alpha:
        ma, mb = float(np.median(a)), float(np.median(b))
        direction = -1 if ma < mb else (1 if ma > mb else 0)
    return p, direction


def summaries_to_jsonl(summaries: List[dict]) -> str:
    """experiment.cpp:297-310."""
    out = []
    for s in summaries:
        v = s["value"]
        out.append('{"algorithm":%s,"problem":%s,"seed":%d,"metric":%s,"value":%s}\n' % (
            json.dumps(s["algorithm"]), json.dumps(s["problem"]), int(s["seed"]), json.dumps(s["metric"]),
            _num(v) if math.isfinite(v) else "null"))
    return "".join(out)


def load_summaries(path: str) -> List[dict]:
    out = []
    with open(path) as f:
        for line in f:
            if line.strip():
                j = json.loads(line)
                j["value"] = math.inf if j["value"] is None else float(j["value"])
                out.append(j)
    return out


def aggregate_results(cfg: ExperimentConfig, summaries: List[dict]) -> str:
    """experiment.cpp:333-370: mean/std per (algorithm, problem) + Wilcoxon
    mark against the reference algorithm ('+': the reference is better)."""
    ref_alg = cfg.reference_algorithm or cfg.algorithms[0]
    lines = ["algorithm,problem,metric,mean,std,mark"]
    for prob in cfg.problems:
        def samples(alg):
            s = [r for r in summaries if r["problem"] == prob and r["algorithm"] == alg]
            return [r["value"] for r in s], (s[-1]["metric"] if s else "")

        ref_s, metric = samples(ref_alg)
        for alg in cfg.algorithms:
            s, m = samples(alg)
            if not s:
                raise RuntimeError(f"aggregate_results: no runs for {alg}/{prob}")
            metric = m or metric
            mean = sum(s) / len(s)
            std = 0.0 if len(s) < 2 else math.sqrt(sum((x - mean) ** 2 for x in s) / (len(s) - 1))
            mark = ""
            if alg != ref_alg:
                _, d = wilcoxon_rank_sum(ref_s, s)
                better = -d if metric == "igd" else d
                mark = "+" if better > 0 else ("-" if better < 0 else "=")
            lines.append(f"{alg},{prob},{metric},{fmt(mean)},{fmt(std)},{mark}")
    return "\n".join(lines) + "\n"


@dataclasses.dataclass
class ExperimentResult:
    jsonl_paths: List[str]
    summary_path: str
    csv_path: str
    csv_text: str


def run_experiment(cfg: ExperimentConfig) -> ExperimentResult:
    """experiment.cpp:165-295 (cells run one at a time on the device)."""
    validate_config(cfg)
    os.makedirs(cfg.output_dir, exist_ok=True)
    problems = {p: g.make_problem(p) for p in cfg.problems}
    cells = [(a, p, s) for p in cfg.problems for a in cfg.algorithms for s in cfg.seeds]
    outcomes = {}
    for alg, prob, seed in cells:
        rc = g.RunConfig(n=cfg.n, k_max=cfg.k_max, eval_budget=cfg.eval_budget, time_budget_s=cfg.time_budget_s,
                         seed=seed, op=operator_for(cfg, prob), record_walltime=cfg.record_walltime)
        res = run_algorithm(alg, problems[prob], rc, reference_front(prob, cfg.igd_reference_points))
        outcomes[(alg, prob, seed)] = (res.history, g.metric_front(res.pop1))
    paths = []
    for alg, prob, seed in cells:
        path = os.path.join(cfg.output_dir, f"{alg}_{prob}_s{seed}.jsonl")
        with open(path, "w") as f:
            f.write(record_to_jsonl(outcomes[(alg, prob, seed)][0]))
        paths.append(path)
    summaries = []
    for prob in cfg.problems:
        front = reference_front(prob, cfg.igd_reference_points)
        ideal = nadir = None
        if front is None:  # normalised HV over all runs' fronts (experiment.cpp:245-265)
            m = problems[prob].m
            fronts = [outcomes[c][1] for c in cells if c[1] == prob]
            cat = np.concatenate([f for f in fronts if len(f)] or [np.zeros((0, m))])
            ideal = cat.min(0) if len(cat) else np.full(m, np.inf)
            nadir = cat.max(0) if len(cat) else np.full(m, -np.inf)
            for k in range(m):
                if not nadir[k] > ideal[k]:
                    if not math.isfinite(ideal[k]):
                        ideal[k] = 0.0
                    nadir[k] = ideal[k] + 1.0
        for alg, p, seed in cells:
            if p != prob:
                continue
            F = outcomes[(alg, p, seed)][1]
            if front is not None:
                value = g.igd(F, front) if len(F) else math.inf
            elif len(F) == 0:
                value = 0.0
            else:
                value = g.hypervolume((F - ideal) / (nadir - ideal), np.full(F.shape[1], 1.1))
            summaries.append({"algorithm": alg, "problem": prob, "seed": seed,
                              "metric": "igd" if front is not None else "hv", "value": value})
    summary_path = os.path.join(cfg.output_dir, "summary.jsonl")
    with open(summary_path, "w") as f:
        f.write(summaries_to_jsonl(summaries))
    csv = aggregate_results(cfg, summaries)
    csv_path = os.path.join(cfg.output_dir, "results.csv")
    with open(csv_path, "w") as f:
        f.write(csv)
    return ExperimentResult(paths, summary_path, csv_path, csv)


def scaling_study(algorithms: List[str], problem: str, sizes: List[int], generations: int, seed: int = 1) -> str:
    """experiment.cpp:372-404: mean per-generation loop time per size."""
    if not sizes or sizes != sorted(sizes):
        raise ValueError("scaling_study: sizes must be ascending")
    if generations == 0:
        raise ValueError("scaling_study: need at least one generation")
    for a in algorithms:
        if a not in ALGORITHMS:
            raise ValueError("scaling_study: unknown algorithm " + a)
    p = g.make_problem(problem)
    lines = ["algorithm,n,mean_gen_ms,ratio"]
    for alg in algorithms:
        base = 0.0
        for i, n in enumerate(sizes):
            r = run_algorithm(alg, p, g.RunConfig(n=n, k_max=generations, seed=seed, record_walltime=True))
            per_gen = r.history[-1].wall_ms / (len(r.history) - 1)
            if i == 0:
                base = per_gen
            lines.append(f"{alg},{n},{fmt(per_gen)},{fmt(per_gen / base)}")
    return "\n".join(lines) + "\n"


def main(argv=None):
    """A minimal `gmpea_cli run|scale|aggregate` (tools/gmpea_cli.cpp:36-126)."""
    import argparse

    ap = argparse.ArgumentParser(prog="python -m paper_2509_19821_b200.experiment")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("-c", "--config", required=True)
    a = sub.add_parser("aggregate")
    a.add_argument("-c", "--config", required=True)
    s = sub.add_parser("scale")
    s.add_argument("--problem", required=True)
    s.add_argument("--algorithms", nargs="+", default=["gmpea"])
    s.add_argument("--sizes", nargs="+", type=int, required=True)
    s.add_argument("--generations", type=int, default=3)
    s.add_argument("--seed", type=int, default=1)
    args = ap.parse_args(argv)
    if args.cmd == "run":
        res = run_experiment(load_experiment_config(args.config))
        print(res.csv_text, end="")
    elif args.cmd == "aggregate":
        cfg = load_experiment_config(args.config)
        csv = aggregate_results(cfg, load_summaries(os.path.join(cfg.output_dir, "summary.jsonl")))
        with open(os.path.join(cfg.output_dir, "results.csv"), "w") as f:
            f.write(csv)
        print(csv, end="")
    else:
        print(scaling_study(args.algorithms, args.problem, args.sizes, args.generations, args.seed), end="")


if __name__ == "__main__":
    main()
