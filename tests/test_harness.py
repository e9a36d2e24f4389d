"""The experiment-harness mirror (paper_2509_19821_b200/experiment.py) and the
WTA scenario module (wta.py) against the reference's formats and tests
(tests/test_experiment.cpp, test_metrics.cpp:197-227, test_wta.cpp)."""
import json
import math
import os

import numpy as np
import pytest


def test_validate_config_lists_every_error(g):
    from paper_2509_19821_b200.experiment import ExperimentConfig, validate_config

    cfg = ExperimentConfig(algorithms=["gmpea", "moead"], problems=["LIRCMOP1", "NOPE"], seeds=[1],
                           eval_budget=100, time_budget_s=1.0, n=0, operators={"lircmop": "ga"})
    with pytest.raises(ValueError) as e:
        validate_config(cfg)
    msg = str(e.value)
    assert msg.startswith("invalid experiment config:")
    for part in ("both evals and seconds budgets set", "population size must be positive",
                 "unknown algorithm: moead", "unknown problem: NOPE", "unknown operator 'ga' for suite lircmop"):
        assert part in msg


def test_records_jsonl_format_roundtrip(g):
    from paper_2509_19821_b200.experiment import parse_jsonl, record_to_jsonl

    h = [g.GenRecord(0, 40, 0.0, 0.25, math.inf, None), g.GenRecord(1, 80, 1.5, 0.5, 0.125, 3.0)]
    txt = record_to_jsonl(h)
    assert txt.splitlines()[0] == '{"gen":0,"evals":40,"wall_ms":0.0,"feasible_ratio":0.25,"igd":null}'
    assert txt.splitlines()[1] == '{"gen":1,"evals":80,"wall_ms":1.5,"feasible_ratio":0.5,"igd":0.125,"hv":3.0}'
    back = parse_jsonl(txt)
    assert back[0].igd == math.inf and back[1].hv == 3.0 and back[1].evals == 80


def test_wilcoxon_reference_behaviour(g):
    from paper_2509_19821_b200.experiment import wilcoxon_rank_sum

    a = list(range(1, 21))
    b = list(range(101, 121))
    p, d = wilcoxon_rank_sum(a, b)
    assert p < 0.05 and d == -1
    p2, d2 = wilcoxon_rank_sum(b, a)
    assert abs(p2 - p) <= 1e-12 * p and d2 == 1
    assert wilcoxon_rank_sum(a, a)[1] == 0 and wilcoxon_rank_sum(a, a)[0] >= 0.05
    assert wilcoxon_rank_sum(a, a[::-1])[1] == 0
    assert wilcoxon_rank_sum([1.0] * 10, [1.0] * 10)[1] == 0
    assert wilcoxon_rank_sum([1.0] * 10, [1.001] + [1.0] * 9)[1] == 0


def test_wilcoxon_matches_reference_binary(g, ref):
    """Same statistic as the reference's metrics.cpp:216-255, bit for bit."""
    from paper_2509_19821_b200.experiment import wilcoxon_rank_sum

    rng = np.random.default_rng(3)
    for _ in range(50):
        a = np.round(rng.normal(0, 1, int(rng.integers(3, 31))), 1)
        b = np.round(rng.normal(0.4, 1, int(rng.integers(3, 31))), 1)
        assert wilcoxon_rank_sum(list(a), list(b)) == ref.wilcoxon(a, b)


def test_wta_scenarios_match_reference(g, orc):
    from paper_2509_19821_b200.wta import wta_scenario

    for num in range(1, 11):
        inst = wta_scenario(f"P{num}")
        want = orc.wta_scenario(num)
        assert inst.n_targets == want["targets"] and inst.n_vehicles == want["vehicles"]
        assert inst.max_strikes == want["strikes"].tolist() and inst.capacity == want["capacity"].tolist()
        assert [v for row in inst.p for v in row] == want["p"].tolist()
    with pytest.raises(ValueError):
        wta_scenario("P11")
    with pytest.raises(ValueError):
        wta_scenario("Q1")


def test_wta_files_roundtrip(tmp_path, g):
    from paper_2509_19821_b200.wta import load_wta, save_wta, wta_scenario

    inst = wta_scenario("P4")
    path = str(tmp_path / "p4.txt")
    save_wta(inst, path)
    back = load_wta(path)
    assert back == inst
    assert inst.gene_index(1, 0, 0) == inst.max_strikes[0] * inst.n_vehicles
    with open(path, "a") as f:
        f.write("bogus 1\n")
    with pytest.raises(RuntimeError, match="unknown key 'bogus'"):
        load_wta(path)


@pytest.mark.gpu
def test_wta_hand_examples(g):
    """test_wta.cpp:58-93,102-125,169-184 through the engine."""
    from paper_2509_19821_b200.wta import WTAInstance, make_wta_problem

    tiny = make_wta_problem(WTAInstance("T1", 1, 1, [1], [[0.8]], [1]))
    r = g.evaluate(tiny, np.array([[0.9], [0.1]]))
    assert np.allclose(r.F[0], [-0.8, 1.0]) and np.allclose(r.G[0], [0.0, 0.0])
    assert np.allclose(r.F[1], [0.0, 0.0]) and np.allclose(r.G[1], [-1.0, -1.0])
    two = make_wta_problem(WTAInstance("T2", 2, 1, [1, 1], [[0.5], [0.5]], [2]))
    assert np.allclose(g.evaluate(two, np.array([[0.9, 0.9]])).F[0], [-1.0, 2.0])
    cap1 = make_wta_problem(WTAInstance("T3", 1, 1, [3], [[0.5, 0.5, 0.5]], [1]))
    # decode: one strike survives (the highest gene; ties to the lower index)
    for genes in ([0.0, 0.2, 0.49], [0.6, 0.9, 0.7], [0.8, 0.8, 0.8]):
        want_hits = 0 if max(genes) < 0.5 else 1
        assert g.evaluate(cap1, np.array([genes])).F[0, 1] == want_hits


@pytest.mark.gpu
def test_run_experiment_end_to_end(tmp_path, g):
    from paper_2509_19821_b200.experiment import ExperimentConfig, load_summaries, run_experiment

    out = str(tmp_path / "exp")
    cfg = ExperimentConfig(algorithms=["gmpea", "gmpea-s"], problems=["LIRCMOP1", "WTA-P1"], seeds=[1, 2, 3],
                           k_max=8, n=30, output_dir=out, record_walltime=False)
    res = run_experiment(cfg)
    assert len(res.jsonl_paths) == 12
    lines = open(os.path.join(out, "gmpea_LIRCMOP1_s1.jsonl")).read().splitlines()
    assert len(lines) == 9 and json.loads(lines[-1])["evals"] == 2 * 30 * 9 and "igd" in json.loads(lines[0])
    assert "igd" not in open(os.path.join(out, "gmpea_WTA-P1_s1.jsonl")).readline()
    s = load_summaries(res.summary_path)
    assert {x["metric"] for x in s} == {"igd", "hv"} and len(s) == 12
    csv = res.csv_text.splitlines()
    assert csv[0] == "algorithm,problem,metric,mean,std,mark" and len(csv) == 5
    assert csv[1].startswith("gmpea,LIRCMOP1,igd,") and csv[1].endswith(",")
    assert csv[2].split(",")[-1] in "+-="
    # byte-identical reruns (record_walltime false)
    again = run_experiment(cfg)
    assert again.csv_text == res.csv_text


@pytest.mark.gpu
def test_run_experiment_custom_reference_points(tmp_path, g):
    """igd_reference_points != 1000: the IGD front comes from the device
    pf_reference (experiment.cpp:170-172 semantics)."""
    from paper_2509_19821_b200.experiment import ExperimentConfig, load_summaries, reference_front, run_experiment

    front = reference_front("LIRCMOP13", 200)
    assert front.shape == (200, 3)
    cfg = ExperimentConfig(algorithms=["gmpea"], problems=["LIRCMOP13"], seeds=[1], k_max=5, n=105,
                           output_dir=str(tmp_path / "exp"), record_walltime=False, igd_reference_points=200)
    res = run_experiment(cfg)
    s = load_summaries(res.summary_path)
    assert len(s) == 1 and s[0]["metric"] == "igd" and s[0]["value"] > 0


@pytest.mark.gpu
def test_run_experiment_with_baselines(tmp_path, g):
    """cnsga2 / ccmo run through the same harness (experiment.cpp:125-128):
    JSONL records with the IGD hook, Wilcoxon marks against gmpea."""
    from paper_2509_19821_b200.experiment import ExperimentConfig, load_summaries, run_experiment

    cfg = ExperimentConfig(algorithms=["gmpea", "cnsga2", "ccmo"], problems=["LIRCMOP1"], seeds=[1, 2, 3], k_max=6,
                           n=30, output_dir=str(tmp_path / "exp"), record_walltime=False)
    res = run_experiment(cfg)
    lines = open(os.path.join(cfg.output_dir, "ccmo_LIRCMOP1_s1.jsonl")).read().splitlines()
    assert len(lines) == 7 and json.loads(lines[-1])["evals"] == 2 * 30 * 7 and "igd" in json.loads(lines[-1])
    lines = open(os.path.join(cfg.output_dir, "cnsga2_LIRCMOP1_s1.jsonl")).read().splitlines()
    assert json.loads(lines[-1])["evals"] == 30 * 7
    assert {x["algorithm"] for x in load_summaries(res.summary_path)} == {"gmpea", "cnsga2", "ccmo"}
    assert len(res.csv_text.splitlines()) == 4
