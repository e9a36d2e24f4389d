"""GPU: the weight-region shard path (sharded engine + halo plan) on one
device — `world` shards in lockstep with device copies standing in for NCCL —
equals the unsharded engine bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n,world,op", [("LIRCMOP13", 6000, 4, 1), ("MW1", 4000, 3, 0), ("LIRCMOP1", 2000, 2, 1)])
def test_local_shards_equal_unsharded(g, name, n, world, op):
    from paper_2509_19821_b200.sharded import run_local_group

    gens = 6
    p = g.make_problem(name)
    cfg = g.RunConfig(n=n, k_max=gens, seed=5, op=op)
    pops, shards = run_local_group(p, cfg, world, gens)
    ref = g.run_gmpea(p, cfg)
    X = np.concatenate([q.X for q in pops])
    F = np.concatenate([q.F for q in pops])
    cv = np.concatenate([q.cv for q in pops])
    assert X.shape == ref.pop1.X.shape
    assert np.array_equal(X, ref.pop1.X) and np.array_equal(F, ref.pop1.F) and np.array_equal(cv, ref.pop1.cv)
    info = shards[1].eng.shard_info()
    assert info["reach"] > 0 and info["window_end"] - info["window_begin"] > info["own_end"] - info["own_begin"]


def test_shard_narrower_than_reach_is_rejected(g):
    p = g.make_problem("LIRCMOP13")
    with pytest.raises(ValueError, match="narrower than twice the neighbourhood reach"):
        g.Engine(p, g.RunConfig(n=1000, k_max=1, shard=(0, 100)))


# ---------------------------------------------- the engine's own shard exchange
def _pop_equal(a, b):
    return np.array_equal(a.X, b.X) and np.array_equal(a.F, b.F) and np.array_equal(a.cv, b.cv) and \
        np.array_equal(a.C, b.C)


@pytest.mark.parametrize("name,n,shards,op", [("LIRCMOP13", 6000, 4, 1), ("MW1", 4000, 3, 0), ("LIRCMOP1", 2000, 2, 1),
                                              ("WTA-P3", 900, 2, 0)])
def test_multi_device_handle_equals_unsharded(g, name, n, shards, op):
    """gmpea_engine_create_multi with every shard on device 0: one
    multi-device CUDA graph per generation (ideal-point MIN over peer memory,
    boundary rows by peer copies) == the unsharded engine, bit for bit."""
    gens = 7
    p = g.make_problem(name)
    cfg = g.RunConfig(n=n, k_max=gens, seed=5, op=op, record_walltime=False)
    ref = g.Engine(p, cfg)
    ref.run()
    eng = g.Engine(p, cfg, devices=[0] * shards)
    assert eng.rows_owned == n and eng.shard_info()["reach"] > 0
    eng.step(3)   # stepping and running mix, as through the C ABI
    eng.run()
    assert _pop_equal(eng.population(1), ref.population(1))
    assert _pop_equal(eng.population(2), ref.population(2))
    assert np.array_equal(eng.ideal(), ref.ideal())
    assert [r.feasible_ratio for r in eng.history()] == [r.feasible_ratio for r in ref.history()]
    assert np.array_equal(eng.replacement_rates(), ref.replacement_rates())
    assert np.array_equal(eng.neighborhoods().b2, ref.neighborhoods().b2)


def test_multi_device_handle_set_population_and_profile(g):
    p = g.make_problem("LIRCMOP13")
    cfg = g.RunConfig(n=5000, k_max=6, seed=2, op=g.VariationOp.de, record_walltime=False)
    rng = np.random.default_rng(3)
    X1, X2 = rng.random((5000, 30)), rng.random((5000, 30))
    out = []
    for dev in (None, [0, 0, 0]):
        e = g.Engine(p, cfg, devices=dev)
        e.set_population(1, X1)
        e.set_population(2, X2)
        e.step(3)
        ms = e.profile(3)
        assert ms.shape == (5,) and ms[4] > 0 and ms[0] > 0
        out.append((e.population(1), e.ideal(), [r.feasible_ratio for r in e.history()]))
    assert _pop_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1]) and out[0][2] == out[1][2]


def test_multi_device_handle_time_budget(g):
    """Time budget across shards: shard 0 keeps the loop clock and every shard
    keeps or discards the same generation; the result equals an unsharded run
    of exactly the generations the history records."""
    p = g.make_problem("LIRCMOP1")
    eng = g.Engine(p, g.RunConfig(n=3000, time_budget_s=0.08, seed=4, op=g.VariationOp.de), devices=[0, 0])
    eng.run()
    h = eng.history()
    gens = len(h) - 1
    assert gens > 5 and h[-1].wall_ms < 80.0
    ref = g.run_gmpea(p, g.RunConfig(n=3000, k_max=gens, seed=4, op=g.VariationOp.de))
    assert _pop_equal(eng.population(1), ref.pop1)


@pytest.mark.parametrize("time_budget", [None, 0.05])
def test_nccl_single_rank_engine_equals_unsharded(g, time_budget):
    """The NCCL data plane at world = 1 (one B200 per gpurun call): the
    all-reduce, the rank-0 clock broadcast and the generation graph with NCCL
    captured in it run, and the run equals the plain engine's."""
    p = g.make_problem("MW7")
    base = dict(n=4000, seed=6, op=g.VariationOp.sbx_pm, record_walltime=False)
    if time_budget is None:
        cfg = g.RunConfig(k_max=8, world=1, rank=0, nccl_id=g.nccl_unique_id(), **base)
        eng = g.Engine(p, cfg)
        eng.run()
        ref = g.run_gmpea(p, g.RunConfig(k_max=8, **base))
    else:
        cfg = g.RunConfig(time_budget_s=time_budget, world=1, rank=0, nccl_id=g.nccl_unique_id(), **base)
        eng = g.Engine(p, cfg)
        eng.run()
        ref = g.run_gmpea(p, g.RunConfig(k_max=len(eng.history()) - 1, **base))
    assert _pop_equal(eng.population(1), ref.pop1)
    assert [r.feasible_ratio for r in eng.history()] == [r.feasible_ratio for r in ref.history]
