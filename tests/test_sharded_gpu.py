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
