"""CPU: the weight-region shard decomposition (paper_2509_19821_b200/sharded.py)
at world size 2 over gloo, with the f64 oracle as the shard backend, equals the
unsharded run bit for bit (global Philox keys + halo + ideal-point all-reduce)."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, os.path.join(ROOT, "tests"))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, n, gens, out_dir):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle import Oracle
    from oracle_shard import OracleShard

    from paper_2509_19821_b200.sharded import TorchComm

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sh = OracleShard(Oracle(), name, n, world, rank, TorchComm(), op=1 if name.startswith("LIR") else 0)
    for _ in range(gens):
        sh.step()
    o = sh.owned(0)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), own=np.array(sh.plan.own), **o)
    dist.destroy_process_group()


def _run(world, name, n, gens, tmp_path):
    import torch.multiprocessing as mp

    d = tmp_path / f"w{world}"
    d.mkdir()
    mp.spawn(_worker, args=(world, _free_port(), name, n, gens, str(d)), nprocs=world, join=True)
    parts = [np.load(d / f"rank{r}.npz") for r in range(world)]
    return {k: np.concatenate([p[k] for p in parts]) for k in ("X", "F", "C", "cv")}, parts


def test_halo_plan_shapes():
    from paper_2509_19821_b200.sharded import halo_plan, shard_ranges

    assert shard_ranges(10, 3) == [(0, 3), (3, 6), (6, 10)]
    p = halo_plan(1000, 4, 1, 20)
    assert p.own == (250, 500) and p.window == (210, 540) and p.vary == (230, 520)
    assert p.sends == [(0, 250, 290), (2, 460, 500)] and p.recvs == [(0, 210, 250), (2, 500, 540)]
    assert halo_plan(1000, 4, 0, 20).recvs == [(1, 250, 290)]
    with pytest.raises(ValueError):
        halo_plan(100, 4, 0, 20)


@pytest.mark.parametrize("name,n", [("LIRCMOP1", 160), ("LIRCMOP13", 1000)])
def test_two_shards_equal_one(tmp_path, name, n):
    gens = 4
    one, _ = _run(1, name, n, gens, tmp_path)
    two, parts = _run(2, name, n, gens, tmp_path)
    assert [tuple(p["own"]) for p in parts] == [(0, n // 2), (n // 2, n)]
    for k in ("X", "F", "C", "cv"):
        assert np.array_equal(one[k], two[k]), k
