"""Weight-region sharded GMPEA runs across GPUs.

The lexicographic Das-Dennis order makes contiguous slot ranges weight-space
slabs.  Rank g owns slots [o0, o1) of both populations.  With the
neighbourhood reach r = max |B[i][l] - i| the engine keeps parent rows of its
window [o0 - 2r, o1 + 2r), regenerates the offspring of [o0 - r, o1 + r) with
the global Philox keys (so they equal their owners' offspring bit for bit —
no offspring travel), all-reduces the ideal point (MIN) between variation and
selection, selects its own slots, and then exchanges the 2r boundary rows
with each neighbour.  Per generation: one m-word all-reduce and two P2P
exchanges of 2r rows (+ keys) per side.

The driver is written against a small backend interface so the same plan and
exchange logic runs on

* `GpuShard`      the CUDA engine (one per GPU, torch.distributed NCCL), and
* `oracle_shard`  (tests only) the f64 oracle on CPU (gloo), which checks the
                  decomposition against an unsharded oracle run.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Tuple

import numpy as np


def shard_ranges(n: int, world: int) -> List[Tuple[int, int]]:
    """Balanced contiguous slot ranges (weight-space slabs)."""
    return [(r * n // world, (r + 1) * n // world) for r in range(world)]


@dataclasses.dataclass
class HaloPlan:
    own: Tuple[int, int]
    window: Tuple[int, int]
    vary: Tuple[int, int]
    # (peer, global row begin, global row end): rows I send / rows I receive
    sends: List[Tuple[int, int, int]]
    recvs: List[Tuple[int, int, int]]


def halo_plan(n: int, world: int, rank: int, reach: int) -> HaloPlan:
    own = shard_ranges(n, world)
    o0, o1 = own[rank]
    if world > 1 and min(b - a for a, b in own) < 2 * reach:
        raise ValueError(f"shards of {n // world} slots are narrower than twice the reach ({2 * reach})")
    w = (max(0, o0 - 2 * reach), min(n, o1 + 2 * reach))
    v = (max(0, o0 - reach), min(n, o1 + reach))
    sends, recvs = [], []
    if rank > 0 and reach > 0:
        sends.append((rank - 1, o0, o0 + 2 * reach))  # the left neighbour's right halo
        recvs.append((rank - 1, w[0], o0))
    if rank < world - 1 and reach > 0:
        sends.append((rank + 1, o1 - 2 * reach, o1))
        recvs.append((rank + 1, o1, w[1]))
    return HaloPlan((o0, o1), w, v, sends, recvs)


# ------------------------------------------------------------------ comms
class TorchComm:
    """torch.distributed plumbing (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group

        # gloo (CPU tests, functional checks of several ranks on one GPU) moves
        # host tensors only: device tensors are staged through host memory
        self.staged = dist.get_backend(group) == "gloo"

    def _host(self, t):
        return t.cpu() if (self.staged and t is not None and t.is_cuda) else t

    def allreduce_min_(self, t):
        h = self._host(t)
        self.dist.all_reduce(h, op=self.dist.ReduceOp.MIN, group=self.group)
        if h is not t:
            t.copy_(h)

    def allreduce_sum_(self, t):
        h = self._host(t)
        self.dist.all_reduce(h, op=self.dist.ReduceOp.SUM, group=self.group)
        if h is not t:
            t.copy_(h)

    def exchange(self, ops):
        """ops: list of (peer, send_tensor, recv_tensor); all posted at once."""
        d = self.dist
        if self.staged:
            hops = [(peer, self._host(snd), self._host(rcv)) for peer, snd, rcv in ops]
            self._exchange(d, hops)
            for (_, _, rcv), (_, _, hr) in zip(ops, hops):
                if rcv is not None and hr is not rcv:
                    rcv.copy_(hr)
            return
        self._exchange(d, ops)

    def _exchange(self, d, ops):
        p2p = []
        for peer, snd, rcv in ops:
            if snd is not None:
                p2p.append(d.P2POp(d.isend, snd, peer, group=self.group))
            if rcv is not None:
                p2p.append(d.P2POp(d.irecv, rcv, peer, group=self.group))
        if p2p:
            for req in d.batch_isend_irecv(p2p):
                req.wait()


# ------------------------------------------------------------------ GPU shard
class _CAI:
    """A raw device range as a __cuda_array_interface__ object."""

    def __init__(self, ptr: int, nbytes: int, typestr: str = "|u1"):
        item = int(typestr[-1])
        self.__cuda_array_interface__ = {"shape": (nbytes // item,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class GpuShard:
    """One rank of a sharded run: the CUDA engine plus its halo plan."""

    def __init__(self, problem, cfg, world: int, rank: int, comm):
        import torch

        from ._lib import Engine, RunConfig

        self.torch = torch
        self.world, self.rank, self.comm = world, rank, comm
        own = shard_ranges(cfg.n, world)[rank]
        if not cfg.stream:
            # the engine must run on torch's current stream so the collectives
            # (or in-process copies) are ordered with its kernels
            if torch.cuda.current_stream().cuda_stream == 0:
                torch.cuda.set_stream(torch.cuda.Stream())
            cfg = dataclasses.replace(cfg, stream=torch.cuda.current_stream().cuda_stream)
        c = dataclasses.replace(cfg, shard=own if world > 1 else None)
        self.eng = Engine(problem, c)
        info = self.eng.shard_info()
        self.plan = halo_plan(cfg.n, world, rank, info["reach"])
        assert self.plan.window == (info["window_begin"], info["window_end"]), (self.plan, info)
        assert self.plan.vary == (info["vary_begin"], info["vary_end"])
        b = self.eng.device_buffers()
        w0, w1 = self.plan.window
        rows = w1 - w0
        dev = torch.device("cuda", torch.cuda.current_device())
        self.z = torch.as_tensor(_CAI(b["ideal_bits"], 16, "<i4"), device=dev)
        self.rows = [torch.as_tensor(_CAI(b["rows"][q], rows * b["row_bytes"]), device=dev) for q in range(2)]
        self.keys = [torch.as_tensor(_CAI(b["keys"][q], rows * 16), device=dev) for q in range(2)]
        self.row_bytes = b["row_bytes"]
        self._z_allreduce()  # the initial ideal point is global too (gmpea.cpp:435-437)

    def _z_allreduce(self):
        t = self.torch
        u = self.z.to(t.int64) & 0xFFFFFFFF  # unsigned order-preserving words
        self.comm.allreduce_min_(u)
        self.z.copy_(u.to(t.int32))

    def _slices(self, q, g0, g1):
        w0 = self.plan.window[0]
        rb = self.row_bytes
        return (self.rows[q][(g0 - w0) * rb:(g1 - w0) * rb], self.keys[q][(g0 - w0) * 16:(g1 - w0) * 16])

    def step(self):
        self.eng.phase(1)
        self._z_allreduce()
        self.eng.phase(2)
        ops = []
        for q in range(2):
            sends = {p: self._slices(q, a, b) for p, a, b in self.plan.sends}
            recvs = {p: self._slices(q, a, b) for p, a, b in self.plan.recvs}
            for peer in sorted(set(sends) | set(recvs)):
                s, r = sends.get(peer), recvs.get(peer)
                ops.append((peer, s[0] if s else None, r[0] if r else None))
                ops.append((peer, s[1] if s else None, r[1] if r else None))
        self.comm.exchange(ops)

    def run(self, gens: int):
        for _ in range(gens):
            self.step()

    def population(self, which=1):
        return self.eng.population(which)  # owned rows

    def history(self):
        """GenRecords with the feasible ratio over all ranks (gmpea.cpp:411-417)."""
        t = self.torch
        h = self.eng.history()
        o0, o1 = self.plan.own
        cnt = t.tensor([round(r.feasible_ratio * (o1 - o0)) for r in h], dtype=t.float64,
                       device=self.z.device)
        self.comm.allreduce_sum_(cnt)
        n = self.eng.shard_info()["n_global"]
        for r, c in zip(h, cnt.tolist()):
            r.feasible_ratio = c / n
        return h


def run_local_group(problem, cfg, world: int, gens: int):
    """Runs `world` GpuShards in one process on one device in lockstep: the
    all-reduce and the halo exchange become device copies between phases (a
    single-GPU check of the shard path; no kernel ever waits on another).
    Returns the shards' owned pop1 populations in slot order."""
    import torch

    class _Nop:
        def allreduce_min_(self, t):
            pass

        def allreduce_sum_(self, t):
            pass

        def exchange(self, ops):
            raise RuntimeError("unused")

    shards = [GpuShard(problem, cfg, world, r, _Nop()) for r in range(world)]

    def zmin():
        u = torch.stack([s.z.to(torch.int64) & 0xFFFFFFFF for s in shards]).min(0).values
        for s in shards:
            s.z.copy_(u.to(torch.int32))

    zmin()
    for _ in range(gens):
        for s in shards:
            s.eng.phase(1)
        zmin()
        for s in shards:
            s.eng.phase(2)
        for s in shards:
            for q in range(2):
                for peer, a, b in s.plan.recvs:
                    dr, dk = s._slices(q, a, b)
                    sr, sk = shards[peer]._slices(q, a, b)
                    dr.copy_(sr)
                    dk.copy_(sk)
    torch.cuda.synchronize()
    pops = [s.population(1) for s in shards]
    return pops, shards
