"""TEST INFRASTRUCTURE: an f64 oracle implementation of one shard of a
weight-region sharded run, driven by the product's own plan and exchange
logic (paper_2509_19821_b200/sharded.py) over torch.distributed.  The CPU
tests run it with gloo at world size 2 and compare against world size 1."""
import numpy as np


class OracleShard:
    def __init__(self, orc, name, n, world, rank, comm, seed=3, op=1, t1=5, t2=20):
        import torch

        from paper_2509_19821_b200.sharded import halo_plan

        self.torch, self.orc, self.name, self.comm = torch, orc, name, comm
        self.seed, self.op = seed, op
        info = orc.problem_info(name)
        self.m, self.d = info["m"], info["d"]
        W = orc.reference_vectors(self.m, n)
        Bg = [orc.knn(W, t1), orc.knn(W, t2)]
        idx = np.arange(n)[:, None]
        reach = int(max(np.abs(B.astype(np.int64) - idx).max() for B in Bg)) if world > 1 else 0
        self.plan = halo_plan(n, world, rank, reach)
        w0, w1 = self.plan.window
        v0, v1 = self.plan.vary
        self.W = W[w0:w1]
        self.B = []
        for B in Bg:
            loc = np.repeat(np.arange(w1 - w0, dtype=np.uint32)[:, None], B.shape[1], 1)  # dummies: self
            loc[v0 - w0:v1 - w0] = B[v0:v1] - w0
            self.B.append(np.ascontiguousarray(loc, np.uint32))
        self.pops = []
        for q in range(2):
            X = orc.init_population(name, n, seed, q + 1)[w0:w1]
            F, G, cv = orc.evaluate(name, X)
            self.pops.append(dict(X=X, F=F, C=G, cv=cv))
        o0, o1 = self.plan.own
        z = np.minimum(self.pops[0]["F"][o0 - w0:o1 - w0].min(0), self.pops[1]["F"][o0 - w0:o1 - w0].min(0))
        self.z = self._zmin(z)
        self.gen = 0

    def _zmin(self, z):
        t = self.torch.tensor(z, dtype=self.torch.float64)
        self.comm.allreduce_min_(t)
        return t.numpy().copy()

    def step(self):
        self.gen += 1
        w0 = self.plan.window[0]
        v0, v1 = self.plan.vary[0] - w0, self.plan.vary[1] - w0
        offs = []
        for q in range(2):
            X = self.pops[q]["X"]
            ox, _ = self.orc.reproduce(self.name, X, self.B[q], self.op, self.seed, self.gen, q + 1, slot_base=w0)
            off = {k: v.copy() for k, v in self.pops[q].items()}  # dummies outside the vary rows
            F, G, cv = self.orc.evaluate(self.name, ox[v0:v1])
            off["X"][v0:v1], off["F"][v0:v1], off["C"][v0:v1], off["cv"][v0:v1] = ox[v0:v1], F, G, cv
            offs.append(off)
        z = np.minimum(self.z, np.minimum(offs[0]["F"][v0:v1].min(0), offs[1]["F"][v0:v1].min(0)))
        self.z = self._zmin(z)
        s1, s2 = self.orc.selection(self.pops + offs, self.W, self.z, 5.0, self.B[0], self.B[1])
        o0, o1 = self.plan.own[0] - w0, self.plan.own[1] - w0
        nw = len(s1)
        for q, s in ((0, s1), (1, s2)):
            for j in range(o0, o1):
                if s[j] >= 0:
                    src = offs[0] if s[j] < nw else offs[1]
                    for k in ("X", "F", "C", "cv"):
                        self.pops[q][k][j] = src[k][s[j] % nw]
        self._exchange()

    def _exchange(self):
        T = self.torch
        w0 = self.plan.window[0]
        ops, back = [], []
        for q in range(2):
            for k in ("X", "F", "C", "cv"):
                arr = self.pops[q][k]
                for peer, a, b in self.plan.sends:
                    ops.append((peer, T.from_numpy(np.ascontiguousarray(arr[a - w0:b - w0])), None))
                for peer, a, b in self.plan.recvs:
                    buf = T.from_numpy(np.zeros_like(arr[a - w0:b - w0]))
                    ops.append((peer, None, buf))
                    back.append((arr, a - w0, b - w0, buf))
        self.comm.exchange(ops)
        for arr, a, b, buf in back:
            arr[a:b] = buf.numpy()

    def owned(self, q=0):
        w0 = self.plan.window[0]
        o0, o1 = self.plan.own
        return {k: v[o0 - w0:o1 - w0].copy() for k, v in self.pops[q].items()}
