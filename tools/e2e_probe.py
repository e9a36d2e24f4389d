"""Breaks the bench's e2e timed region into its parts (set_population x2,
K steps, final population D2H) to see where the host-path time goes."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2509_19821_b200 as g

name, n, op, K = sys.argv[1] if len(sys.argv) > 1 else "LIRCMOP13", 1_000_000, 1, 100
prob = g.make_problem(name)
def pinned(shape):
    return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
rng = np.random.default_rng(7)
X1, X2 = pinned((n, prob.d)), pinned((n, prob.d))
X1[:] = prob.lower + (prob.upper - prob.lower) * rng.random((n, prob.d))
X2[:] = prob.lower + (prob.upper - prob.lower) * rng.random((n, prob.d))
for rep in range(3):
    eng = g.Engine(prob, g.RunConfig(n=n, k_max=K, seed=11, op=op))
    out = g.Population(pinned((n, prob.d)), pinned((n, prob.m)), pinned((n, prob.n_constraints)), pinned(n))
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    eng.set_population(1, X1); t.append(time.perf_counter())
    eng.set_population(2, X2); t.append(time.perf_counter())
    recs = torch.zeros((K, 16), dtype=torch.uint8, pin_memory=True).numpy()
    for k in range(K):
        eng.step(1)
        eng.record_async(recs[k])
    eng.sync(); t.append(time.perf_counter())
    eng.population(1, out=out); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(name, "set1 %.2f set2 %.2f steps %.2f pop %.2f total %.2f ms" % (*d, sum(d)),
          "H2D GB/s %.1f" % (X1.nbytes / d[0] / 1e6), "D2H GB/s %.1f" % ((out.X.nbytes + out.F.nbytes + out.C.nbytes + out.cv.nbytes) / d[3] / 1e6))
    eng.close()
