import sys, numpy as np
sys.path.insert(0, "tests")
import paper_2509_19821_b200 as g
from test_gpu_baselines import _cases
out = {}
for k, (F, cv) in enumerate(_cases(1)):
    out[f"{k}/F"] = F; out[f"{k}/cv"] = cv; out[f"{k}/fit"] = g.spea2_fitness(F, cv, True)
np.savez("gpurun_out/dbg.npz", **out)
