import sys, numpy as np
sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import paper_2509_19821_b200 as g
fx = np.load("tests/golden/pf_restated.npz")
for name in sys.argv[1:]:
    got = g.pf_reference(g.make_problem(name), 64)
    nd = fx[f"{name}/nd64"]
    ref = fx[f"{name}/64"]
    dist = np.abs(got[:, None, :] - nd[None, :, :]).max(-1).min(1)
    print(name, "nd", len(nd), "bad rows", np.where(dist > 1e-9)[0])
    for i in np.where(dist > 1e-9)[0][:6]:
        j = np.abs(nd - got[i]).max(1).argmin()
        print("  got", got[i], "nearest nd", nd[j], "ref row", ref[i])
