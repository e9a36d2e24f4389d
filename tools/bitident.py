"""Runs a few problems with the library in GMPEA_LIB and saves the final
populations, for bit-identity checks between builds:
    GMPEA_LIB=a.so python tools/bitident.py out_a.npz; ... ; python tools/bitident.py --cmp a.npz b.npz"""
import sys

import numpy as np

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k], equal_nan=True)]
    print("identical" if not bad else f"DIFFER: {bad}")
    sys.exit(0)
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19821_b200 as g  # noqa: E402

out = {}
for name, op, n in (("MW7", 0, 20000), ("DASCMOP9", 0, 20000), ("WTA-P10", 0, 4000), ("C1-DTLZ1", 0, 20000),
                    ("LIRCMOP13", 1, 20000)):
    e = g.Engine(g.make_problem(name), g.RunConfig(n=n, k_max=30, seed=3, op=op, record_walltime=False))
    e.run()
    for w in ("1", "2"):
        pop = e.population(int(w))
        for f in ("X", "F", "C", "cv"):
            out[f"{name}/{w}/{f}"] = getattr(pop, f)
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1])
