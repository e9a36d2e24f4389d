mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "restated" > gpurun_out/pytest_pf.log 2>&1; echo pytest=$?; tail -25 gpurun_out/pytest_pf.log
python - <<'PY'
import numpy as np, sys
sys.path.insert(0, "tests")
import paper_2509_19821_b200 as g
fx = np.load("tests/golden/pf_restated.npz")
for name in [f"MW{i}" for i in range(1, 15)] + [f"DASCMOP{i}" for i in range(1, 10)]:
    for n in (64, 1000):
        ref = fx[f"{name}/{n}"]; got = g.pf_reference(g.make_problem(name), n)
        if got.shape != ref.shape: print(name, n, "shape", got.shape, ref.shape); continue
        close = np.all(np.abs(got - ref) <= 1e-7 * np.maximum(1.0, np.abs(ref)), axis=1).mean()
        print(name, n, "close %.3f" % close, "maxdiff %.2e" % np.abs(got - ref).max())
PY
