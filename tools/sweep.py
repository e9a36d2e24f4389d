"""Population sweep (BASELINE.json configs[4]): throughput and whole-step HBM
roofline fraction on MW7 for N = 10^3 .. 10^7 on one B200 (the multi-GPU
points come from bench.py under torchrun).

    python tools/sweep.py [--problem MW7] [--out profiles/r01_sweep_mw7.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problem", default="MW7")
    ap.add_argument("--sizes", default="1000,10000,100000,1000000,10000000")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_sweep_mw7.json"))
    args = ap.parse_args()
    import torch

    import paper_2509_19821_b200 as g

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    p = g.make_problem(args.problem)
    op = 1 if args.problem.startswith("LIRCMOP") else 0
    b_alg = 8 * (p.d + p.m + p.n_constraints + 1) + 4 * p.m + 4 * 12.5
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    out = []
    for n in (int(x) for x in args.sizes.split(",")):
        steps = max(20, min(2000, 20_000_000 // n))
        warm = max(5, steps // 10)
        eng = g.Engine(p, g.RunConfig(n=n, k_max=warm + 2 * steps + 4, seed=1, op=op, stream=stream.cuda_stream))
        eng.step(warm)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.step(steps)
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        kms = eng.profile(min(steps, 50))
        rate = 2 * n / (ms * 1e-3)
        rec = {"problem": args.problem, "N": n, "steps": steps, "ms_per_generation": ms,
               "ind_gen_per_s": rate, "whole_step_GBps": rate * b_alg / 1e9,
               "whole_step_frac_of_hbm": rate * b_alg / 1e9 / peak,
               "kernel_ms": {"vary_eval": kms[0], "op1": kms[1], "select": kms[2], "end_gen": kms[3]}}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        eng.close()
    with open(args.out, "w") as f:
        json.dump({"B_alg_bytes": b_alg, "hbm_peak_GBps": peak, "points": out}, f, indent=1)


if __name__ == "__main__":
    main()
