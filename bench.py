"""GMPEA-B200 benchmark (driver contract: one JSON line on rank 0).

A step is one GMPEA generation (gmpea.cpp:457-489: reproduce x2, evaluate x2,
update_ideal, environmental selection) over both populations.  The headline
workload is BASELINE.json configs[2]: LIRCMOP13 (m = 3, D = 30, DE — the
suite default, experiment.cpp:117-123) at N = 1,000,000 subproblems, the
N = 1M metric "individual-generations/sec" (2N per generation, the
reference's evals unit, gmpea.cpp:433,487).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Multi-GPU (torchrun, one rank per GPU): the same N = 1M run split into
weight-region shards — an ideal-point all-reduce and a
boundary-row exchange over NCCL per generation; value = 2N per generation /
max step time over ranks (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (problem, n, op)
    "lircmop13-1m": ("LIRCMOP13", 1_000_000, 1),
    "lircmop14-1m": ("LIRCMOP14", 1_000_000, 1),
    "mw1-1m": ("MW1", 1_000_000, 0),
    "mw7-1m": ("MW7", 1_000_000, 0),
    "mw7-10m": ("MW7", 10_000_000, 0),
    "wta-p10-100k": ("WTA-P10", 100_000, 0),
}
METRIC = "individual-generations/sec at N=1M"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


def alg_bytes(d, m, nc, t1, t2):
    """Algorithmic bytes per individual:
    vary_eval reads the parent row + its neighbour row and writes the child
    row (X, G, packed F|cv); op1 reads two packed keys + the unit weight and
    writes two keys + a byte; select reads the parent key, weight and reverse
    row.  Winner copies are data-dependent and not counted."""
    tbar = (t1 + t2) / 2.0
    vary = 4 * d + 4 * tbar + 4 * (d + nc + 4)
    op1 = (2 * 16 + 16 + 2 * 16 + 1) / 2.0
    sel = 16 + 16 + 4 * tbar
    return {"vary_eval": vary, "op1": op1, "select": sel,
            "survey_B_alg": 8 * (d + m + nc + 1) + 4 * m + 4 * tbar}


class Clocks:
    """nvidia-smi samples during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.05)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[4 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        return s.get(kernel, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def cpu_reference(problem, n, op, gens, warmup, threads, seed=1, topo=None):
    """The reference's own loop (oracle/_ref) on host cores; returns
    (ind-gen/s, seconds, replicas, kind)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Reference  # checker / baseline only

    if not Reference.available():
        raise RuntimeError("oracle/_ref not built")
    ref = Reference()
    secs = ref.loop_bench(problem, n, op, topo.b1, topo.b2, warmup, gens, threads, seed)
    value = threads * 2 * n * gens / float(secs.max())
    return value, float(secs.max()), "reference"


def host_topology(problem, n):
    import paper_2509_19821_b200 as g

    p = g.make_problem(problem)
    return g.lattice_neighborhoods(p.m, n, 5, 20)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="lircmop13-1m", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-gens", type=int, default=2)
    args = ap.parse_args()
    world, rank, local = dist_env()
    problem, n, op = WORKLOADS[args.workload]
    config = {"workload": f"{args.workload}: {problem} (BASELINE configs[2]), N={n}, t1=5, t2=20, "
                          f"theta=5, op={'de' if op else 'sbx_pm'}, seed=1",
              "problem": problem, "N": n, "l2": "working set > 126 MB L2 (no flush needed)"}

    if args.impl == "reference":
        if rank != 0:
            return
        threads = int(os.environ.get("GMPEA_REF_THREADS", "0")) or max(1, min(os.cpu_count() or 1, 8))
        topo = host_topology(problem, n)
        vals = []
        for _ in range(args.steps):
            v, secs, kind = cpu_reference(problem, n, op, 1, 0, threads, topo=topo)
            vals.append(v)
        value = float(np.median(vals))
        line = {"metric": METRIC, "value": value, "unit": "ind-gen/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 2 * n / value * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (Philox/mt19937 initial populations)", "impl": "reference",
                "config": config,
                "cpu_baseline": {"value": value, "unit": "ind-gen/s", "cores": threads, "kind": kind,
                                 "sample": f"{threads} independent reference runs x 1 generation of "
                                           f"N={n} per step (topology injected, setup untimed)"},
                "e2e": {"value": value, "unit": "ind-gen/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    import paper_2509_19821_b200 as g

    stream = torch.cuda.Stream()  # the engine's launching stream (events are recorded on it)
    torch.cuda.set_stream(stream)
    prob = g.make_problem(problem)
    PRE_MAX = 20000  # untimed generations keeping the GPU busy while the clock sampler settles
    budget_gens = args.warmup + 4 * args.steps + 16 + PRE_MAX
    if world == 1:
        cfg = g.RunConfig(n=n, k_max=0, eval_budget=2 * n * budget_gens, seed=1, op=op, device=local,
                          stream=stream.cuda_stream)
        eng = g.Engine(prob, cfg)
        advance = eng.step  # CUDA-graph replay, one graph per generation
    else:
        # weight-region shards of the same N = 1M run (strong scaling): ideal
        # point all-reduce + boundary-row exchange over NCCL every generation
        from paper_2509_19821_b200.sharded import GpuShard, TorchComm

        cfg = g.RunConfig(n=n, k_max=budget_gens, seed=1, op=op, device=local, stream=stream.cuda_stream)
        shard = GpuShard(prob, cfg, world, rank, TorchComm())
        eng = shard.eng
        advance = shard.run
    t0 = time.perf_counter()
    advance(args.warmup)
    torch.cuda.synchronize()
    t_gen = (time.perf_counter() - t0) / max(1, args.warmup)
    pre = int(min(PRE_MAX, max(0, 0.6 / max(t_gen, 1e-6))))  # ~0.6 s of load before the timed region
    if world > 1:
        t = torch.tensor([pre], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        pre = int(t.item())
        torch.distributed.barrier()

    # ---- timed region: K generations, CUDA events on the engine's stream; the
    # clock sampler runs across the untimed load generations and the region
    clocks = Clocks(local)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clocks:
        advance(pre)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        start.record(stream)
        advance(args.steps)
        end.record(stream)
        torch.cuda.synchronize()
    eng.sync()
    ms_total = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms_total], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = 2 * n / (ms_step * 1e-3)  # whole job: all ranks together process the N-slot generation
    # per-kernel device times (events around every launch) on this rank's
    # engine; run after the timed region (the shards no longer exchange)
    kms = eng.profile(args.steps)

    # ---- e2e: the public API with (pinned) host buffers
    def pinned(shape):
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()

    rng = np.random.default_rng(7)
    X1, X2 = pinned((n, prob.d)), pinned((n, prob.d))
    X1[:] = prob.lower + (prob.upper - prob.lower) * rng.random((n, prob.d))
    X2[:] = prob.lower + (prob.upper - prob.lower) * rng.random((n, prob.d))
    if world == 1:
        eng2 = g.Engine(prob, g.RunConfig(n=n, k_max=args.steps, seed=11, op=op, device=local))
        step1 = lambda: eng2.step(1)  # noqa: E731
    else:
        sh2 = GpuShard(prob, g.RunConfig(n=n, k_max=args.steps, seed=11, op=op, device=local,
                                         stream=stream.cuda_stream), world, rank, TorchComm())
        eng2 = sh2.eng
        step1 = sh2.step
    rows = eng2.rows_owned
    out = g.Population(pinned((rows, prob.d)), pinned((rows, prob.m)), pinned((rows, prob.n_constraints)),
                       pinned(rows))
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    eng2.set_population(1, X1)
    eng2.set_population(2, X2)
    if world > 1:
        sh2._z_allreduce()
    for _ in range(args.steps):
        step1()
        eng2.last_record()  # D2H of the generation's record (feasible ratio), host-synchronous
    pop = eng2.population(1, out=out)
    t1 = time.perf_counter()
    e2e_s = t1 - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = X1.nbytes + X2.nbytes
    d2h = 48 * args.steps + pop.X.nbytes + pop.F.nbytes + pop.C.nbytes + pop.cv.nbytes
    e2e = {"value": 2 * n * args.steps / e2e_s, "unit": "ind-gen/s",
           "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
           "note": "pinned host buffers: set_population x2 (H2D + evaluation) + K x (step + GenRecord "
                   "read) + final pop1 (X, F, C, cv) D2H, host wall clock, max over ranks"}
    eng2.close()

    if rank != 0:
        eng.close()
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    pk, pk_kind = peaks()
    ab = alg_bytes(prob.d, prob.m, prob.n_constraints, 5, 20)
    names = ["vary_eval", "op1", "select"]
    shares = {k: float(kms[i] / kms[4]) for i, k in enumerate(names)}
    dom = max(names, key=lambda k: kms[names.index(k)])
    di = names.index(dom)
    units = 2 * n if dom != "op1" else n
    per_unit = ab[dom] * (2 if dom == "op1" else 1)
    achieved = per_unit * units / (kms[di] * 1e-3) / 1e9
    traffic = ncu_traffic(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "peak_kind": pk_kind,
                "alg_bytes_per_unit": per_unit, "units_per_launch": units,
                "kernel_ms": {k: float(kms[i]) for i, k in enumerate(names)},
                "kernel_share": shares,
                "whole_step": {"alg_bytes_per_individual": ab["survey_B_alg"],
                               "achieved_GBps": ab["survey_B_alg"] * 2 * n / (ms_step * 1e-3) / 1e9}}

    cpu = None
    if not args.no_cpu_baseline:
        try:
            topo = eng.neighborhoods()
            threads = max(1, min(os.cpu_count() or 1, 8))
            v, secs, kind = cpu_reference(problem, n, op, args.cpu_gens, 0, threads, topo=topo)
            cpu = {"value": v, "unit": "ind-gen/s", "cores": threads, "kind": kind,
                   "sample": f"{threads} concurrent reference runs x {args.cpu_gens} generations of "
                             f"N={n} ({secs:.1f} s), topology injected, setup untimed"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "ind-gen/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    eng.close()

    line = {"metric": METRIC, "value": value, "unit": "ind-gen/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong",  # N = 1M slots in total, split into weight-region shards
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (Philox-initialised populations)",
            "config": config, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks.summary(), "gpu_launches": int(args.steps * 5 + 1)}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
