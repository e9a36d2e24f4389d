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
    # BASELINE configs[2]'s DAS-CMOP half (restated problems, SBX as the
    # reference's operator_for gives every non-LIRCMOP suite)
    "dascmop7-1m": ("DASCMOP7", 1_000_000, 0),
    "dascmop9-1m": ("DASCMOP9", 1_000_000, 0),
    # a reference-suite C-DTLZ problem at the same population size
    "c1dtlz1-1m": ("C1-DTLZ1", 1_000_000, 0),
}
# which BASELINE.json config each workload measures
CONFIG_OF = {
    "lircmop13-1m": "BASELINE configs[2]",
    "lircmop14-1m": "BASELINE configs[2]",
    "dascmop7-1m": "BASELINE configs[2]",
    "dascmop9-1m": "BASELINE configs[2]",
    "mw1-1m": "north-star MW target at N=1M",
    "mw7-1m": "BASELINE configs[4] sweep point",
    "mw7-10m": "BASELINE configs[4] sweep point",
    "wta-p10-100k": "BASELINE configs[3]",
    "c1dtlz1-1m": "reference suite at N=1M",
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
    """SM clock and throttle-reason samples DURING the timed region
    (B200_PROFILING.md): an NVML poller thread (~2 ms period), so even a
    50 ms region is sampled; falls back to nvidia-smi if NVML is missing."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.max_mhz = None
        self._stop = None

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:  # noqa: BLE001
            return self
        self._stop = threading.Event()

        def poll():
            while not self._stop.is_set():
                try:
                    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((float(mhz), int(r)))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(0.002)

        self._t = threading.Thread(target=poll, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        reasons = sorted({k for _, r in self.samples for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(np.median([m for m, _ in self.samples])), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def ncu_traffic(kernel, workload):
    """dram bytes per launch of `kernel` from the committed ncu --set full
    summary: the entry "kernel@workload", or the plain "kernel" entry, which
    is the headline workload's capture (None for other workloads without one)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        e = s.get(f"{kernel}@{workload}") or (s.get(kernel) if workload == "lircmop13-1m" else None)
        return (e or {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def cpu_reference(problem, n_sub, op, gens, warmup, threads, seed=1):
    """The reference's own loop (oracle/_ref, gmpea.cpp:457-489) on host
    cores: `threads` concurrent replicas of an n_sub-slot population, each
    running warmup + gens generations; topology from the oracle's windowed
    lattice KNN (identical to build_neighborhoods, tests/test_oracle_pins.py),
    setup untimed.  Returns (ind-gen/s over all replicas, loop seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, Reference  # checker / baseline only

    if not Reference.available():
        raise RuntimeError("oracle/_ref not built")
    ref = Reference()
    m = ref._info_any(problem)["m"]
    b1, b2 = Oracle().lattice_knn(m, n_sub, 5, 20, threads)
    secs = ref.loop_bench(problem, n_sub, op, b1, b2, warmup, gens, threads, seed)
    return threads * 2 * n_sub * gens / float(secs.max()), float(secs.max())


def ref_threads():
    return int(os.environ.get("GMPEA_REF_THREADS", "0")) or max(1, os.cpu_count() or 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)   # generations 11-110
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="lircmop13-1m", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-gens", type=int, default=20)
    args = ap.parse_args()
    world, rank, local = dist_env()
    problem, n, op = WORKLOADS[args.workload]
    config = {"workload": f"{args.workload}: {problem} ({CONFIG_OF[args.workload]}), N={n}, t1=5, t2=20, "
                          f"theta=5, op={'de' if op else 'sbx_pm'}, seed=1",
              "problem": problem, "N": n, "l2": "working set > 126 MB L2 (no flush needed)"}

    if args.impl == "reference":
        if rank != 0:
            return
        # bounded sample of the workload: `threads` concurrent replicas of
        # N/threads slots (N slot-generations per step in total), one
        # generation per step, all host threads busy
        threads = ref_threads()
        n_sub = int(os.environ.get("GMPEA_REF_SLOTS", "0")) or -(-n // threads)
        value, secs = cpu_reference(problem, n_sub, op, args.steps, min(args.warmup, 3), threads)
        sample = (f"{threads} concurrent reference runs (oracle/_ref, unmodified gmpea loop) x N={n_sub} "
                  f"slots x {args.steps} timed generations ({secs:.1f} s), windowed-lattice topology, "
                  f"setup untimed")
        line = {"metric": METRIC, "value": value, "unit": "ind-gen/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": threads * 2 * n_sub / value * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (mt19937_64 initial populations)", "impl": "reference",
                "config": config,
                "cpu_baseline": {"value": value, "unit": "ind-gen/s", "cores": threads, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": value, "unit": "ind-gen/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    # GMPEA_DIST_BACKEND=gloo: a functional check of the sharded path with
    # several ranks on fewer GPUs (host-staged exchange, no rank's kernel waits
    # on another's); never a bench number.  The product path is NCCL.
    backend = os.environ.get("GMPEA_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group(backend)
    import paper_2509_19821_b200 as g

    stream = torch.cuda.Stream()  # the engine's launching stream (events are recorded on it)
    torch.cuda.set_stream(stream)
    prob = g.make_problem(problem)
    budget_gens = args.warmup + 4 * args.steps + 16
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
    advance(args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()

    # ---- timed region: K generations, CUDA events on the engine's stream,
    # clocks sampled by NVML while it runs
    clocks = Clocks(local)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clocks:
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
    # replacement rate over the timed generations (it drifts
    # over a run, so it is reported with the throughput)
    rr = eng.replacement_rates()
    rep_rate = float(np.mean(rr[args.warmup + 1:args.warmup + 1 + args.steps]))
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
    # each step's result (the generation record: pop1 feasible count) is
    # copied D2H into pinned memory in stream order, without a host stall
    # between steps; the host reads them after the final population copy
    recs = torch.zeros((args.steps, 16), dtype=torch.uint8, pin_memory=True).numpy()
    for k in range(args.steps):
        step1()
        eng2.record_async(recs[k])
    pop = eng2.population(1, out=out)  # synchronises the stream
    feas = recs.view(np.uint32)[:, 0].astype(np.float64) / rows
    t1 = time.perf_counter()
    e2e_s = t1 - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = X1.nbytes + X2.nbytes
    d2h = recs.nbytes + pop.X.nbytes + pop.F.nbytes + pop.C.nbytes + pop.cv.nbytes
    e2e = {"value": 2 * n * args.steps / e2e_s, "unit": "ind-gen/s",
           "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
           "note": "pinned host buffers: set_population x2 (H2D + evaluation) + K x (step + async D2H "
                   "of the step's generation record) + final pop1 (X, F, C, cv) D2H, host wall clock, "
                   "max over ranks",
           "feasible_ratio_last": float(feas[-1])}
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
    traffic = ncu_traffic(dom, args.workload)
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
            threads = ref_threads()
            n_sub = -(-n // threads)
            v, secs = cpu_reference(problem, n_sub, op, args.cpu_gens, 1, threads)
            cpu = {"value": v, "unit": "ind-gen/s", "cores": threads, "kind": "reference",
                   "sample": f"{threads} concurrent reference runs x N={n_sub} slots x {args.cpu_gens} "
                             f"generations ({secs:.1f} s), windowed-lattice topology, setup untimed"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "ind-gen/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    eng.close()

    if backend != "nccl":
        config["functional_check"] = f"{world} ranks over {backend} on {torch.cuda.device_count()} GPU(s): not a bench number"
    line = {"metric": METRIC, "value": value, "unit": "ind-gen/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong",  # N = 1M slots in total, split into weight-region shards
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (Philox-initialised populations)",
            "config": config, "replacement_rate": rep_rate, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks.summary(), "gpu_launches": int(3 * args.steps + 1 if world == 1 else 4 * args.steps)}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
