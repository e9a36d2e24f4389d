"""GMPEA-B200 benchmark (driver contract: one JSON line on rank 0).

A step is one GMPEA generation (gmpea.cpp:457-489: reproduce x2, evaluate x2,
update_ideal, environmental selection) over both populations.  The headline
workload is BASELINE.json configs[2]: LIRCMOP13 (m = 3, D = 30, DE — the
suite default, experiment.cpp:117-123) at N = 1,000,000 subproblems, the
N = 1M metric "individual-generations/sec" (2N per generation, the
reference's evals unit, gmpea.cpp:433,487).  The metric's second half, "IGD
at fixed 1 s budget", is the line's `quality_1s` (LIRCMOP13: the engine at
N = 10^5 and the reference's own loop at N = 1000 on one core, both with
run_gmpea's deadline semantics, gmpea.cpp:458,481-486).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Multi-GPU: one process per GPU (torchrun; `--gpus N` without torchrun
re-launches itself under torch.distributed.run).  The same N = 1M run is split
into weight-region shards; the engine all-reduces the ideal
point and exchanges the boundary rows over NCCL inside every generation's
CUDA graph (torch.distributed only shares the NCCL id and takes the max of
the ranks' times).  value = 2N per generation / max step time over ranks
(strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
    50 ms region is sampled."""

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


def relaunch_distributed(nproc):
    """`python bench.py --gpus N` outside torchrun: run this script under
    torch.distributed.run with one rank per GPU (rank 0 prints the line)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


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


def quality_1s(g, problem="LIRCMOP13", op=1, budget=1.0, gpu_n=100_000, ref_n=1000, seed=1):
    """The metric's second half: final IGD after a fixed 1 s loop budget with
    run_gmpea's semantics (checked before each generation, the crossing one
    discarded: gmpea.cpp:458,481-486), scored with metric_front + IGD against
    the reference's own 1000-point pf_reference front (tests/golden/fronts.npz).
    The engine runs on this GPU at N = gpu_n; the reference's own run_gmpea
    (oracle/_ref) on one host core at N = ref_n."""
    front = np.load(os.path.join(ROOT, "tests", "golden", "fronts.npz"))[problem]
    p = g.make_problem(problem)
    out = {"problem": problem, "budget_s": budget, "seed": seed, "front": "reference pf_reference, 1000 points"}
    # tens of thousands of generations at N = 10^5 can meet the reference's PM
    # hazard (its own evaluation error, which the engine raises as it does)
    r, retries = retry_hazard(lambda sd: g.run_gmpea(p, g.RunConfig(n=gpu_n, time_budget_s=budget, seed=sd, op=op)),
                              first_seed=seed)
    fr = g.metric_front(r.pop1)
    out["engine"] = {"n": gpu_n, "seed": seed + retries, "generations": r.history[-1].gen,
                     "loop_ms": r.history[-1].wall_ms, "front_points": int(len(fr)),
                     "igd": float(g.igd(fr, front)) if len(fr) else float("inf")}
    if retries:
        out["engine"]["hazard_retries"] = retries
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from oracle import Reference  # the reference arm (baseline only)

        ref = Reference()
        pop, hist = ref.run_gmpea(problem, ref_n, k_max=0, seed=seed, op=op, time_budget_s=budget,
                                  record_walltime=True)
        rfr = ref.metric_front(pop["F"], pop["cv"])
        out["reference"] = {"n": ref_n, "cores": 1, "generations": int(hist[-1][0]), "loop_ms": float(hist[-1][2]),
                            "front_points": int(len(rfr)),
                            "igd": float(ref.igd(rfr, front)) if len(rfr) else float("inf")}
    except Exception as e:  # noqa: BLE001
        out["reference"] = {"unavailable": str(e)}
    return out


HAZARD = "evaluation failed at generation"


def retry_hazard(fn, dist=None, first_seed=1, tries=4):
    """Runs fn(seed), moving to the next seed when the run stops with the
    reference's own evaluation error (the PM hazard: an out-of-bounds child
    mutated into NaN, gmpea.cpp:146-150, which the engine reproduces instead
    of clipping away; at N = 10^6 a few thousand generations can meet it).
    All ranks agree on a retry.  Returns (result, retries)."""
    for k in range(tries):
        err = None
        try:
            out = fn(first_seed + k)
        except RuntimeError as e:
            if HAZARD not in str(e) or k == tries - 1:
                raise
            err, out = e, None
        failed = 1 if err is not None else 0
        if dist is not None:
            import torch

            t = torch.tensor([failed], dtype=torch.int64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            failed = int(t.item())
        if not failed:
            return out, k
    raise RuntimeError("unreachable")


def throughput(g, eng, steps, warmup, stream):
    """Device-timed generations of an engine: (ms per step, clocks)."""
    import torch

    eng.step(warmup)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    eng.step(steps)
    end.record(stream)
    torch.cuda.synchronize()
    eng.sync()
    return start.elapsed_time(end) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)   # generations 11-110
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="lircmop13-1m", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip quality_1s and the mw1-1m sub-line")
    ap.add_argument("--cpu-gens", type=int, default=20)
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
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
    # several ranks on fewer GPUs (caller-driven exchange, host-staged, no
    # rank's kernel waits on another's); never a bench number.  The product
    # path is the engine's own NCCL exchange.
    backend = os.environ.get("GMPEA_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        # plumbing only (the NCCL id, the max of the ranks' times): gloo on host
        dist.init_process_group("gloo")
    import paper_2509_19821_b200 as g

    stream = torch.cuda.Stream()  # the engine's launching stream (events are recorded on it)
    torch.cuda.set_stream(stream)
    prob = g.make_problem(problem)
    budget_gens = args.warmup + 4 * args.steps + 16

    def shard_cfg(**kw):
        """the run's config: unsharded, or this rank's NCCL shard"""
        if world == 1:
            return g.RunConfig(n=n, seed=kw.pop("seed", 1), op=op, device=local, stream=stream.cuda_stream, **kw)
        if backend == "nccl":
            ids = [g.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(ids, src=0)
            return g.RunConfig(n=n, seed=kw.pop("seed", 1), op=op, device=local, stream=stream.cuda_stream,
                               world=world, rank=rank, nccl_id=ids[0], **kw)
        return g.RunConfig(n=n, seed=kw.pop("seed", 1), op=op, device=local, stream=stream.cuda_stream, **kw)

    legacy = world > 1 and backend != "nccl"
    if legacy:
        from paper_2509_19821_b200.sharded import GpuShard, TorchComm

    def timed(seed):
        if legacy:
            shard = GpuShard(prob, shard_cfg(k_max=budget_gens, seed=seed), world, rank, TorchComm())
            eng, advance = shard.eng, shard.run
        else:
            eng = g.Engine(prob, shard_cfg(k_max=0, eval_budget=2 * n * budget_gens, seed=seed))
            advance = eng.step  # one CUDA graph per generation (NCCL inside it when sharded)
        advance(args.warmup)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        # ---- timed region: K generations, CUDA events on the engine's stream,
        # clocks sampled by NVML while it runs
        clocks = Clocks(local)
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clocks:
            start.record(stream)
            advance(args.steps)
            end.record(stream)
            torch.cuda.synchronize()
        eng.sync()  # raises the reference's evaluation error, if the run met it
        return eng, clocks, start.elapsed_time(end)

    (eng, clocks, ms_total), retries = retry_hazard(timed, dist)
    if dist:
        t = torch.tensor([ms_total], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = 2 * n / (ms_step * 1e-3)  # whole job: all ranks together process the N-slot generation
    # replacement rate over the timed generations (it drifts
    # over a run, so it is reported with the throughput); all ranks together
    rr = eng.replacement_rates()
    rep_rate = float(np.mean(rr[args.warmup + 1:args.warmup + 1 + args.steps]))
    # per-kernel device times (events around every launch, this rank's
    # engine, the exchange included), after the timed region
    kms = eng.profile(args.steps)
    info = eng.shard_info()

    # ---- e2e: the public API with (pinned) host buffers
    def pinned(shape):
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()

    rng = np.random.default_rng(7)
    X1, X2 = pinned((n, prob.d)), pinned((n, prob.d))
    X1[:] = prob.lower + (prob.upper - prob.lower) * rng.random((n, prob.d))
    X2[:] = prob.lower + (prob.upper - prob.lower) * rng.random((n, prob.d))
    recs = torch.zeros((args.steps, 16), dtype=torch.uint8, pin_memory=True).numpy()

    def end_to_end(seed):
        if legacy:
            sh2 = GpuShard(prob, shard_cfg(k_max=args.steps, seed=seed), world, rank, TorchComm())
            eng2, step1 = sh2.eng, sh2.step
        else:
            eng2 = g.Engine(prob, shard_cfg(k_max=args.steps, seed=seed))
            step1 = lambda: eng2.step(1)  # noqa: E731
        rows = eng2.rows_owned
        out = g.Population(pinned((rows, prob.d)), pinned((rows, prob.m)), pinned((rows, prob.n_constraints)),
                           pinned(rows))
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        eng2.set_population(1, X1)  # asynchronous: H2D + conversion + evaluation in stream order
        eng2.set_population(2, X2)
        if legacy:
            sh2._z_allreduce()
        # each step's result (the generation record: feasible count of the rank's
        # slots) is copied D2H into pinned memory in stream order, without a host
        # stall between steps; the host reads them after the final population copy
        for k in range(args.steps):
            step1()
            eng2.record_async(recs[k])
        pop = eng2.population(1, out=out)  # one synchronisation for the whole readback
        t1 = time.perf_counter()
        return eng2, pop, rows, t1 - t0

    (eng2, pop, rows, e2e_s), retries2 = retry_hazard(end_to_end, dist, first_seed=11)
    info2 = eng2.shard_info()
    feas = recs.view(np.uint32)[:, 0].astype(np.float64) / rows
    # bytes this rank copied: its parent window of each population in, its
    # owned rows of pop1 and the records out
    h2d = 2 * (info2["window_end"] - info2["window_begin"]) * prob.d * 8
    d2h = recs.nbytes + pop.X.nbytes + pop.F.nbytes + pop.C.nbytes + pop.cv.nbytes
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        b = torch.tensor([h2d, d2h], dtype=torch.float64)
        dist.all_reduce(b, op=dist.ReduceOp.SUM)
        h2d, d2h = (int(v) for v in b.tolist())
    e2e = {"value": 2 * n * args.steps / e2e_s, "unit": "ind-gen/s",
           "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
           "note": "pinned host buffers: set_population x2 (f64 H2D + evaluation, asynchronous) + K x (step + "
                   "async D2H of the step's generation record) + final pop1 (X, F, C, cv) D2H with one "
                   "synchronisation; host wall clock, max over ranks; bytes summed over ranks",
           "feasible_ratio_last": float(feas[-1])}
    eng2.close()

    if rank != 0:
        eng.close()
        if dist:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel, per rank (this rank's own rows)
    pk, pk_kind = peaks()
    ab = alg_bytes(prob.d, prob.m, prob.n_constraints, 5, 20)
    names = ["vary_eval", "op1", "select"]
    shares = {k: float(kms[i] / kms[4]) for i, k in enumerate(names)}
    dom = max(names, key=lambda k: kms[names.index(k)])
    di = names.index(dom)
    vary_rows = info["vary_end"] - info["vary_begin"]
    own_rows = info["own_end"] - info["own_begin"]
    units = {"vary_eval": 2 * vary_rows, "op1": vary_rows, "select": 2 * own_rows}[dom]
    per_unit = ab[dom] * (2 if dom == "op1" else 1)
    achieved = per_unit * units / (kms[di] * 1e-3) / 1e9
    traffic = ncu_traffic(dom, args.workload) if world == 1 else None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "peak_kind": pk_kind,
                "alg_bytes_per_unit": per_unit, "units_per_launch": units,
                "scope": "rank 0's kernel over its own rows" if world > 1 else "the whole run",
                "kernel_ms": {k: float(kms[i]) for i, k in enumerate(names)},
                "exchange_ms": float(kms[3]),
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

    extras = {}
    if world == 1 and not args.no_extras and args.workload == "lircmop13-1m":
        # the north-star's MW target (>= 1e8 ind-gen/s per B200 on MW at N = 1M)
        mp = g.make_problem("MW1")
        me = g.Engine(mp, g.RunConfig(n=1_000_000, k_max=0, eval_budget=2_000_000 * 64, seed=1, op=0,
                                      device=local, stream=stream.cuda_stream))
        mms = throughput(g, me, 20, 5, stream)
        mk = me.profile(5)
        me.close()
        mab = alg_bytes(mp.d, mp.m, mp.n_constraints, 5, 20)
        extras["mw1_1m"] = {"value": 2e6 / (mms * 1e-3), "unit": "ind-gen/s", "ms_per_step": mms, "steps": 20,
                            "warmup": 5, "vary_eval_ms": float(mk[0]),
                            "vary_eval_roofline_frac": mab["vary_eval"] * 2e6 / (mk[0] * 1e-3) / 1e9 / pk["hbm_gbs"],
                            "north_star_target": 1e8}
        extras["quality_1s"] = quality_1s(g)

    if legacy:
        config["functional_check"] = f"{world} ranks over {backend} on {torch.cuda.device_count()} GPU(s): not a bench number"
    elif world > 1:
        config["shards"] = f"{world} weight-region shards, NCCL z all-reduce + boundary-row send/recv in the generation graph"
    line = {"metric": METRIC, "value": value, "unit": "ind-gen/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong",  # N = 1M slots in total, split into weight-region shards
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (Philox-initialised populations)",
            "config": config, "replacement_rate": rep_rate, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks.summary(), "gpu_launches": int(3 * args.steps), **extras}
    if retries or retries2:
        line["hazard_retries"] = {"timed": retries, "e2e": retries2,
                                  "why": "the run met the reference's own evaluation error (PM hazard, "
                                         "gmpea.cpp:146-150); the next seed was measured"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
