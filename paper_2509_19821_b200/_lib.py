"""ctypes bindings of libgmpea_b200.so and the Python mirror of the reference API."""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.environ.get("GMPEA_LIB") or os.path.join(HERE, "libgmpea_b200.so")

GMPEA_OK, GMPEA_EINVAL, GMPEA_ERUNTIME, GMPEA_ECUDA = 0, 1, 2, 3
GMPEA_OP_SBX_PM, GMPEA_OP_DE = 0, 1
GMPEA_AGG_PBI, GMPEA_AGG_TCH = 0, 1

_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


class CudaError(RuntimeError):
    """The CUDA runtime failed (or no device is present)."""


class _OpParams(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("sbx_prob", "sbx_eta", "pm_eta", "de_cr", "de_f", "pm_prob")]


class _View(C.Structure):
    _fields_ = [(k, _dp) for k in ("X", "F", "C", "cv")]


class _RunConfig(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("k_max", C.c_int64), ("time_budget_s", C.c_double),
        ("eval_budget", C.c_int64), ("seed", C.c_uint64), ("op", C.c_int32),
        ("params", _OpParams), ("theta", C.c_double), ("t1", C.c_int32), ("t2", C.c_int32),
        ("record_walltime", C.c_int32), ("device", C.c_int32), ("stream", C.c_uint64),
        ("igd_reference", _dp), ("igd_reference_rows", C.c_int64),
        ("shard_begin", C.c_int64), ("shard_end", C.c_int64), ("aggregation", C.c_int32),
        ("world", C.c_int32), ("rank", C.c_int32), ("nccl_id", C.c_void_p),
    ]


class _ShardInfo(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n_global", "window_begin", "window_end", "vary_begin", "vary_end",
                                         "own_begin", "own_end", "reach")]


class _DevBuffers(C.Structure):
    _fields_ = [("ideal_bits", C.c_void_p), ("rows", C.c_void_p * 2), ("keys", C.c_void_p * 2),
                ("row_bytes", C.c_int64)]


class _GenRecord(C.Structure):
    _fields_ = [("gen", C.c_int64), ("evals", C.c_int64), ("wall_ms", C.c_double),
                ("feasible_ratio", C.c_double), ("igd", C.c_double), ("hv", C.c_double),
                ("has_igd", C.c_int32), ("has_hv", C.c_int32)]


def _load():
    if not os.path.exists(LIB):
        raise ImportError(
            f"{LIB} is missing: build it with `python -m paper_2509_19821_b200.build` "
            "(the engine has no CPU fallback)")
    lib = C.CDLL(LIB)
    lib.gmpea_last_error.restype = C.c_char_p
    lib.gmpea_problem_names.restype = C.c_char_p
    lib.gmpea_engine_effective_n.restype = C.c_int64
    lib.gmpea_problem_destroy.restype = None
    lib.gmpea_engine_destroy.restype = None
    return lib


_L = _load()


def lib_path() -> str:
    return LIB


def _check(rc: int) -> None:
    if rc == GMPEA_OK:
        return
    msg = _L.gmpea_last_error().decode()
    if rc == GMPEA_EINVAL:
        raise ValueError(msg)
    if rc == GMPEA_ECUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a: Optional[np.ndarray], t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


# --------------------------------------------------------------------- problems
class Problem:
    """A registered benchmark problem living on the device (ProblemDef,
    problems.hpp:19-37)."""

    def __init__(self, handle, name: str):
        self._h = handle
        self.name = name
        d, m, nin, neq = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(_L.gmpea_problem_info(handle, C.byref(d), C.byref(m), C.byref(nin), C.byref(neq)))
        self.d, self.m, self.n_ineq, self.n_eq = d.value, m.value, nin.value, neq.value
        lo = np.zeros(self.d)
        hi = np.zeros(self.d)
        _check(_L.gmpea_problem_bounds(handle, _p(lo), _p(hi)))
        self.bounds = list(zip(lo.tolist(), hi.tolist()))
        self.lower, self.upper = lo, hi

    @property
    def n_constraints(self) -> int:
        return self.n_ineq + self.n_eq

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _L.gmpea_problem_destroy(h)
            self._h = None

    def __repr__(self):
        return f"Problem({self.name!r}, d={self.d}, m={self.m}, n_ineq={self.n_ineq})"


def make_problem(name: str) -> Problem:
    h = C.c_void_p()
    _check(_L.gmpea_problem_create(name.encode(), C.byref(h)))
    return Problem(h, name)


def make_wta_problem(scenario: str, targets: int, vehicles: int, strikes: Sequence[int],
                     capacity: Sequence[int], p: Sequence[float]) -> Problem:
    """A WTA scenario from explicit tables (load_wta + make_wta_problem, wta.cpp:112-192)."""
    s = np.ascontiguousarray(strikes, np.int32)
    c = np.ascontiguousarray(capacity, np.int32)
    pv = _f64(p)
    h = C.c_void_p()
    _check(_L.gmpea_problem_create_wta(scenario.encode(), targets, vehicles, _p(s, _i32p), _p(c, _i32p),
                                       _p(pv), C.byref(h)))
    return Problem(h, "WTA-" + scenario)


def problem_names() -> List[str]:
    return [n for n in _L.gmpea_problem_names().decode().split("\n") if n]


# --------------------------------------------------------------------- populations
@dataclasses.dataclass
class Population:
    """Paired X (N x d), F (N x m), raw constraints C (N x nc) and cv (N)
    (gmpea.hpp:23-30)."""

    X: np.ndarray
    F: np.ndarray
    C: np.ndarray
    cv: np.ndarray

    def size(self) -> int:
        return int(self.X.shape[0])

    def copy(self) -> "Population":
        return Population(self.X.copy(), self.F.copy(), self.C.copy(), self.cv.copy())


@dataclasses.dataclass
class EvalResult:
    F: np.ndarray
    G: np.ndarray


def _evaluate(problem: Problem, X):
    X = _f64(X)
    if X.ndim != 2 or X.shape[1] != problem.d:
        raise ValueError("evaluate: wrong decision dimension")
    n = X.shape[0]
    F = np.zeros((n, problem.m))
    G = np.zeros((n, problem.n_constraints))
    cv = np.zeros(n)
    _check(_L.gmpea_evaluate(problem._h, _p(X), C.c_int64(n), _p(F), _p(G), _p(cv)))
    return X, F, G, cv


def evaluate(problem: Problem, X) -> EvalResult:
    _, F, G, _ = _evaluate(problem, X)
    return EvalResult(F, G)


def evaluate_population(problem: Problem, X) -> Population:
    X, F, G, cv = _evaluate(problem, X)
    return Population(X, F, G, cv)


# --------------------------------------------------------------------- topology
@dataclasses.dataclass
class NeighborhoodTopology:
    b1: np.ndarray  # N x t1, uint32
    b2: np.ndarray  # N x t2
    t1: int
    t2: int


def reference_vectors(m: int, target_n: int) -> np.ndarray:
    if target_n <= 0:
        raise ValueError("reference_vectors: target_n must be positive")
    W = np.zeros((target_n, m))
    _check(_L.gmpea_reference_vectors(m, C.c_int64(target_n), _p(W)))
    return W


def build_neighborhoods(W, t1: int, t2: int) -> NeighborhoodTopology:
    W = _f64(W)
    n, m = W.shape
    B1 = np.zeros((n, t1), np.uint32)
    B2 = np.zeros((n, t2), np.uint32)
    _check(_L.gmpea_build_neighborhoods(_p(W), C.c_int64(n), m, t1, t2, _p(B1, _u32p), _p(B2, _u32p)))
    return NeighborhoodTopology(B1, B2, t1, t2)


def lattice_neighborhoods(m: int, n: int, t1: int, t2: int) -> NeighborhoodTopology:
    """build_neighborhoods(reference_vectors(m, n), t1, t2) without forming W on the host."""
    B1 = np.zeros((n, t1), np.uint32)
    B2 = np.zeros((n, t2), np.uint32)
    _check(_L.gmpea_lattice_neighborhoods(m, C.c_int64(n), t1, t2, _p(B1, _u32p), _p(B2, _u32p)))
    return NeighborhoodTopology(B1, B2, t1, t2)


# --------------------------------------------------------------------- operators
class VariationOp(enum.IntEnum):
    sbx_pm = GMPEA_OP_SBX_PM
    de = GMPEA_OP_DE


@dataclasses.dataclass
class OperatorParams:
    """OperatorParams (gmpea.hpp:58-66); pm_prob None means 1/d."""

    sbx_prob: float = 1.0
    sbx_eta: float = 20.0
    pm_eta: float = 20.0
    de_cr: float = 1.0
    de_f: float = 0.5
    pm_prob: Optional[float] = None

    def _c(self) -> _OpParams:
        return _OpParams(self.sbx_prob, self.sbx_eta, self.pm_eta, self.de_cr, self.de_f,
                         -1.0 if self.pm_prob is None else float(self.pm_prob))


def reproduce(pop: Population, neighborhoods, problem: Problem, op=VariationOp.sbx_pm,
              params: Optional[OperatorParams] = None, *, seed: int = 1, gen: int = 1,
              pop_id: int = 1) -> np.ndarray:
    """One offspring per subproblem from its own neighbourhood row
    (gmpea.cpp:169-206).  The reference's Rng& is replaced by the Philox key
    (seed, gen, pop_id)."""
    X = _f64(pop.X if isinstance(pop, Population) else pop)
    nb = np.ascontiguousarray(neighborhoods, np.uint32)
    n = X.shape[0]
    if nb.shape[0] != n:
        raise ValueError("reproduce: topology/population mismatch")
    off = np.zeros_like(X)
    prm = (params or OperatorParams())._c()
    _check(_L.gmpea_reproduce(problem._h, _p(X), C.c_int64(n), _p(nb, _u32p), nb.shape[1], int(op),
                              C.byref(prm), C.c_uint64(seed), C.c_uint32(gen), C.c_uint32(pop_id),
                              _p(off)))
    return off


class Aggregation(enum.IntEnum):
    """Subproblem aggregation: PBI (scalarize.cpp:72-89, the reference's) or
    the weighted Tchebycheff function max_k max(w_k, 1e-6)|f_k - z_k| (an
    engine extension the reference does not have; parity vs the oracle)."""

    pbi = GMPEA_AGG_PBI
    tchebycheff = GMPEA_AGG_TCH


@dataclasses.dataclass
class SelectionContext:
    """SelectionContext{W, z, theta} (gmpea.hpp:75-79) plus the aggregation."""

    W: np.ndarray
    z: np.ndarray
    theta: float = 5.0
    aggregation: Aggregation = Aggregation.pbi


def _view(p: Population, keep: list) -> _View:
    arrs = [_f64(p.X), _f64(p.F), _f64(p.C), _f64(p.cv)]
    keep.extend(arrs)
    return _View(*[_p(a) for a in arrs])


def environmental_selection(pop1: Population, pop2: Population, off1: Population, off2: Population,
                            topo: NeighborhoodTopology, ctx: SelectionContext, *,
                            return_winners: bool = False):
    """OP1 -> OP2 -> OP3 (gmpea.cpp:392-399).  Returns the next (pop1, pop2);
    with return_winners also the per-slot source codes (-1 parent, c off1
    row c, n + c off2 row c)."""
    n, d = pop1.X.shape
    m = pop1.F.shape[1]
    nc = pop1.C.shape[1]
    keep: list = []
    v = [_view(p, keep) for p in (pop1, pop2, off1, off2)]
    outs = [Population(np.zeros((n, d)), np.zeros((n, m)), np.zeros((n, nc)), np.zeros(n)) for _ in range(2)]
    ov = [_View(*[_p(a) for a in (o.X, o.F, o.C, o.cv)]) for o in outs]
    W, z = _f64(ctx.W), _f64(ctx.z)
    B1 = np.ascontiguousarray(topo.b1, np.uint32)
    B2 = np.ascontiguousarray(topo.b2, np.uint32)
    w1 = np.zeros(n, np.int32)
    w2 = np.zeros(n, np.int32)
    _check(_L.gmpea_environmental_selection_ex(
        C.c_int64(n), d, m, nc, C.byref(v[0]), C.byref(v[1]), C.byref(v[2]), C.byref(v[3]), _p(W), _p(z),
        C.c_double(ctx.theta), int(ctx.aggregation), _p(B1, _u32p), B1.shape[1], _p(B2, _u32p), B2.shape[1], C.byref(ov[0]),
        C.byref(ov[1]), _p(w1, _i32p), _p(w2, _i32p)))
    if return_winners:
        return outs[0], outs[1], w1, w2
    return outs[0], outs[1]


# --------------------------------------------------------------------- metrics
def igd(approx, reference) -> float:
    A, R = _f64(approx), _f64(reference)
    if A.ndim != 2:
        A = A.reshape(0, R.shape[1])
    if A.shape[0] and A.shape[1] != R.shape[1]:
        raise ValueError("igd: objective count mismatch")
    out = C.c_double()
    _check(_L.gmpea_igd(_p(A), C.c_int64(A.shape[0]), _p(R), C.c_int64(R.shape[0]), R.shape[1], C.byref(out)))
    return out.value


def metric_front(pop: Population) -> np.ndarray:
    """Feasible, deduplicated, mutually nondominated rows of pop.F (metrics.cpp:155-175)."""
    F, cv = _f64(pop.F), _f64(pop.cv)
    idx = np.zeros(F.shape[0], np.int64)
    cnt = C.c_int64()
    _check(_L.gmpea_metric_front(_p(F), _p(cv), C.c_int64(F.shape[0]), F.shape[1], _p(idx, _i64p), C.byref(cnt)))
    return F[idx[:cnt.value]]


def hypervolume(points, ref_point) -> float:
    P, r = _f64(points), _f64(ref_point)
    if P.ndim == 2 and P.shape[0] and P.shape[1] != r.shape[0]:
        raise ValueError("hypervolume: reference dimension mismatch")
    out = C.c_double()
    _check(_L.gmpea_hypervolume(_p(P), C.c_int64(P.shape[0] if P.ndim == 2 else 0), r.shape[0], _p(r),
                                C.byref(out)))
    return out.value


def pf_reference(problem: "Problem", n_points: int = 1000) -> np.ndarray:
    """pf_reference (fronts.cpp:54-84): the analytic Pareto front sampled to
    n_points rows, built and evaluated in fp64 on the device.  MW and
    DAS-CMOP (restated suites) get restated front candidates: each position's
    smallest feasible distance, found by a level scan and bisection.
    RuntimeError for WTA (no analytic front), as the reference."""
    cap = max(int(n_points), 1)
    out = np.zeros((cap, problem.m))
    rows = C.c_int64()
    rc = _L.gmpea_pf_reference(problem._h, C.c_int64(n_points), _p(out), C.c_int64(cap), C.byref(rows))
    if rc == GMPEA_EINVAL and "capacity" in _L.gmpea_last_error().decode():
        # a front smaller than requested never exceeds n_points; only a
        # retried, unsubsampled front can (fronts.cpp:76)
        cap = 4 * 50000 + 100000
        out = np.zeros((cap, problem.m))
        rc = _L.gmpea_pf_reference(problem._h, C.c_int64(n_points), _p(out), C.c_int64(cap), C.byref(rows))
    _check(rc)
    return out[:rows.value].copy()


# ------------------------------------------------ comparison-algorithm operators
def nondominated_sort(F, cv, use_cdp: bool = True) -> np.ndarray:
    """nondominated_sort (baselines.cpp:22-55): 0-based front rank per row."""
    F, cv = _f64(F), _f64(cv)
    n, m = F.shape
    rank = np.zeros(n, np.int64)
    _check(_L.gmpea_nondominated_sort(_p(F), _p(cv), C.c_int64(n), m, int(bool(use_cdp)), _p(rank, _i64p)))
    return rank


def crowding_distance(F, front) -> np.ndarray:
    """crowding_distance (baselines.cpp:56-91) of the rows `front` of F."""
    F = _f64(F)
    n, m = F.shape
    fr = np.ascontiguousarray(front, np.int64)
    d = np.zeros(len(fr))
    _check(_L.gmpea_crowding_distance(_p(F), C.c_int64(n), m, _p(fr, _i64p), C.c_int64(len(fr)), _p(d)))
    return d


def spea2_fitness(F, cv, use_cdp: bool = True) -> np.ndarray:
    """spea2_fitness (baselines.cpp:93-127)."""
    F, cv = _f64(F), _f64(cv)
    n, m = F.shape
    fit = np.zeros(n)
    _check(_L.gmpea_spea2_fitness(_p(F), _p(cv), C.c_int64(n), m, int(bool(use_cdp)), _p(fit)))
    return fit


def spea2_select(F, cv, use_cdp: bool, capacity: int) -> np.ndarray:
    """spea2_select (baselines.cpp:129-189): kept row indices, ascending."""
    F, cv = _f64(F), _f64(cv)
    n, m = F.shape
    keep = np.zeros(max(n, 1), np.int64)
    cnt = C.c_int64()
    _check(_L.gmpea_spea2_select(_p(F), _p(cv), C.c_int64(n), m, int(bool(use_cdp)), C.c_int64(capacity),
                                 _p(keep, _i64p), C.byref(cnt)))
    return keep[:cnt.value].copy()


# --------------------------------------------------------------------- the run
@dataclasses.dataclass
class RunConfig:
    """RunConfig (gmpea.hpp:113-127) plus engine placement."""

    n: int = 100
    k_max: int = 0
    time_budget_s: Optional[float] = None
    eval_budget: Optional[int] = None
    seed: int = 1
    op: VariationOp = VariationOp.sbx_pm
    op_params: OperatorParams = dataclasses.field(default_factory=OperatorParams)
    theta: float = 5.0
    t1: int = 5
    t2: int = 20
    record_walltime: bool = True
    device: int = 0
    stream: int = 0
    shard: Optional[tuple] = None  # (begin, end) owned slots of a caller-driven sharded run
    aggregation: Aggregation = Aggregation.pbi
    # weight-region shards over NCCL, one process per GPU: this
    # rank of `world`, with the 128-byte id of nccl_unique_id() from rank 0
    world: int = 0
    rank: int = 0
    nccl_id: Optional[bytes] = None
    # the per-generation IGD hook (RunConfig::igd_metric as experiment.cpp:200-205
    # installs it): igd(metric_front(pop1), igd_reference) on the device
    igd_reference: Optional[np.ndarray] = None

    def _c(self) -> _RunConfig:
        c = _RunConfig()
        _check(_L.gmpea_run_config_default(C.byref(c)))
        c.n = self.n
        c.k_max = self.k_max
        c.time_budget_s = -1.0 if self.time_budget_s is None else float(self.time_budget_s)
        c.eval_budget = -1 if self.eval_budget is None else int(self.eval_budget)
        c.seed = self.seed
        c.op = int(self.op)
        c.params = self.op_params._c()
        c.theta = self.theta
        c.t1, c.t2 = self.t1, self.t2
        c.record_walltime = 1 if self.record_walltime else 0
        c.device = self.device
        c.stream = self.stream
        if self.shard is not None:
            c.shard_begin, c.shard_end = int(self.shard[0]), int(self.shard[1])
        c.aggregation = int(self.aggregation)
        c.world, c.rank = int(self.world), int(self.rank)
        if self.igd_reference is not None:
            self._igd_ref = _f64(self.igd_reference)  # kept alive with the config (copied at create)
            c.igd_reference = _p(self._igd_ref)
            c.igd_reference_rows = self._igd_ref.shape[0]
        if self.nccl_id is not None:
            if len(self.nccl_id) != 128:
                raise ValueError("nccl_id: 128 bytes expected")
            self._nccl_buf = C.create_string_buffer(bytes(self.nccl_id), 128)  # kept alive with the config
            c.nccl_id = C.cast(self._nccl_buf, C.c_void_p)
        return c


@dataclasses.dataclass
class GenRecord:
    gen: int
    evals: int
    wall_ms: float
    feasible_ratio: float
    igd: Optional[float] = None
    hv: Optional[float] = None


@dataclasses.dataclass
class RunResult:
    pop1: Population
    history: List[GenRecord]
    effective_n: int


def nccl_unique_id() -> bytes:
    """A new NCCL unique id for RunConfig.nccl_id (rank 0 makes it, the caller
    shares it with the other ranks)."""
    buf = C.create_string_buffer(128)
    _check(_L.gmpea_nccl_unique_id(buf))
    return buf.raw


class Engine:
    """One run (the engine behind run_gmpea): on one device, one NCCL rank of a
    sharded run (cfg.world / rank / nccl_id), or -- with devices -- one handle
    driving a sharded run over several devices of this process."""

    def __init__(self, problem: Problem, cfg: RunConfig, devices: Optional[Sequence[int]] = None):
        self.problem = problem
        self.cfg = cfg
        self._c = cfg._c()
        h = C.c_void_p()
        if devices is not None:
            dv = np.ascontiguousarray(devices, np.int32)
            _check(_L.gmpea_engine_create_multi(problem._h, C.byref(self._c), _p(dv, _i32p), len(dv), C.byref(h)))
        else:
            _check(_L.gmpea_engine_create(problem._h, C.byref(self._c), C.byref(h)))
        self._h = h
        self.n = int(_L.gmpea_engine_effective_n(h))
        info = self.shard_info()
        self.rows_owned = info["own_end"] - info["own_begin"]  # rows population() returns

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _L.gmpea_engine_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    def set_population(self, which: int, X) -> None:
        X = _f64(X)
        if X.shape != (self.n, self.problem.d):
            raise ValueError("set_population: shape mismatch")
        _check(_L.gmpea_engine_set_population(self._h, which, _p(X)))

    def run(self) -> None:
        _check(_L.gmpea_engine_run(self._h))

    def step(self, gens: int) -> None:
        _check(_L.gmpea_engine_step(self._h, C.c_int64(gens)))

    def sync(self) -> None:
        _check(_L.gmpea_engine_sync(self._h))

    def history(self) -> List[GenRecord]:
        cnt = C.c_int64()
        _check(_L.gmpea_engine_history(self._h, None, 0, C.byref(cnt)))
        buf = (_GenRecord * cnt.value)()
        _check(_L.gmpea_engine_history(self._h, buf, cnt.value, C.byref(cnt)))
        return [GenRecord(r.gen, r.evals, r.wall_ms, r.feasible_ratio,
                          r.igd if r.has_igd else None, r.hv if r.has_hv else None) for r in buf]

    def replacement_rates(self) -> np.ndarray:
        """per generation: share of the owned slots of both populations that
        took an offspring in OP3 (entry 0, initialisation, is 0)."""
        cnt = C.c_int64()
        _check(_L.gmpea_engine_replacements(self._h, None, 0, C.byref(cnt)))
        buf = np.zeros(cnt.value, np.int64)
        _check(_L.gmpea_engine_replacements(self._h, buf.ctypes.data_as(C.POINTER(C.c_int64)), cnt.value,
                                            C.byref(cnt)))
        return buf / (2.0 * self.rows_owned)

    def record_async(self, dst: np.ndarray) -> None:
        """Enqueue a copy of the newest generation's raw record (16 bytes:
        feasible u32, replaced u32, loop_ns u64) into dst without waiting;
        dst should be pinned (e.g. torch pinned memory viewed as numpy) and
        is valid after the next sync()."""
        if dst.nbytes < 16 or not dst.flags["C_CONTIGUOUS"]:
            raise ValueError("record_async: need 16 contiguous bytes")
        _check(_L.gmpea_engine_record_async(self._h, C.c_void_p(dst.ctypes.data)))

    def last_record(self) -> GenRecord:
        r = _GenRecord()
        _check(_L.gmpea_engine_last_record(self._h, C.byref(r)))
        return GenRecord(r.gen, r.evals, r.wall_ms, r.feasible_ratio)

    def population(self, which: int = 1, out: Optional[Population] = None) -> Population:
        """pop `which` as f64 rows; `out` may supply (pinned) destination arrays."""
        n, p = self.rows_owned, self.problem
        if out is None:
            out = Population(np.zeros((n, p.d)), np.zeros((n, p.m)), np.zeros((n, p.n_constraints)), np.zeros(n))
        _check(_L.gmpea_engine_get_population(self._h, which, _p(out.X), _p(out.F), _p(out.C), _p(out.cv)))
        return out

    def offspring(self, which: int = 1, out: Optional[Population] = None) -> Population:
        """Diagnostic: offspring stream `which` of the last generation as
        variation + evaluation produced it (before OP1)."""
        n, p = self.rows_owned, self.problem
        if out is None:
            out = Population(np.zeros((n, p.d)), np.zeros((n, p.m)), np.zeros((n, p.n_constraints)), np.zeros(n))
        _check(_L.gmpea_engine_get_offspring(self._h, which, _p(out.X), _p(out.F), _p(out.C), _p(out.cv)))
        return out

    def ideal(self) -> np.ndarray:
        z = np.zeros(self.problem.m)
        _check(_L.gmpea_engine_ideal(self._h, _p(z)))
        return z

    def neighborhoods(self) -> NeighborhoodTopology:
        t1, t2 = min(self.cfg.t1, self.n), min(self.cfg.t2, self.n)
        B1 = np.zeros((self.rows_owned, t1), np.uint32)
        B2 = np.zeros((self.rows_owned, t2), np.uint32)
        _check(_L.gmpea_engine_neighborhoods(self._h, _p(B1, _u32p), _p(B2, _u32p)))
        return NeighborhoodTopology(B1, B2, t1, t2)

    # ---- sharded runs
    def shard_info(self) -> dict:
        o = _ShardInfo()
        _check(_L.gmpea_engine_shard_info(self._h, C.byref(o)))
        return {k: getattr(o, k) for k, _ in _ShardInfo._fields_}

    def phase(self, ph: int) -> None:
        _check(_L.gmpea_engine_phase(self._h, ph))

    def device_buffers(self) -> dict:
        o = _DevBuffers()
        _check(_L.gmpea_engine_device_buffers(self._h, C.byref(o)))
        return {"ideal_bits": o.ideal_bits, "rows": [o.rows[0], o.rows[1]], "keys": [o.keys[0], o.keys[1]],
                "row_bytes": o.row_bytes}

    def profile(self, gens: int) -> np.ndarray:
        """Per-kernel average device ms: [vary_eval, op1, select, end_gen, total]."""
        ms = np.zeros(5)
        _check(_L.gmpea_engine_profile(self._h, C.c_int64(gens), _p(ms)))
        return ms


BASELINE_ALGORITHMS = {"cnsga2": 0, "ccmo": 1}


def run_baseline(problem: Problem, algorithm: str, cfg: RunConfig,
                 igd_front: Optional[np.ndarray] = None) -> RunResult:
    """run_cnsga2 / run_ccmo (baselines.cpp:320-459) on the device; with
    igd_front the per-generation IGD hook runs on the device too."""
    if algorithm not in BASELINE_ALGORITHMS:
        raise ValueError("unknown algorithm: " + algorithm)
    c = cfg._c()
    n, p = cfg.n, problem
    X, F = np.zeros((n, p.d)), np.zeros((n, p.m))
    Cm, cv = np.zeros((n, p.n_constraints)), np.zeros(n)
    ref = None if igd_front is None else _f64(igd_front)
    nref = 0 if ref is None else ref.shape[0]
    nh = C.c_int64()
    bounded = not cfg.eval_budget and not cfg.time_budget_s
    cap = max(cfg.k_max, 0) + 2 if bounded else (cfg.eval_budget // n + 2 if cfg.eval_budget and not cfg.time_budget_s
                                                 else 1 << 20)
    buf = (_GenRecord * cap)()
    _check(_L.gmpea_run_baseline(problem._h, BASELINE_ALGORITHMS[algorithm], C.byref(c),
                                 _p(ref) if ref is not None else None, C.c_int64(nref), None, None, buf, C.c_int64(cap),
                                 C.byref(nh), _p(X), _p(F), _p(Cm), _p(cv)))
    hist = [GenRecord(r.gen, r.evals, r.wall_ms, r.feasible_ratio,
                      r.igd if r.has_igd else None, r.hv if r.has_hv else None) for r in buf[:min(nh.value, cap)]]
    return RunResult(Population(X, F, Cm, cv), hist, n)


def run_gmpea(problem: Problem, cfg: RunConfig) -> RunResult:
    """run_gmpea (gmpea.cpp:421-493) on the device."""
    eng = Engine(problem, cfg)
    try:
        eng.run()
        return RunResult(eng.population(1), eng.history(), eng.n)
    finally:
        eng.close()
