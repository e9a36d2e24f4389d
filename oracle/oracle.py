"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU checkers built by oracle/Makefile:

* ``Oracle``   -> oracle/liboracle.so, the f64 plain-loop restatement
  (oracle/gmpea_oracle.cpp) of the reference hot path;
* ``Reference`` -> oracle/_ref/libgmpea_ref.so, the UNMODIFIED reference
  library compiled from /root/reference/proj/src plus a marshalling shim
  (oracle/ref_shim.cpp).  Present only where /root/reference was available
  at build time; ``Reference.available()`` says whether it can be loaded.

Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline / reference
arm import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgmpea_ref.so")

_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def build_oracle(force: bool = False) -> None:
    if force or not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def build_ref() -> bool:
    """Builds oracle/_ref from /root/reference when the sources are present."""
    if not os.path.isdir("/root/reference/proj/src"):
        return os.path.exists(REF_SO)
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    return True


class OracleError(RuntimeError):
    pass


class _Lib:
    prefix = ""

    def _check(self, rc):
        if rc != 0:
            msg = getattr(self.lib, self.prefix + "last_error")().decode()
            if rc == 1:
                raise ValueError(msg)
            raise OracleError(msg)


class Oracle(_Lib):
    prefix = "orc_"

    def __init__(self):
        build_oracle()
        lib = C.CDLL(ORACLE_SO)
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_pbi.restype = C.c_double
        lib.orc_cv.restype = C.c_double
        self.lib = lib

    # -- problems ---------------------------------------------------------
    def problem_info(self, name):
        d, m, nin, neq = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        self._check(self.lib.orc_problem_info(name.encode(), C.byref(d), C.byref(m), C.byref(nin),
                                              C.byref(neq), None, None))  # sizes first
        lo = np.zeros(d.value)
        hi = np.zeros(d.value)
        self._check(self.lib.orc_problem_info(name.encode(), C.byref(d), C.byref(m), C.byref(nin),
                                              C.byref(neq), _ptr(lo, _dp), _ptr(hi, _dp)))
        return dict(d=d.value, m=m.value, n_ineq=nin.value, n_eq=neq.value,
                    lo=lo[:d.value].copy(), hi=hi[:d.value].copy())

    def front_candidates(self, name, n_samples):
        """Restated MW / DAS-CMOP front candidates (decision rows)."""
        f = self.lib.orc_front_candidates
        f.restype = C.c_int64
        rows = f(name.encode(), C.c_int64(n_samples), None, C.c_int64(0))
        if rows < 0:
            raise OracleError(self.lib.orc_last_error().decode())
        d = self.problem_info(name)["d"]
        out = np.zeros((rows, d))
        f(name.encode(), C.c_int64(n_samples), _ptr(out, _dp), C.c_int64(out.size))
        return out

    def evaluate(self, name, X):
        info = self.problem_info(name)
        X = _f64(X)
        n = X.shape[0]
        nc = info["n_ineq"] + info["n_eq"]
        F = np.zeros((n, info["m"]))
        G = np.zeros((n, nc))
        cv = np.zeros(n)
        self._check(self.lib.orc_evaluate(name.encode(), _ptr(X, _dp), C.c_int64(n), _ptr(F, _dp),
                                          _ptr(G, _dp), _ptr(cv, _dp)))
        return F, G, cv

    def wta_register(self, scenario, targets, vehicles, strikes, capacity, p):
        """Registers a loaded scenario under the problem name "WTA-<scenario>"."""
        s = np.ascontiguousarray(strikes, np.int32)
        c = np.ascontiguousarray(capacity, np.int32)
        pv = _f64(p)
        self._check(self.lib.orc_wta_register(scenario.encode(), int(targets), int(vehicles), _ptr(s, _i32p),
                                              _ptr(c, _i32p), _ptr(pv, _dp)))

    def wta_scenario(self, num):
        t, v = C.c_int32(), C.c_int32()
        strikes = np.zeros(512, np.int32)
        cap = np.zeros(512, np.int32)
        p = np.zeros(2048)
        self._check(self.lib.orc_wta_scenario(num, C.byref(t), C.byref(v), _ptr(strikes, _i32p),
                                              _ptr(cap, _i32p), _ptr(p, _dp)))
        s = strikes[:t.value].copy()
        return dict(targets=t.value, vehicles=v.value, strikes=s, capacity=cap[:v.value].copy(),
                    p=p[:int(s.sum())].copy())

    # -- scalarization ----------------------------------------------------
    def pbi(self, f, w, z, theta=5.0):
        f, w, z = _f64(f), _f64(w), _f64(z)
        return self.lib.orc_pbi(_ptr(f, _dp), _ptr(w, _dp), _ptr(z, _dp), len(f), C.c_double(theta))

    def cv(self, raw, n_ineq, n_eq=0):
        raw = _f64(raw)
        return self.lib.orc_cv(_ptr(raw, _dp), int(n_ineq), int(n_eq))

    # -- topology ---------------------------------------------------------
    def reference_vectors(self, m, n):
        W = np.zeros((n, m))
        self._check(self.lib.orc_reference_vectors(m, C.c_int64(n), _ptr(W, _dp)))
        return W

    def knn(self, W, t):
        W = _f64(W)
        n, m = W.shape
        out = np.zeros((n, t), np.uint32)
        self._check(self.lib.orc_knn(_ptr(W, _dp), C.c_int64(n), m, t, _ptr(out, _u32p)))
        return out

    def knn_rows(self, W, rows, t, threads=0):
        """Brute-force t-NN of the given rows of W only (sampled parity at large N)."""
        W = _f64(W)
        n, m = W.shape
        rows = np.ascontiguousarray(rows, np.int64)
        out = np.zeros((len(rows), t), np.uint32)
        threads = threads or (os.cpu_count() or 1)
        self._check(self.lib.orc_knn_rows(_ptr(W, _dp), C.c_int64(n), m, t, _ptr(rows, _i64p), C.c_int64(len(rows)),
                                          _ptr(out, _u32p), threads))
        return out

    def lattice_knn(self, m, n, t1, t2, threads=0):
        B1 = np.zeros((n, t1), np.uint32)
        B2 = np.zeros((n, t2), np.uint32)
        threads = threads or (os.cpu_count() or 1)
        self._check(self.lib.orc_lattice_knn(m, C.c_int64(n), t1, t2, _ptr(B1, _u32p), _ptr(B2, _u32p), threads))
        return B1, B2

    # -- selection --------------------------------------------------------
    def selection(self, pops, W, z, theta, B1, B2, want_marks=False, agg=0):
        """pops = [pop1, pop2, off1, off2], each a dict with F (n x m), cv (n).
        agg: 0 = PBI (the reference's), 1 = Tchebycheff (engine extension).
        Returns (src1, src2[, marks1, marks2]); src = -1 parent kept,
        c in [0,n) off1 row c, n + c off2 row c."""
        F = [_f64(p["F"]) for p in pops]
        cv = [_f64(p["cv"]) for p in pops]
        n, m = F[0].shape
        W, z = _f64(W), _f64(z)
        B1 = np.ascontiguousarray(B1, np.uint32)
        B2 = np.ascontiguousarray(B2, np.uint32)
        t1, t2 = B1.shape[1], B2.shape[1]
        s1 = np.zeros(n, np.int32)
        s2 = np.zeros(n, np.int32)
        m1 = np.zeros((n, t1), np.uint8) if want_marks else None
        m2 = np.zeros((n, t2), np.uint8) if want_marks else None
        self._check(self.lib.orc_selection_ex(
            n, m, *[_ptr(a, _dp) for pair in zip(F, cv) for a in pair], _ptr(W, _dp), _ptr(z, _dp),
            C.c_double(theta), int(agg), t1, _ptr(B1, _u32p), t2, _ptr(B2, _u32p), _ptr(s1, _i32p),
            _ptr(s2, _i32p), _ptr(m1, _u8p), _ptr(m2, _u8p)))
        return (s1, s2, m1, m2) if want_marks else (s1, s2)

    # -- variation --------------------------------------------------------
    def reproduce(self, name, X, nb, op, seed, gen, pop, params=None, pm_prob=-1.0, slot_base=0):
        """op: 0 = sbx_pm, 1 = de.  params = (sbx_prob, sbx_eta, pm_eta, de_cr, de_f)."""
        X = _f64(X)
        nb = np.ascontiguousarray(nb, np.uint32)
        n, d = X.shape
        prm = _f64(params if params is not None else (1.0, 20.0, 20.0, 1.0, 0.5))
        off = np.zeros((n, d))
        picks = np.zeros((n, 3), np.int32)
        self._check(self.lib.orc_reproduce(name.encode(), _ptr(X, _dp), C.c_int64(n), _ptr(nb, _u32p),
                                           nb.shape[1], op, _ptr(prm, _dp), C.c_double(pm_prob),
                                           C.c_uint64(seed), C.c_uint32(gen), C.c_uint32(pop),
                                           _ptr(off, _dp), _ptr(picks, _i32p), C.c_uint32(slot_base)))
        return off, picks

    def run_gmpea(self, name, n, k_max, seed=1, op=0, fp32=False):
        """run_gmpea's loop in f64 with the engine's Philox draws (fp32=True:
        state rounded to fp32 after every step, as the engine stores it).
        Returns pop1 (X, F, cv)."""
        info = self.problem_info(name)
        X, F, cv = np.zeros((n, info["d"])), np.zeros((n, info["m"])), np.zeros(n)
        self._check(self.lib.orc_run_gmpea(name.encode(), C.c_int64(n), C.c_int64(k_max), C.c_uint64(seed), op,
                                           1 if fp32 else 0, _ptr(X, _dp), _ptr(F, _dp), _ptr(cv, _dp)))
        return X, F, cv

    def init_population(self, name, n, seed, pop):
        d = self.problem_info(name)["d"]
        X = np.zeros((n, d))
        self._check(self.lib.orc_init_population(name.encode(), C.c_int64(n), C.c_uint64(seed),
                                                 C.c_uint32(pop), _ptr(X, _dp)))
        return X

    def philox(self, ctr, key):
        c = np.ascontiguousarray(ctr, np.uint32)
        k = np.ascontiguousarray(key, np.uint32)
        o = np.zeros(4, np.uint32)
        self.lib.orc_philox(_ptr(c, _u32p), _ptr(k, _u32p), _ptr(o, _u32p))
        return o

    # -- metrics ----------------------------------------------------------
    def igd(self, A, R):
        A, R = _f64(A), _f64(R)
        out = C.c_double()
        self._check(self.lib.orc_igd(_ptr(A, _dp), C.c_int64(A.shape[0]), _ptr(R, _dp),
                                     C.c_int64(R.shape[0]), R.shape[1], C.byref(out)))
        return out.value

    def metric_front(self, F, cv):
        F, cv = _f64(F), _f64(cv)
        idx = np.zeros(F.shape[0], np.int64)
        cnt = C.c_int64()
        self._check(self.lib.orc_metric_front(_ptr(F, _dp), _ptr(cv, _dp), C.c_int64(F.shape[0]),
                                              F.shape[1], _ptr(idx, _i64p), C.byref(cnt)))
        return idx[:cnt.value]

    def hypervolume(self, P, ref):
        P, ref = _f64(P), _f64(ref)
        out = C.c_double()
        self._check(self.lib.orc_hypervolume(_ptr(P, _dp), C.c_int64(P.shape[0]), P.shape[1],
                                             _ptr(ref, _dp), C.byref(out)))
        return out.value


class Reference(_Lib):
    """The unmodified reference (oracle/_ref/libgmpea_ref.so)."""

    prefix = "ref_"

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        # the shim links the restated MW evaluators from the oracle sources
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_pbi.restype = C.c_double
        lib.ref_cv.restype = C.c_double
        self.lib = lib

    def problem_info(self, name):
        d, m, nin, neq = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        self._check(self.lib.ref_problem_info(name.encode(), C.byref(d), C.byref(m), C.byref(nin),
                                              C.byref(neq)))
        return dict(d=d.value, m=m.value, n_ineq=nin.value, n_eq=neq.value)

    def evaluate(self, name, X):
        info = self.problem_info(name)
        X = _f64(X)
        n = X.shape[0]
        F = np.zeros((n, info["m"]))
        G = np.zeros((n, info["n_ineq"] + info["n_eq"]))
        cv = np.zeros(n)
        self._check(self.lib.ref_evaluate(name.encode(), _ptr(X, _dp), C.c_int64(n), _ptr(F, _dp),
                                          _ptr(G, _dp), _ptr(cv, _dp)))
        return F, G, cv

    def wta_scenario(self, num):
        t, v = C.c_int32(), C.c_int32()
        strikes = np.zeros(64, np.int32)
        cap = np.zeros(64, np.int32)
        p = np.zeros(256)
        self._check(self.lib.ref_wta_scenario(num, C.byref(t), C.byref(v), _ptr(strikes, _i32p),
                                              _ptr(cap, _i32p), _ptr(p, _dp)))
        s = strikes[:t.value].copy()
        return dict(targets=t.value, vehicles=v.value, strikes=s, capacity=cap[:v.value].copy(),
                    p=p[:int(s.sum())].copy())

    def wta_file_evaluate(self, path, X, d, nc, m=2):
        """load_wta(path) -> make_wta_problem -> evaluate_population (the reference's own)."""
        X = _f64(X)
        n = X.shape[0]
        F, G, cv = np.zeros((n, m)), np.zeros((n, nc)), np.zeros(n)
        self._check(self.lib.ref_wta_file_evaluate(path.encode(), _ptr(X, _dp), C.c_int64(n), _ptr(F, _dp),
                                                   _ptr(G, _dp), _ptr(cv, _dp)))
        return F, G, cv

    def pbi(self, f, w, z, theta=5.0):
        f, w, z = _f64(f), _f64(w), _f64(z)
        return self.lib.ref_pbi(_ptr(f, _dp), _ptr(w, _dp), _ptr(z, _dp), len(f), C.c_double(theta))

    def cv(self, raw, n_ineq, n_eq=0):
        raw = _f64(raw)
        return self.lib.ref_cv(_ptr(raw, _dp), int(n_ineq), int(n_eq))

    def reference_vectors(self, m, n):
        W = np.zeros((n, m))
        self._check(self.lib.ref_reference_vectors(m, C.c_int64(n), _ptr(W, _dp)))
        return W

    def build_neighborhoods(self, W, t1, t2):
        W = _f64(W)
        n, m = W.shape
        B1 = np.zeros((n, t1), np.uint32)
        B2 = np.zeros((n, t2), np.uint32)
        self._check(self.lib.ref_build_neighborhoods(_ptr(W, _dp), C.c_int64(n), m, t1, t2,
                                                     _ptr(B1, _u32p), _ptr(B2, _u32p)))
        return B1, B2

    def _pop_arrays(self, pops):
        keep = []
        arrs = {}
        for key in ("X", "F", "C", "cv"):
            lst = [_f64(p[key]) for p in pops]
            keep.extend(lst)
            arr = (_dp * len(lst))(*[_ptr(a, _dp) for a in lst])
            arrs[key] = arr
        return keep, arrs

    def environmental_selection(self, pops, W, z, theta, B1, B2):
        keep, a = self._pop_arrays(pops)
        n, d = pops[0]["X"].shape
        m = pops[0]["F"].shape[1]
        nc = pops[0]["C"].shape[1]
        W, z = _f64(W), _f64(z)
        B1 = np.ascontiguousarray(B1, np.uint32)
        B2 = np.ascontiguousarray(B2, np.uint32)
        outs = [dict(X=np.zeros((n, d)), F=np.zeros((n, m)), C=np.zeros((n, nc)), cv=np.zeros(n))
                for _ in range(2)]
        o = {k: (_dp * 2)(*[_ptr(outs[i][k], _dp) for i in range(2)]) for k in ("X", "F", "C", "cv")}
        self._check(self.lib.ref_environmental_selection(
            C.c_int64(n), d, m, nc, a["X"], a["F"], a["C"], a["cv"], _ptr(W, _dp), _ptr(z, _dp),
            C.c_double(theta), B1.shape[1], _ptr(B1, _u32p), B2.shape[1], _ptr(B2, _u32p),
            o["X"], o["F"], o["C"], o["cv"]))
        return outs

    def op2_marks(self, pops, W, z, theta, B1, B2):
        keep, a = self._pop_arrays(pops)
        n, d = pops[0]["X"].shape
        m = pops[0]["F"].shape[1]
        nc = pops[0]["C"].shape[1]
        W, z = _f64(W), _f64(z)
        B1 = np.ascontiguousarray(B1, np.uint32)
        B2 = np.ascontiguousarray(B2, np.uint32)
        m1 = np.zeros(B1.shape, np.uint8)
        m2 = np.zeros(B2.shape, np.uint8)
        self._check(self.lib.ref_op2_marks(
            C.c_int64(n), d, m, nc, a["X"], a["F"], a["C"], a["cv"], _ptr(W, _dp), _ptr(z, _dp),
            C.c_double(theta), B1.shape[1], _ptr(B1, _u32p), B2.shape[1], _ptr(B2, _u32p),
            _ptr(m1, _u8p), _ptr(m2, _u8p)))
        return m1, m2

    def wilcoxon(self, a, b, alpha=0.05):
        a, b = _f64(a), _f64(b)
        p, d = C.c_double(), C.c_int32()
        self._check(self.lib.ref_wilcoxon(_ptr(a, _dp), C.c_int64(len(a)), _ptr(b, _dp), C.c_int64(len(b)),
                                          C.c_double(alpha), C.byref(p), C.byref(d)))
        return p.value, d.value

    def igd(self, A, R):
        A, R = _f64(A), _f64(R)
        out = C.c_double()
        self._check(self.lib.ref_igd(_ptr(A, _dp), C.c_int64(A.shape[0]), _ptr(R, _dp),
                                     C.c_int64(R.shape[0]), R.shape[1], C.byref(out)))
        return out.value

    def hypervolume(self, P, ref):
        P, ref = _f64(P), _f64(ref)
        out = C.c_double()
        self._check(self.lib.ref_hypervolume(_ptr(P, _dp), C.c_int64(P.shape[0]), P.shape[1],
                                             _ptr(ref, _dp), C.byref(out)))
        return out.value

    def metric_front(self, F, cv):
        F, cv = _f64(F), _f64(cv)
        out = np.zeros_like(F)
        rows = C.c_int64()
        self._check(self.lib.ref_metric_front(_ptr(F, _dp), _ptr(cv, _dp), C.c_int64(F.shape[0]),
                                              F.shape[1], _ptr(out, _dp), C.byref(rows)))
        return out[:rows.value]

    def pf_reference(self, name, npoints):
        cap = max(npoints, 1) * 4 + 100000
        out = np.zeros((cap, 3))
        rows = C.c_int64()
        m = self._info_any(name)["m"]
        out = np.zeros((cap, m))
        self._check(self.lib.ref_pf_reference(name.encode(), C.c_int64(npoints), _ptr(out, _dp),
                                              C.c_int64(cap), C.byref(rows)))
        return out[:rows.value].copy()

    def run_gmpea(self, name, n, k_max=0, seed=1, op=0, time_budget_s=-1.0, eval_budget=-1,
                  t1=5, t2=20, theta=5.0, record_walltime=True):
        info = self._info_any(name)
        X = np.zeros((n, info["d"]))
        F = np.zeros((n, info["m"]))
        Cm = np.zeros((n, info["n_ineq"] + info["n_eq"]))
        cv = np.zeros(n)
        cap = 1_000_000
        hist = np.zeros((cap, 4))
        rows = C.c_int64()
        self._check(self.lib.ref_run_gmpea(
            name.encode(), C.c_int64(n), C.c_int64(k_max), C.c_uint64(seed), op,
            C.c_double(time_budget_s), C.c_int64(eval_budget), t1, t2, C.c_double(theta),
            1 if record_walltime else 0, _ptr(X, _dp), _ptr(F, _dp), _ptr(Cm, _dp), _ptr(cv, _dp),
            _ptr(hist, _dp), C.c_int64(cap), C.byref(rows)))
        return dict(X=X, F=F, C=Cm, cv=cv), hist[:rows.value].copy()

    # -- comparison algorithms (baselines.hpp) --------------------------------
    def nondominated_sort(self, F, cv, use_cdp):
        F, cv = _f64(F), _f64(cv)
        n, m = F.shape
        rank = np.zeros(n, np.int64)
        self._check(self.lib.ref_nondominated_sort(_ptr(F, _dp), _ptr(cv, _dp), C.c_int64(n), m,
                                                   1 if use_cdp else 0, _ptr(rank, _i64p)))
        return rank

    def crowding_distance(self, F, front):
        F = _f64(F)
        n, m = F.shape
        fr = np.ascontiguousarray(front, np.int64)
        d = np.zeros(len(fr))
        self._check(self.lib.ref_crowding_distance(_ptr(F, _dp), C.c_int64(n), m, _ptr(fr, _i64p),
                                                   C.c_int64(len(fr)), _ptr(d, _dp)))
        return d

    def spea2_fitness(self, F, cv, use_cdp):
        F, cv = _f64(F), _f64(cv)
        n, m = F.shape
        fit = np.zeros(n)
        self._check(self.lib.ref_spea2_fitness(_ptr(F, _dp), _ptr(cv, _dp), C.c_int64(n), m,
                                               1 if use_cdp else 0, _ptr(fit, _dp)))
        return fit

    def spea2_select(self, F, cv, use_cdp, capacity):
        F, cv = _f64(F), _f64(cv)
        n, m = F.shape
        keep = np.zeros(max(n, 1), np.int64)
        cnt = C.c_int64()
        self._check(self.lib.ref_spea2_select(_ptr(F, _dp), _ptr(cv, _dp), C.c_int64(n), m, 1 if use_cdp else 0,
                                              C.c_int64(capacity), _ptr(keep, _i64p), C.byref(cnt)))
        return keep[:cnt.value].copy()

    def run_baseline(self, algo, name, n, k_max, seed=1):
        info = self._info_any(name)
        X = np.zeros((n, info["d"]))
        F = np.zeros((n, info["m"]))
        Cm = np.zeros((n, info["n_ineq"] + info["n_eq"]))
        cv = np.zeros(n)
        cap = 100_000
        hist = np.zeros((cap, 4))
        rows = C.c_int64()
        self._check(self.lib.ref_run_baseline({"cnsga2": 0, "ccmo": 1}[algo], name.encode(), C.c_int64(n),
                                              C.c_int64(k_max), C.c_uint64(seed), _ptr(X, _dp), _ptr(F, _dp),
                                              _ptr(Cm, _dp), _ptr(cv, _dp), _ptr(hist, _dp), C.c_int64(cap),
                                              C.byref(rows)))
        return dict(X=X, F=F, C=Cm, cv=cv), hist[:rows.value].copy()

    def _info_any(self, name):
        if name.startswith("MW") or name.startswith("DAS"):
            return Oracle().problem_info(name)
        return self.problem_info(name)

    def loop_bench(self, name, n, op, B1, B2, warmup, gens, replicas, seed=1):
        B1 = np.ascontiguousarray(B1, np.uint32)
        B2 = np.ascontiguousarray(B2, np.uint32)
        secs = np.zeros(replicas)
        self._check(self.lib.ref_loop_bench(name.encode(), C.c_int64(n), op, B1.shape[1],
                                            _ptr(B1, _u32p), B2.shape[1], _ptr(B2, _u32p), warmup,
                                            gens, replicas, C.c_uint64(seed), _ptr(secs, _dp)))
        return secs
