// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library, compiled together
// with the reference's own sources where they lie (/root/reference/proj/src)
// by oracle/Makefile into oracle/_ref/libgmpea_ref.so (git-ignored).  Nothing
// from the reference is copied into this repo; this file only marshals plain
// arrays into the reference's public API (proj/include/gmpea/*.hpp):
//   evaluate / evaluate_population (problems.hpp:47-51, gmpea.hpp:33)
//   reference_vectors / build_neighborhoods (gmpea.hpp:37-51)
//   op1/op2/op3/environmental_selection (gmpea.hpp:84-111)
//   reproduce / update_ideal (gmpea.hpp:54,70-73)
//   igd / hypervolume / metric_front (metrics.hpp:15-29), pf_reference
//   run_gmpea (gmpea.hpp:144)
// plus ref_loop_bench: the reference's own loop body (gmpea.cpp:457-489, the
// same public calls in the same order) with an injected neighbourhood
// topology, used as the CPU baseline at population sizes where the
// reference's O(N^2 log N) build_neighborhoods is impractical.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "gmpea/baselines.hpp"
#include "gmpea/gmpea.hpp"
#include "gmpea/metrics.hpp"
#include "gmpea/problems.hpp"
#include "gmpea/scalarize.hpp"
#include "gmpea/wta.hpp"

using namespace gmpea;

extern "C" {
void* orc_problem_new(const char* name);
void orc_problem_free(void* h);
void orc_problem_eval_row(const void* h, const double* x, double* f, double* g);
int64_t orc_problem_front_rows(const void* h, int64_t n_samples);
void orc_problem_front_candidates(const void* h, int64_t n_samples, double* out);
int orc_problem_info(const char* name, int32_t* d, int32_t* m, int32_t* nin, int32_t* neq,
                     double* lo, double* hi);
}

namespace {
thread_local std::string g_err;

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Matrix mat(const double* p, std::size_t r, std::size_t c) {
    Matrix M(r, c);
    if (r * c) std::memcpy(M.data.data(), p, r * c * sizeof(double));
    return M;
}

void put(const Matrix& M, double* out) {
    if (out && !M.data.empty()) std::memcpy(out, M.data.data(), M.data.size() * sizeof(double));
}

Population popn(const double* X, const double* F, const double* C, const double* cv, std::size_t n,
                std::size_t d, std::size_t m, std::size_t nc) {
    Population p;
    p.X = mat(X, n, d);
    p.F = mat(F, n, m);
    p.C = mat(C, n, nc);
    p.cv.assign(cv, cv + n);
    return p;
}

void unpop(const Population& p, double* X, double* F, double* C, double* cv) {
    put(p.X, X);
    put(p.F, F);
    put(p.C, C);
    if (cv) std::copy(p.cv.begin(), p.cv.end(), cv);
}

NeighborhoodTopology topo_of(const uint32_t* B1, std::size_t t1, const uint32_t* B2,
                             std::size_t t2, std::size_t n) {
    NeighborhoodTopology t;
    t.t1 = t1;
    t.t2 = t2;
    t.b1.resize(n);
    t.b2.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        t.b1[i].assign(B1 + i * t1, B1 + (i + 1) * t1);
        t.b2[i].assign(B2 + i * t2, B2 + (i + 1) * t2);
    }
    return t;
}

// reference problems, or (for MW* / DAS-CMOP*) the oracle's restated evaluator
// wrapped as a reference ProblemDef so the reference loop can run it
ProblemDef problem_for(const std::string& name) {
    if (name.rfind("MW", 0) != 0 && name.rfind("DAS", 0) != 0) return make_problem(name);
    int32_t d, m, nin, neq;
    std::vector<double> lo(64), hi(64);
    if (orc_problem_info(name.c_str(), &d, &m, &nin, &neq, lo.data(), hi.data()) != 0)
        throw std::invalid_argument("unknown problem: " + name);
    ProblemDef p;
    p.name = name;
    p.d = d;
    p.m = m;
    p.n_ineq = nin;
    p.n_eq = neq;
    for (int j = 0; j < d; ++j) p.bounds.emplace_back(lo[j], hi[j]);
    std::shared_ptr<void> h(orc_problem_new(name.c_str()), orc_problem_free);
    p.eval_row = [h](std::span<const double> x, std::span<double> f, std::span<double> g) {
        orc_problem_eval_row(h.get(), x.data(), f.data(), g.data());
    };
    // the oracle's restated front candidates (no reference counterpart)
    p.front_candidates = [h, d](std::size_t n_samples) {
        const int64_t rows = orc_problem_front_rows(h.get(), static_cast<int64_t>(n_samples));
        Matrix M(static_cast<std::size_t>(rows), static_cast<std::size_t>(d));
        orc_problem_front_candidates(h.get(), static_cast<int64_t>(n_samples), M.data.data());
        return M;
    };
    return p;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_problem_info(const char* name, int32_t* d, int32_t* m, int32_t* nin, int32_t* neq) {
    return guarded([&] {
        ProblemDef p = make_problem(name);
        *d = static_cast<int32_t>(p.d);
        *m = static_cast<int32_t>(p.m);
        *nin = static_cast<int32_t>(p.n_ineq);
        *neq = static_cast<int32_t>(p.n_eq);
    });
}

int ref_evaluate(const char* name, const double* X, int64_t n, double* F, double* G, double* cv) {
    return guarded([&] {
        ProblemDef p = make_problem(name);
        Population pop = evaluate_population(p, mat(X, n, p.d));
        put(pop.F, F);
        put(pop.C, G);
        if (cv) std::copy(pop.cv.begin(), pop.cv.end(), cv);
    });
}

// a scenario file through the reference's own loader and problem wrapper:
// load_wta (wta.cpp:148-192) + make_wta_problem (:112-129) + evaluate_population
int ref_wta_file_evaluate(const char* path, const double* X, int64_t n, double* F, double* G, double* cv) {
    return guarded([&] {
        ProblemDef p = make_wta_problem(load_wta(path));
        Population pop = evaluate_population(p, mat(X, n, p.d));
        put(pop.F, F);
        put(pop.C, G);
        if (cv) std::copy(pop.cv.begin(), pop.cv.end(), cv);
    });
}

int ref_wta_scenario(int32_t num, int32_t* targets, int32_t* vehicles, int32_t* strikes,
                     int32_t* cap, double* p) {
    return guarded([&] {
        WTAInstance w = wta_scenario("P" + std::to_string(num));
        *targets = static_cast<int32_t>(w.n_targets);
        *vehicles = static_cast<int32_t>(w.n_vehicles);
        std::size_t o = 0;
        for (std::size_t i = 0; i < w.n_targets; ++i) {
            if (strikes) strikes[i] = static_cast<int32_t>(w.max_strikes[i]);
            for (double v : w.p[i]) {
                if (p) p[o] = v;
                ++o;
            }
        }
        for (std::size_t v = 0; v < w.n_vehicles; ++v)
            if (cap) cap[v] = static_cast<int32_t>(w.capacity[v]);
    });
}

double ref_pbi(const double* f, const double* w, const double* z, int32_t m, double theta) {
    return pbi({f, static_cast<std::size_t>(m)}, {w, static_cast<std::size_t>(m)},
               {z, static_cast<std::size_t>(m)}, theta);
}

double ref_cv(const double* raw, int32_t nin, int32_t neq) {
    return cv_from_raw({raw, static_cast<std::size_t>(nin + neq)},
                       ConstraintSpec{static_cast<std::size_t>(nin), static_cast<std::size_t>(neq), 1e-6});
}

int ref_reference_vectors(int32_t m, int64_t n, double* W) {
    return guarded([&] { put(reference_vectors(m, n), W); });
}

int ref_build_neighborhoods(const double* W, int64_t n, int32_t m, int32_t t1, int32_t t2,
                            uint32_t* B1, uint32_t* B2) {
    return guarded([&] {
        NeighborhoodTopology t = build_neighborhoods(mat(W, n, m), t1, t2);
        for (int64_t i = 0; i < n; ++i) {
            std::copy(t.b1[i].begin(), t.b1[i].end(), B1 + i * t1);
            std::copy(t.b2[i].begin(), t.b2[i].end(), B2 + i * t2);
        }
    });
}

// pops: [pop1, pop2, off1, off2] each (X, F, C, cv); outs: [out1, out2]
int ref_environmental_selection(int64_t n, int32_t d, int32_t m, int32_t nc,
                                const double* const* X, const double* const* F,
                                const double* const* C, const double* const* cv,
                                const double* W, const double* z, double theta, int32_t t1,
                                const uint32_t* B1, int32_t t2, const uint32_t* B2,
                                double* const* oX, double* const* oF, double* const* oC,
                                double* const* ocv) {
    return guarded([&] {
        Population p[4];
        for (int k = 0; k < 4; ++k) p[k] = popn(X[k], F[k], C[k], cv[k], n, d, m, nc);
        Matrix Wm = mat(W, n, m);
        std::vector<double> zv(z, z + m);
        SelectionContext ctx{Wm, zv, theta};
        NeighborhoodTopology topo = topo_of(B1, t1, B2, t2, n);
        auto [a, b] = environmental_selection(p[0], p[1], p[2], p[3], topo, ctx);
        unpop(a, oX[0], oF[0], oC[0], ocv[0]);
        unpop(b, oX[1], oF[1], oC[1], ocv[1]);
    });
}

// OP2 marks alone (1 = replace), after OP1 on the given offspring
int ref_op2_marks(int64_t n, int32_t d, int32_t m, int32_t nc, const double* const* X,
                  const double* const* F, const double* const* C, const double* const* cv,
                  const double* W, const double* z, double theta, int32_t t1, const uint32_t* B1,
                  int32_t t2, const uint32_t* B2, uint8_t* marks1, uint8_t* marks2) {
    return guarded([&] {
        Population p[4];
        for (int k = 0; k < 4; ++k) p[k] = popn(X[k], F[k], C[k], cv[k], n, d, m, nc);
        Matrix Wm = mat(W, n, m);
        std::vector<double> zv(z, z + m);
        SelectionContext ctx{Wm, zv, theta};
        NeighborhoodTopology topo = topo_of(B1, t1, B2, t2, n);
        op1_offspring_cooperation(p[2], p[3], ctx);
        auto [i1, i2] = op2_update_indexing(topo, p[2], p[3], p[0], p[1], ctx);
        for (int64_t i = 0; i < n; ++i) {
            for (int l = 0; l < t1; ++l) marks1[i * t1 + l] = i1.rows[i][l] == IndexVector::sentinel;
            for (int l = 0; l < t2; ++l) marks2[i * t2 + l] = i2.rows[i][l] == IndexVector::sentinel;
        }
    });
}

int ref_wilcoxon(const double* a, int64_t na, const double* b, int64_t nb, double alpha, double* p,
                 int32_t* direction) {
    return guarded([&] {
        WilcoxonResult w = wilcoxon_rank_sum(std::vector<double>(a, a + na), std::vector<double>(b, b + nb), alpha);
        *p = w.p_value;
        *direction = w.direction;
    });
}

int ref_igd(const double* A, int64_t na, const double* R, int64_t nr, int32_t m, double* out) {
    return guarded([&] { *out = igd(mat(A, na, m), mat(R, nr, m)); });
}

int ref_hypervolume(const double* P, int64_t n, int32_t m, const double* refp, double* out) {
    return guarded([&] {
        *out = hypervolume(mat(P, n, m), std::span<const double>(refp, static_cast<std::size_t>(m)));
    });
}

int ref_metric_front(const double* F, const double* cv, int64_t n, int32_t m, double* out,
                     int64_t* rows) {
    return guarded([&] {
        Population p;
        p.X = Matrix(n, 1);
        p.F = mat(F, n, m);
        p.C = Matrix(n, 0);
        p.cv.assign(cv, cv + n);
        Matrix fr = metric_front(p);
        put(fr, out);
        *rows = static_cast<int64_t>(fr.rows);
    });
}

int ref_pf_reference(const char* name, int64_t npoints, double* out, int64_t cap, int64_t* rows) {
    return guarded([&] {
        ProblemDef p = problem_for(name);
        Matrix fr = pf_reference(p, npoints);
        if (static_cast<int64_t>(fr.rows) > cap) throw std::invalid_argument("pf_reference: cap too small");
        put(fr, out);
        *rows = static_cast<int64_t>(fr.rows);
    });
}

// the unmodified reference loop; hist = (gen, evals, wall_ms, feasible_ratio)
int ref_run_gmpea(const char* name, int64_t n, int64_t k_max, uint64_t seed, int32_t op,
                  double time_budget_s, int64_t eval_budget, int32_t t1, int32_t t2, double theta,
                  int32_t record_walltime, double* X, double* F, double* C, double* cv,
                  double* hist, int64_t hist_cap, int64_t* hist_rows) {
    return guarded([&] {
        ProblemDef p = problem_for(name);
        RunConfig cfg;
        cfg.n = n;
        cfg.k_max = k_max;
        if (time_budget_s > 0) cfg.time_budget_s = time_budget_s;
        if (eval_budget > 0) cfg.eval_budget = eval_budget;
        cfg.seed = seed;
        cfg.op = op == 1 ? VariationOp::de : VariationOp::sbx_pm;
        cfg.theta = theta;
        cfg.t1 = t1;
        cfg.t2 = t2;
        cfg.record_walltime = record_walltime != 0;
        RunResult r = run_gmpea(p, cfg);
        unpop(r.pop1, X, F, C, cv);
        int64_t k = 0;
        for (const GenRecord& g : r.history) {
            if (k >= hist_cap) break;
            hist[k * 4 + 0] = static_cast<double>(g.gen);
            hist[k * 4 + 1] = static_cast<double>(g.evals);
            hist[k * 4 + 2] = g.wall_ms;
            hist[k * 4 + 3] = g.feasible_ratio;
            ++k;
        }
        *hist_rows = k;
    });
}

// ---- comparison algorithms (baselines.hpp): operators and runs
int ref_nondominated_sort(const double* F, const double* cv, int64_t n, int32_t m, int32_t use_cdp,
                          int64_t* rank) {
    return guarded([&] {
        Matrix M = mat(F, n, m);
        std::vector<double> c(cv, cv + n);
        auto r = nondominated_sort(M, c, use_cdp != 0);
        for (int64_t i = 0; i < n; ++i) rank[i] = static_cast<int64_t>(r[i]);
    });
}

int ref_crowding_distance(const double* F, int64_t n, int32_t m, const int64_t* front, int64_t k,
                          double* dist) {
    return guarded([&] {
        Matrix M = mat(F, n, m);
        std::vector<std::size_t> fr(front, front + k);
        auto d = crowding_distance(M, fr);
        std::copy(d.begin(), d.end(), dist);
    });
}

int ref_spea2_fitness(const double* F, const double* cv, int64_t n, int32_t m, int32_t use_cdp, double* fit) {
    return guarded([&] {
        Matrix M = mat(F, n, m);
        std::vector<double> c(cv, cv + n);
        auto f = spea2_fitness(M, c, use_cdp != 0);
        std::copy(f.begin(), f.end(), fit);
    });
}

int ref_spea2_select(const double* F, const double* cv, int64_t n, int32_t m, int32_t use_cdp, int64_t capacity,
                     int64_t* keep, int64_t* count) {
    return guarded([&] {
        Matrix M = mat(F, n, m);
        std::vector<double> c(cv, cv + n);
        auto k = spea2_select(M, c, use_cdp != 0, capacity);
        for (size_t i = 0; i < k.size(); ++i) keep[i] = static_cast<int64_t>(k[i]);
        *count = static_cast<int64_t>(k.size());
    });
}

// run_cnsga2 / run_ccmo (baselines.cpp:320-459); algo 0 = cnsga2, 1 = ccmo
int ref_run_baseline(int32_t algo, const char* name, int64_t n, int64_t k_max, uint64_t seed, double* X, double* F,
                     double* C, double* cv, double* hist, int64_t hist_cap, int64_t* hist_rows) {
    return guarded([&] {
        ProblemDef p = problem_for(name);
        RunConfig cfg;
        cfg.n = n;
        cfg.k_max = k_max;
        cfg.seed = seed;
        cfg.record_walltime = false;
        RunResult r = algo == 0 ? run_cnsga2(p, cfg) : run_ccmo(p, cfg);
        unpop(r.pop1, X, F, C, cv);
        int64_t k = 0;
        for (const GenRecord& g : r.history) {
            if (k >= hist_cap) break;
            hist[k * 4 + 0] = static_cast<double>(g.gen);
            hist[k * 4 + 1] = static_cast<double>(g.evals);
            hist[k * 4 + 2] = g.wall_ms;
            hist[k * 4 + 3] = g.feasible_ratio;
            ++k;
        }
        *hist_rows = k;
    });
}

// The reference loop body (gmpea.cpp:457-489: reproduce x2, evaluate_population
// x2, update_ideal x2, environmental_selection) on `replicas` independent
// populations, one std::thread each (the reference's only parallelism is
// independent runs, experiment.cpp:217-225).  The topology (B1, B2) is
// injected; W = reference_vectors(m, n).  Times `gens` generations after
// `warmup` untimed ones and returns per-replica loop seconds in secs[].
int ref_loop_bench(const char* name, int64_t n, int32_t op, int32_t t1, const uint32_t* B1,
                   int32_t t2, const uint32_t* B2, int32_t warmup, int32_t gens, int32_t replicas,
                   uint64_t seed, double* secs) {
    return guarded([&] {
        ProblemDef p = problem_for(name);
        Matrix W = reference_vectors(p.m, n);
        NeighborhoodTopology topo = topo_of(B1, t1, B2, t2, n);
        VariationOp vop = op == 1 ? VariationOp::de : VariationOp::sbx_pm;
        std::vector<std::string> errs(replicas);
        auto body = [&](int r) {
            try {
                Rng rng(seed + static_cast<uint64_t>(r));
                auto rand_pop = [&] {
                    Matrix X(n, p.d);
                    for (int64_t i = 0; i < n; ++i)
                        for (std::size_t c = 0; c < p.d; ++c)
                            X.at(i, c) = rng.uniform(p.bounds[c].first, p.bounds[c].second);
                    return X;
                };
                Population pop1 = evaluate_population(p, rand_pop());
                Population pop2 = evaluate_population(p, rand_pop());
                std::vector<double> z(p.m, std::numeric_limits<double>::infinity());
                z = update_ideal(std::move(z), pop1.F);
                z = update_ideal(std::move(z), pop2.F);
                OperatorParams prm;
                double loop_s = 0.0;
                for (int g = 0; g < warmup + gens; ++g) {
                    Population prev1 = pop1, prev2 = pop2;  // gmpea.cpp:461
                    auto g0 = std::chrono::steady_clock::now();
                    Matrix ox1 = reproduce(pop1, topo.b1, p, rng, vop, prm);
                    Matrix ox2 = reproduce(pop2, topo.b2, p, rng, vop, prm);
                    Population off1 = evaluate_population(p, std::move(ox1));
                    Population off2 = evaluate_population(p, std::move(ox2));
                    z = update_ideal(std::move(z), off1.F);
                    z = update_ideal(std::move(z), off2.F);
                    SelectionContext ctx{W, z, 5.0};
                    std::tie(pop1, pop2) =
                        environmental_selection(pop1, pop2, std::move(off1), std::move(off2), topo, ctx);
                    double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - g0).count();
                    if (g >= warmup) loop_s += dt;
                }
                secs[r] = loop_s;
            } catch (const std::exception& e) {
                errs[r] = e.what();
            }
        };
        std::vector<std::thread> th;
        for (int r = 0; r < replicas; ++r) th.emplace_back(body, r);
        for (auto& t : th) t.join();
        for (const auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
    });
}

}  // extern "C"
