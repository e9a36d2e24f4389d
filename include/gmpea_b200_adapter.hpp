// gmpea_b200_adapter.hpp — C++ adapter that presents the engine through the
// reference's own types (proj/include/gmpea/*.hpp).  Header-only; include it
// from the reference tree and link libgmpea_b200.so.  See INTEGRATION.md.
//
//   gmpea_b200::run_gmpea(const ProblemDef&, const RunConfig&[, const Matrix* igd_front])
//        replaces gmpea::run_gmpea (gmpea.hpp:144, gmpea.cpp:421-493); with
//        igd_front the IGD hook runs on the device (experiment.cpp:200-205)
//   gmpea_b200::run_gmpea(const WTAInstance&, const RunConfig&)  -> RunResult
//        a loaded scenario (load_wta, wta.cpp:148-192) with its own tables
//   gmpea_b200::evaluate_population(const ProblemDef&, Matrix) -> Population
//        replaces gmpea::evaluate_population (gmpea.hpp:33)
//   gmpea_b200::environmental_selection(...)                   -> pair<Population>
//        replaces gmpea::environmental_selection (gmpea.hpp:108-111)
//   gmpea_b200::run_cnsga2 / run_ccmo(const ProblemDef&, const RunConfig&)
//        replace gmpea::run_cnsga2 / run_ccmo (baselines.hpp:33-34)
//   gmpea_b200::nondominated_sort / crowding_distance / spea2_fitness /
//   spea2_select  replace the baselines.hpp operators (results identical)
//   gmpea_b200::pf_reference(const ProblemDef&, size_t) -> Matrix
//        replaces gmpea::pf_reference (fronts.cpp:54-84)
//
// Exceptions: GMPEA_EINVAL -> std::invalid_argument, everything else ->
// std::runtime_error, with the engine's (reference-identical) messages.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <span>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gmpea/gmpea.hpp"
#include "gmpea/wta.hpp"
#include "gmpea_b200.h"

namespace gmpea_b200 {

inline void check(int rc) {
    if (rc == GMPEA_OK) return;
    if (rc == GMPEA_EINVAL) throw std::invalid_argument(gmpea_last_error());
    throw std::runtime_error(gmpea_last_error());
}

struct ProblemHandle {
    gmpea_problem* p = nullptr;
    explicit ProblemHandle(const gmpea::ProblemDef& def) {
        // registered suites are resolved by name (problems.cpp:542-550); the
        // engine carries its own device evaluator for each of them
        check(gmpea_problem_create(def.name.c_str(), &p));
        int32_t d, m, nin, neq;
        check(gmpea_problem_info(p, &d, &m, &nin, &neq));
        if ((std::size_t)d != def.d || (std::size_t)m != def.m || (std::size_t)nin != def.n_ineq ||
            (std::size_t)neq != def.n_eq) {
            gmpea_problem_destroy(p);
            throw std::invalid_argument("gmpea-b200: problem shape differs from " + def.name);
        }
        probe(def);
    }
    // a loaded WTA scenario with its own tables (make_wta_problem, wta.cpp:112-129)
    explicit ProblemHandle(const gmpea::WTAInstance& w) {
        std::vector<int32_t> strikes(w.max_strikes.begin(), w.max_strikes.end());
        std::vector<int32_t> cap(w.capacity.begin(), w.capacity.end());
        std::vector<double> pv;
        for (const auto& row : w.p) pv.insert(pv.end(), row.begin(), row.end());
        check(gmpea_problem_create_wta(w.scenario.c_str(), (int32_t)w.n_targets, (int32_t)w.n_vehicles,
                                       strikes.data(), cap.data(), pv.data(), &p));
    }
    ~ProblemHandle() { gmpea_problem_destroy(p); }
    ProblemHandle(const ProblemHandle&) = delete;
    ProblemHandle& operator=(const ProblemHandle&) = delete;

    // The reference's plugin is any ProblemDef (problems.hpp:19-37) and the
    // engine only knows its registered evaluators: evaluate probe rows through
    // def.eval_row and the device, and refuse a ProblemDef whose evaluation
    // differs (e.g. a loaded WTA scenario that reuses the name "WTA-P3" with
    // other tables; run those through the WTAInstance overloads).
    void probe(const gmpea::ProblemDef& def) {
        const std::size_t d = def.d, m = def.m, nc = def.n_ineq + def.n_eq, rows = 16;
        std::vector<double> X(rows * d), F(rows * m), G(rows * nc), Fr(m), Gr(nc);
        uint64_t state = 0x9E3779B97F4A7C15ull;
        for (std::size_t r = 0; r < rows; ++r)
            for (std::size_t j = 0; j < d; ++j) {
                state = state * 6364136223846793005ull + 1442695040888963407ull;
                const double u = (double)(uint32_t)(state >> 40) / 16777216.0;  // fp32-exact in [0, 1)
                const double lo = def.bounds[j].first, hi = def.bounds[j].second;
                X[r * d + j] = (double)(float)(lo + (hi - lo) * u);
                if (!(X[r * d + j] >= lo && X[r * d + j] <= hi)) X[r * d + j] = lo;
            }
        check(gmpea_evaluate(p, X.data(), (int64_t)rows, F.data(), G.data(), nullptr));
        auto close = [](double a, double b) { return std::abs(a - b) <= 1e-5 * std::max(1.0, std::abs(b)); };
        for (std::size_t r = 0; r < rows; ++r) {
            def.eval_row(std::span<const double>(X.data() + r * d, d), std::span<double>(Fr), std::span<double>(Gr));
            bool same = true;
            for (std::size_t k = 0; k < m; ++k) same = same && close(F[r * m + k], Fr[k]);
            for (std::size_t k = 0; k < nc; ++k) same = same && close(G[r * nc + k], Gr[k]);
            if (!same) {
                gmpea_problem_destroy(p);
                p = nullptr;
                throw std::invalid_argument("gmpea-b200: " + def.name +
                                            " evaluates differently from the engine's problem of that name");
            }
        }
    }
};

inline gmpea_operator_params to_c(const gmpea::OperatorParams& o) {
    gmpea_operator_params c;
    c.sbx_prob = o.sbx_prob;
    c.sbx_eta = o.sbx_eta;
    c.pm_eta = o.pm_eta;
    c.de_cr = o.de_cr;
    c.de_f = o.de_f;
    c.pm_prob = o.pm_prob ? *o.pm_prob : -1.0;
    return c;
}

inline gmpea::Population read_population(gmpea_engine* e, int which, const gmpea::ProblemDef& def,
                                         std::size_t n) {
    gmpea::Population pop;
    pop.X = gmpea::Matrix(n, def.d);
    pop.F = gmpea::Matrix(n, def.m);
    pop.C = gmpea::Matrix(n, def.n_ineq + def.n_eq);
    pop.cv.assign(n, 0.0);
    check(gmpea_engine_get_population(e, which, pop.X.data.data(), pop.F.data.data(), pop.C.data.data(),
                                      pop.cv.data()));
    return pop;
}

// run_gmpea (gmpea.cpp:421-493) on the device.  Metric hooks, when set, are
// called on pop1 after every generation, outside the loop timer, as the
// reference does (gmpea.cpp:442-453).  igd_front: the IGD hook the harness
// installs, igd(metric_front(pop1), *igd_front) (experiment.cpp:200-205), runs
// on the device instead of copying pop1 back every generation.
inline gmpea::RunResult run_on(gmpea_problem* prob, const gmpea::ProblemDef& def, const gmpea::RunConfig& cfg,
                               const gmpea::Matrix* igd_front);

inline gmpea::RunResult run_gmpea(const gmpea::ProblemDef& def, const gmpea::RunConfig& cfg,
                                  const gmpea::Matrix* igd_front = nullptr) {
    ProblemHandle ph(def);
    return run_on(ph.p, def, cfg, igd_front);
}

// a loaded scenario with its own tables (load_wta + make_wta_problem)
inline gmpea::RunResult run_gmpea(const gmpea::WTAInstance& w, const gmpea::RunConfig& cfg) {
    ProblemHandle ph(w);
    return run_on(ph.p, gmpea::make_wta_problem(w), cfg, nullptr);
}

inline gmpea::RunResult run_on(gmpea_problem* prob, const gmpea::ProblemDef& def, const gmpea::RunConfig& cfg,
                               const gmpea::Matrix* igd_front) {
    gmpea_run_config c;
    gmpea_run_config_default(&c);
    c.n = (int64_t)cfg.n;
    c.k_max = (int64_t)cfg.k_max;
    c.time_budget_s = cfg.time_budget_s ? *cfg.time_budget_s : -1.0;
    c.eval_budget = cfg.eval_budget ? (int64_t)*cfg.eval_budget : -1;
    c.seed = cfg.seed;
    c.op = cfg.op == gmpea::VariationOp::de ? GMPEA_OP_DE : GMPEA_OP_SBX_PM;
    c.params = to_c(cfg.op_params);
    c.theta = cfg.theta;
    c.t1 = (int32_t)cfg.t1;
    c.t2 = (int32_t)cfg.t2;
    c.record_walltime = cfg.record_walltime ? 1 : 0;
    if (igd_front) {
        if (igd_front->cols != def.m) throw std::invalid_argument("igd: objective count mismatch");
        c.igd_reference = igd_front->data.data();
        c.igd_reference_rows = (int64_t)igd_front->rows;
    }
    gmpea_engine* e = nullptr;
    check(gmpea_engine_create(prob, &c, &e));
    std::unique_ptr<gmpea_engine, void (*)(gmpea_engine*)> guard(e, gmpea_engine_destroy);
    gmpea::RunResult res;
    res.effective_n = (std::size_t)gmpea_engine_effective_n(e);
    // host hooks: the HV hook, and an IGD hook the device does not run
    const bool hooks = (!igd_front && (bool)cfg.igd_metric) || (bool)cfg.hv_metric;
    auto to_rec = [](const gmpea_gen_record& r) {
        gmpea::GenRecord g;
        g.gen = (std::size_t)r.gen;
        g.evals = (std::size_t)r.evals;
        g.wall_ms = r.wall_ms;
        g.feasible_ratio = r.feasible_ratio;
        if (r.has_igd) g.igd = r.igd;
        return g;
    };
    if (!hooks) {
        check(gmpea_engine_run(e));
        int64_t n = 0;
        check(gmpea_engine_history(e, nullptr, 0, &n));
        std::vector<gmpea_gen_record> h((std::size_t)n);
        check(gmpea_engine_history(e, h.data(), n, &n));
        for (const auto& r : h) res.history.push_back(to_rec(r));
    } else {
        // generation by generation so the host hooks see every pop1
        auto hook = [&](gmpea::GenRecord g) {
            gmpea::Population p1 = read_population(e, 1, def, res.effective_n);
            if (cfg.igd_metric && !igd_front) g.igd = cfg.igd_metric(p1);
            if (cfg.hv_metric) g.hv = cfg.hv_metric(p1);
            res.history.push_back(g);
        };
        gmpea_gen_record r;
        check(gmpea_engine_last_record(e, &r));
        hook(to_rec(r));
        for (;;) {
            int64_t before = r.gen;
            check(gmpea_engine_step(e, 1));
            check(gmpea_engine_sync(e));
            check(gmpea_engine_last_record(e, &r));
            if (r.gen == before) break;  // limit reached or deadline crossed
            hook(to_rec(r));
        }
        if (igd_front) {  // the device hook's values (last_record carries none)
            int64_t n = 0;
            check(gmpea_engine_history(e, nullptr, 0, &n));
            std::vector<gmpea_gen_record> h((std::size_t)n);
            check(gmpea_engine_history(e, h.data(), n, &n));
            for (std::size_t k = 0; k < res.history.size() && k < h.size(); ++k)
                if (h[k].has_igd) res.history[k].igd = h[k].igd;
        }
    }
    res.pop1 = read_population(e, 1, def, res.effective_n);
    return res;
}

// evaluate_population (gmpea.cpp:15-23) on the device
inline gmpea::Population evaluate_population(const gmpea::ProblemDef& def, gmpea::Matrix X) {
    ProblemHandle ph(def);
    if (X.cols != def.d) throw std::invalid_argument("evaluate: wrong decision dimension");
    gmpea::Population pop;
    pop.F = gmpea::Matrix(X.rows, def.m);
    pop.C = gmpea::Matrix(X.rows, def.n_ineq + def.n_eq);
    pop.cv.assign(X.rows, 0.0);
    check(gmpea_evaluate(ph.p, X.data.data(), (int64_t)X.rows, pop.F.data.data(), pop.C.data.data(),
                         pop.cv.data()));
    pop.X = std::move(X);
    return pop;
}

// environmental_selection (gmpea.cpp:392-399) on the device; surviving rows
// are bit-identical copies of the inputs
inline std::pair<gmpea::Population, gmpea::Population> environmental_selection(
    const gmpea::Population& pop1, const gmpea::Population& pop2, const gmpea::Population& off1,
    const gmpea::Population& off2, const gmpea::NeighborhoodTopology& topo, const gmpea::SelectionContext& ctx) {
    const std::size_t n = pop1.size();
    auto view = [](const gmpea::Population& p) {
        return gmpea_population_view{p.X.data.data(), p.F.data.data(), p.C.data.data(), p.cv.data()};
    };
    std::vector<uint32_t> B1, B2;
    for (const auto& r : topo.b1) B1.insert(B1.end(), r.begin(), r.end());
    for (const auto& r : topo.b2) B2.insert(B2.end(), r.begin(), r.end());
    gmpea::Population o1 = pop1, o2 = pop2;
    gmpea_population_view v1 = view(pop1), v2 = view(pop2), v3 = view(off1), v4 = view(off2);
    gmpea_population_out w1{o1.X.data.data(), o1.F.data.data(), o1.C.data.data(), o1.cv.data()};
    gmpea_population_out w2{o2.X.data.data(), o2.F.data.data(), o2.C.data.data(), o2.cv.data()};
    check(gmpea_environmental_selection((int64_t)n, (int32_t)pop1.X.cols, (int32_t)pop1.F.cols,
                                        (int32_t)pop1.C.cols, &v1, &v2, &v3, &v4, ctx.W.data.data(), ctx.z.data(),
                                        ctx.theta, B1.data(), (int32_t)topo.t1, B2.data(), (int32_t)topo.t2, &w1,
                                        &w2, nullptr, nullptr));
    return {std::move(o1), std::move(o2)};
}

namespace detail {
inline void pop_hook(void* user, int64_t n, const double* X, const double* F, const double* C, const double* cv,
                     double* igd, double* hv, int32_t* has_igd, int32_t* has_hv) {
    const auto& cfg = *static_cast<const std::pair<const gmpea::RunConfig*, const gmpea::ProblemDef*>*>(user);
    const gmpea::ProblemDef& def = *cfg.second;
    gmpea::Population p;
    p.X = gmpea::Matrix((std::size_t)n, def.d);
    p.F = gmpea::Matrix((std::size_t)n, def.m);
    p.C = gmpea::Matrix((std::size_t)n, def.n_ineq + def.n_eq);
    std::copy(X, X + n * def.d, p.X.data.begin());
    std::copy(F, F + n * def.m, p.F.data.begin());
    std::copy(C, C + n * (def.n_ineq + def.n_eq), p.C.data.begin());
    p.cv.assign(cv, cv + n);
    if (cfg.first->igd_metric) {
        *igd = cfg.first->igd_metric(p);
        *has_igd = 1;
    }
    if (cfg.first->hv_metric) {
        *hv = cfg.first->hv_metric(p);
        *has_hv = 1;
    }
}

inline gmpea::RunResult run_baseline(int algo, const gmpea::ProblemDef& def, const gmpea::RunConfig& cfg) {
    ProblemHandle ph(def);
    gmpea_run_config c;
    gmpea_run_config_default(&c);
    c.n = (int64_t)cfg.n;
    c.k_max = (int64_t)cfg.k_max;
    c.time_budget_s = cfg.time_budget_s ? *cfg.time_budget_s : -1.0;
    c.eval_budget = cfg.eval_budget ? (int64_t)*cfg.eval_budget : -1;
    c.seed = cfg.seed;
    c.params = to_c(cfg.op_params);
    c.record_walltime = cfg.record_walltime ? 1 : 0;
    std::pair<const gmpea::RunConfig*, const gmpea::ProblemDef*> user{&cfg, &def};
    const bool hooks = (bool)cfg.igd_metric || (bool)cfg.hv_metric;
    const std::size_t n = cfg.n;
    gmpea::RunResult res;
    res.effective_n = n;
    res.pop1.X = gmpea::Matrix(n, def.d);
    res.pop1.F = gmpea::Matrix(n, def.m);
    res.pop1.C = gmpea::Matrix(n, def.n_ineq + def.n_eq);
    res.pop1.cv.assign(n, 0.0);
    int64_t nh = 0;
    std::vector<gmpea_gen_record> h(1 << 16);
    for (;;) {
        check(gmpea_run_baseline(ph.p, algo, &c, nullptr, 0, hooks ? detail::pop_hook : nullptr,
                                 hooks ? &user : nullptr, h.data(), (int64_t)h.size(), &nh, res.pop1.X.data.data(),
                                 res.pop1.F.data.data(), res.pop1.C.data.data(), res.pop1.cv.data()));
        if (nh <= (int64_t)h.size()) break;
        h.resize((std::size_t)nh);  // deterministic: rerun with room for every record
    }
    for (int64_t k = 0; k < nh; ++k) {
        gmpea::GenRecord g;
        g.gen = (std::size_t)h[k].gen;
        g.evals = (std::size_t)h[k].evals;
        g.wall_ms = h[k].wall_ms;
        g.feasible_ratio = h[k].feasible_ratio;
        if (h[k].has_igd) g.igd = h[k].igd;
        if (h[k].has_hv) g.hv = h[k].hv;
        res.history.push_back(g);
    }
    return res;
}
}  // namespace detail

// run_cnsga2 / run_ccmo (baselines.cpp:320-459) on the device; metric hooks are
// called on pop1 after every generation, outside the loop timer
inline gmpea::RunResult run_cnsga2(const gmpea::ProblemDef& def, const gmpea::RunConfig& cfg) {
    return detail::run_baseline(GMPEA_ALGO_CNSGA2, def, cfg);
}
inline gmpea::RunResult run_ccmo(const gmpea::ProblemDef& def, const gmpea::RunConfig& cfg) {
    return detail::run_baseline(GMPEA_ALGO_CCMO, def, cfg);
}

// baselines.hpp operators on the device
inline std::vector<std::size_t> nondominated_sort(const gmpea::Matrix& F, const std::vector<double>& cv,
                                                  bool use_cdp) {
    std::vector<int64_t> r(F.rows);
    check(gmpea_nondominated_sort(F.data.data(), cv.data(), (int64_t)F.rows, (int32_t)F.cols, use_cdp ? 1 : 0,
                                  r.data()));
    return std::vector<std::size_t>(r.begin(), r.end());
}
inline std::vector<double> crowding_distance(const gmpea::Matrix& F, const std::vector<std::size_t>& front) {
    std::vector<int64_t> fr(front.begin(), front.end());
    std::vector<double> d(front.size());
    check(gmpea_crowding_distance(F.data.data(), (int64_t)F.rows, (int32_t)F.cols, fr.data(), (int64_t)fr.size(),
                                  d.data()));
    return d;
}
inline std::vector<double> spea2_fitness(const gmpea::Matrix& F, const std::vector<double>& cv, bool use_cdp) {
    std::vector<double> f(F.rows);
    check(gmpea_spea2_fitness(F.data.data(), cv.data(), (int64_t)F.rows, (int32_t)F.cols, use_cdp ? 1 : 0, f.data()));
    return f;
}
inline std::vector<std::size_t> spea2_select(const gmpea::Matrix& F, const std::vector<double>& cv, bool use_cdp,
                                             std::size_t capacity) {
    std::vector<int64_t> k(std::max<std::size_t>(F.rows, 1));
    int64_t cnt = 0;
    check(gmpea_spea2_select(F.data.data(), cv.data(), (int64_t)F.rows, (int32_t)F.cols, use_cdp ? 1 : 0,
                             (int64_t)capacity, k.data(), &cnt));
    return std::vector<std::size_t>(k.begin(), k.begin() + cnt);
}

// pf_reference (fronts.cpp:54-84) built on the device
inline gmpea::Matrix pf_reference(const gmpea::ProblemDef& def, std::size_t n_points) {
    ProblemHandle ph(def);
    const std::size_t cap = std::max<std::size_t>(n_points, 1) + 4 * 50000 + 100000;
    std::vector<double> out(cap * def.m);
    int64_t rows = 0;
    check(gmpea_pf_reference(ph.p, (int64_t)n_points, out.data(), (int64_t)cap, &rows));
    gmpea::Matrix M((std::size_t)rows, def.m);
    std::copy(out.begin(), out.begin() + rows * def.m, M.data.begin());
    return M;
}

}  // namespace gmpea_b200
