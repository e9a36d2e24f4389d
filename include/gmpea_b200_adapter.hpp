// gmpea_b200_adapter.hpp — C++ adapter that presents the engine through the
// reference's own types (proj/include/gmpea/*.hpp).  Header-only; include it
// from the reference tree and link libgmpea_b200.so.  See INTEGRATION.md.
//
//   gmpea_b200::run_gmpea(const ProblemDef&, const RunConfig&)  -> RunResult
//        replaces gmpea::run_gmpea (gmpea.hpp:144, gmpea.cpp:421-493)
//   gmpea_b200::evaluate_population(const ProblemDef&, Matrix) -> Population
//        replaces gmpea::evaluate_population (gmpea.hpp:33)
//   gmpea_b200::environmental_selection(...)                   -> pair<Population>
//        replaces gmpea::environmental_selection (gmpea.hpp:108-111)
//
// Exceptions: GMPEA_EINVAL -> std::invalid_argument, everything else ->
// std::runtime_error, with the engine's (reference-identical) messages.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gmpea/gmpea.hpp"
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
            (std::size_t)neq != def.n_eq)
            throw std::invalid_argument("gmpea-b200: problem shape differs from " + def.name);
    }
    ~ProblemHandle() { gmpea_problem_destroy(p); }
    ProblemHandle(const ProblemHandle&) = delete;
    ProblemHandle& operator=(const ProblemHandle&) = delete;
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
// reference does (gmpea.cpp:442-453).
inline gmpea::RunResult run_gmpea(const gmpea::ProblemDef& def, const gmpea::RunConfig& cfg) {
    ProblemHandle ph(def);
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
    gmpea_engine* e = nullptr;
    check(gmpea_engine_create(ph.p, &c, &e));
    std::unique_ptr<gmpea_engine, void (*)(gmpea_engine*)> guard(e, gmpea_engine_destroy);
    gmpea::RunResult res;
    res.effective_n = (std::size_t)gmpea_engine_effective_n(e);
    const bool hooks = (bool)cfg.igd_metric || (bool)cfg.hv_metric;
    auto to_rec = [](const gmpea_gen_record& r) {
        gmpea::GenRecord g;
        g.gen = (std::size_t)r.gen;
        g.evals = (std::size_t)r.evals;
        g.wall_ms = r.wall_ms;
        g.feasible_ratio = r.feasible_ratio;
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
            if (cfg.igd_metric) g.igd = cfg.igd_metric(p1);
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

}  // namespace gmpea_b200
