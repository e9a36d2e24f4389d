// Registers the B200 engine next to the reference's own algorithms, exactly
// as INTEGRATION.md describes, and runs both on one reference ProblemDef.
// Built by tests/test_integration.py against the UNMODIFIED reference library
// (oracle/_ref/libgmpea_ref.so) and libgmpea_b200.so.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <span>
#include <string>

#include "gmpea/baselines.hpp"
#include "gmpea/gmpea.hpp"
#include "gmpea/metrics.hpp"
#include "gmpea/problems.hpp"
#include "gmpea/wta.hpp"
#include "gmpea_b200_adapter.hpp"

using namespace gmpea;

// the maintainer's one-line registration (experiment.cpp:125-138)
static RunResult run_algorithm_with_b200(const std::string& algorithm, const ProblemDef& problem,
                                         const RunConfig& cfg) {
    if (algorithm == "gmpea-b200") return gmpea_b200::run_gmpea(problem, cfg);
    if (algorithm == "cnsga2-b200") return gmpea_b200::run_cnsga2(problem, cfg);
    if (algorithm == "ccmo-b200") return gmpea_b200::run_ccmo(problem, cfg);
    if (algorithm == "cnsga2") return run_cnsga2(problem, cfg);
    if (algorithm == "ccmo") return run_ccmo(problem, cfg);
    return run_gmpea(problem, cfg);
}

int main(int argc, char** argv) {
    const std::string name = argc > 1 ? argv[1] : "LIRCMOP13";
    ProblemDef p = make_problem(name);
    Matrix ref = pf_reference(p, 1000);
    RunConfig cfg;
    cfg.n = 300;
    cfg.k_max = 100;
    cfg.op = name.rfind("LIRCMOP", 0) == 0 ? VariationOp::de : VariationOp::sbx_pm;
    cfg.record_walltime = false;
    RunResult a = run_algorithm_with_b200("gmpea", p, cfg);
    RunResult b = run_algorithm_with_b200("gmpea-b200", p, cfg);
    std::printf("problem %s n=%zu gens ref=%zu b200=%zu\n", name.c_str(), cfg.n, a.history.size() - 1,
                b.history.size() - 1);
    std::printf("igd ref=%.6g b200=%.6g\n", igd(metric_front(a.pop1), ref), igd(metric_front(b.pop1), ref));
    std::printf("evals ref=%zu b200=%zu\n", a.history.back().evals, b.history.back().evals);
    // operator level: the engine's evaluation of the reference's own final rows
    Population re = gmpea_b200::evaluate_population(p, a.pop1.X);
    double worst = 0.0;
    for (std::size_t i = 0; i < re.F.data.size(); ++i) {
        double d = std::abs(re.F.data[i] - a.pop1.F.data[i]) / std::max(1.0, std::abs(a.pop1.F.data[i]));
        worst = std::max(worst, d);
    }
    std::printf("evaluate max rel diff %.3g\n", worst);
    // hooks: IGD per generation through the reference's own metric functions
    RunConfig h = cfg;
    h.k_max = 5;
    h.igd_metric = [&](const Population& pop) { return igd(metric_front(pop), ref); };
    RunResult c = run_algorithm_with_b200("gmpea-b200", p, h);
    std::printf("hook records %zu last igd %.6g\n", c.history.size(), *c.history.back().igd);
    // the same IGD hook on the device (the harness passes its front)
    RunResult cd = gmpea_b200::run_gmpea(p, h, &ref);
    double hd = 0.0;
    for (std::size_t k = 0; k < c.history.size() && k < cd.history.size(); ++k)
        hd = std::max(hd, std::abs(*c.history[k].igd - *cd.history[k].igd));
    std::printf("device_hook records %zu/%zu max_diff %.3g\n", cd.history.size(), c.history.size(), hd);
    // a ProblemDef that reuses a registered name with another evaluator is refused
    ProblemDef fake = p;
    fake.eval_row = [&p](std::span<const double> x, std::span<double> f, std::span<double> g) {
        p.eval_row(x, f, g);
        f[0] += 0.5;
    };
    int refused = 0;
    try {
        gmpea_b200::run_gmpea(fake, h);
    } catch (const std::invalid_argument&) {
        refused = 1;
    }
    // a loaded WTA scenario with edited tables under a built-in name: refused by
    // the ProblemDef path, run with its own tables through the WTAInstance path
    WTAInstance w = wta_scenario("P3");
    for (auto& row : w.p)
        for (double& v : row) v = std::min(1.0, v * 0.5 + 0.4);
    w.capacity[0] += 3;
    int wta_refused = 0;
    try {
        gmpea_b200::run_gmpea(make_wta_problem(w), h);
    } catch (const std::invalid_argument&) {
        wta_refused = 1;
    }
    RunConfig wc = cfg;
    wc.k_max = 3;
    wc.op = VariationOp::sbx_pm;
    RunResult wr = gmpea_b200::run_gmpea(w, wc);
    Population we = evaluate_population(make_wta_problem(w), wr.pop1.X);  // the reference's own evaluator
    double wd = 0.0;
    for (std::size_t i = 0; i < we.F.data.size(); ++i)
        wd = std::max(wd, std::abs(we.F.data[i] - wr.pop1.F.data[i]) / std::max(1.0, std::abs(we.F.data[i])));
    std::printf("plugin refused %d wta_refused %d wta_gens %zu wta_eval_diff %.3g\n", refused, wta_refused,
                wr.history.size() - 1, wd);
    // comparison algorithms through the same registration, with the IGD hook
    RunConfig bc = cfg;
    bc.n = 60;
    bc.k_max = 10;
    bc.igd_metric = h.igd_metric;
    RunResult n1 = run_algorithm_with_b200("cnsga2", p, bc), n2 = run_algorithm_with_b200("cnsga2-b200", p, bc);
    RunResult c1 = run_algorithm_with_b200("ccmo", p, bc), c2 = run_algorithm_with_b200("ccmo-b200", p, bc);
    std::printf("baselines records cnsga2 %zu/%zu ccmo %zu/%zu evals %zu/%zu %zu/%zu\n", n1.history.size(),
                n2.history.size(), c1.history.size(), c2.history.size(), n1.history.back().evals,
                n2.history.back().evals, c1.history.back().evals, c2.history.back().evals);
    // operator level: the reference's and the engine's operators on the same rows
    std::vector<std::size_t> r1 = nondominated_sort(c1.pop1.F, c1.pop1.cv, true);
    std::vector<std::size_t> r2 = gmpea_b200::nondominated_sort(c1.pop1.F, c1.pop1.cv, true);
    std::vector<double> f1 = spea2_fitness(c1.pop1.F, c1.pop1.cv, false);
    std::vector<double> f2 = gmpea_b200::spea2_fitness(c1.pop1.F, c1.pop1.cv, false);
    Matrix fr2 = gmpea_b200::pf_reference(p, 1000);
    double fd = 0.0;
    for (std::size_t i = 0; i < fr2.data.size() && fr2.data.size() == ref.data.size(); ++i)
        fd = std::max(fd, std::abs(fr2.data[i] - ref.data[i]));
    std::printf("operators ranks_equal %d fitness_equal %d front_rows %zu/%zu\n", (int)(r1 == r2), (int)(f1 == f2),
                fr2.rows, ref.rows);
    return 0;
}
