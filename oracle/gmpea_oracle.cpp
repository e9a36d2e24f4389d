// oracle/gmpea_oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain-loop, f64 CPU restatement of the reference GMPEA hot path
// (/root/reference/proj, "the reference"), written from the reference's
// semantics, not copied.  It exists to check the CUDA engine: only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may load
// it.  The product library (paper_2509_19821_b200/libgmpea_b200.so) never
// links or calls it.
//
// Pinning: everything the reference also has
// (LIRCMOP1-14, C/DC-DTLZ, WTA, CV, PBI, FPR, OP1/OP2/OP3, lattice, KNN, IGD,
// HV, metric_front) is checked bit-for-bit against the reference compiled from
// its own sources (oracle/_ref, built by oracle/Makefile) and against the
// committed golden fixtures in tests/golden/.  Two parts have no reference
// counterpart and are "parity unpinned" in the sense of the task statement:
//   * MW1-MW14 (absent from the reference) — restated from the
//     MW test-suite definitions (Ma & Wang, IEEE TEVC 2019, as distributed
//     with PlatEMO);
//   * DAS-CMOP1-9 (absent from the reference as well) — restated from the
//     DAS-CMOP toolkit (Fan et al., Evolutionary Computation 28(3), 2020) with
//     the difficulty triplet (eta, zeta, gamma) = (0.5, 0.5, 0.5);
//   * reproduce() drawing from the Philox key schema (oracle/philox.h) instead
//     of the reference's sequential mt19937_64 — it follows
//     proj/src/gmpea.cpp:113-206 draw for draw (b==a redraw, jrand
//     short-circuit, PM skip, rejection sampling) but the draws themselves
//     differ, so only its structure is pinned (identity cases of
//     tests/test_gmpea.cpp:141-188).
//
// All entry points are extern "C" (orc_*), plain pointers, row-major f64.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <thread>
#include <stdexcept>
#include <string>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "philox.h"

namespace {

constexpr double kPi = 3.141592653589793;  // == std::numbers::pi (problems.cpp:16)
thread_local std::string g_err;

// ---------------------------------------------------------------------------
// problems (reference: proj/src/problems.cpp, proj/src/wta.cpp)

enum Family { FAM_LIR = 1, FAM_DTLZ = 2, FAM_WTA = 3, FAM_MW = 4, FAM_DAS = 5 };
enum DtlzKind {
    C1_DTLZ1 = 1, C1_DTLZ3, C2_DTLZ2, C3_DTLZ4, DC1_DTLZ1, DC1_DTLZ3,
    DC2_DTLZ1, DC2_DTLZ3, DC3_DTLZ1, DC3_DTLZ3
};

struct Wta {
    int targets = 0, vehicles = 0;
    std::vector<int> strikes, cap;
    std::vector<std::vector<double>> p;
};

struct Problem {
    std::string name;
    int fam = 0, id = 0;
    int d = 0, m = 0, nin = 0, neq = 0;
    std::vector<double> lo, hi;
    Wta w;
};

// mt19937_64-backed draws of the reference Rng (include/gmpea/rng.hpp:18-30),
// needed only to regenerate the WTA scenarios (wta.cpp:37-47).
struct MtRng {
    std::mt19937_64 e;
    explicit MtRng(uint64_t s) : e(s) {}
    double uniform() { return static_cast<double>(e() >> 11) * 0x1.0p-53; }
    uint64_t index(uint64_t n) {
        uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        uint64_t v;
        do { v = e(); } while (v >= limit);
        return v % n;
    }
};

// custom WTA scenarios by name (make_wta_problem over a loaded WTAInstance,
// wta.cpp:112-129, 148-192)
std::mutex g_wta_mu;
std::map<std::string, Wta> g_wta_custom;

// wta.cpp:23-49 (num > 10: the same formula continued, synthetic instances)
Wta wta_scenario(int num) {
    Wta w;
    w.targets = 4 + 2 * (num - 1);
    w.vehicles = 3 + (num - 1) / 2;
    MtRng r(0x57A0000ull + static_cast<uint64_t>(num));
    w.strikes.resize(w.targets);
    w.cap.resize(w.vehicles);
    for (int i = 0; i < w.targets; ++i) w.strikes[i] = 1 + static_cast<int>(r.index(3));
    for (int v = 0; v < w.vehicles; ++v) w.cap[v] = 2 + static_cast<int>(r.index(3));
    w.p.resize(w.targets);
    for (int i = 0; i < w.targets; ++i) {
        w.p[i].resize(w.strikes[i]);
        for (int k = 0; k < w.strikes[i]; ++k) w.p[i][k] = 0.35 + 0.6 * r.uniform();
    }
    return w;
}

// problems.cpp:22-35 (LIRCMOP1-4 distance terms)
void lir_fixed(const double* x, int n, double& g1, double& g2) {
    double s = std::sin(0.5 * kPi * x[0]);
    double c = std::cos(0.5 * kPi * x[0]);
    g1 = 0.0;
    g2 = 0.0;
    for (int j = 2; j < n; j += 2) { double t = x[j] - s; g1 += t * t; }
    for (int j = 1; j < n; j += 2) { double t = x[j] - c; g2 += t * t; }
}

// problems.cpp:39-51 (LIRCMOP5-12 distance terms)
void lir_shifted(const double* x, int n, double& g1, double& g2) {
    const double dn = static_cast<double>(n);
    g1 = 0.0;
    g2 = 0.0;
    for (int j = 2; j < n; j += 2) {
        double t = x[j] - std::sin(0.5 * static_cast<double>(j + 1) * kPi * x[0] / dn);
        g1 += t * t;
    }
    for (int j = 1; j < n; j += 2) {
        double t = x[j] - std::cos(0.5 * static_cast<double>(j + 1) * kPi * x[0] / dn);
        g2 += t * t;
    }
}

// problems.cpp:54-59
double ellipse(double f1, double f2, double p, double q, double a, double b, double r,
               double th) {
    double u = (f1 - p) * std::cos(th) - (f2 - q) * std::sin(th);
    double v = (f1 - p) * std::sin(th) + (f2 - q) * std::cos(th);
    return r - u * u / (a * a) - v * v / (b * b);
}

// problems.cpp:66-137
void eval_lircmop(int id, const double* x, int n, double* f, double* g) {
    const double x1 = x[0];
    if (id <= 4) {
        double g1, g2;
        lir_fixed(x, n, g1, g2);
        f[0] = x1 + g1;
        f[1] = (id == 1 || id == 3) ? 1.0 - x1 * x1 + g2 : 1.0 - std::sqrt(x1) + g2;
        g[0] = -((0.51 - g1) * (g1 - 0.5));
        g[1] = -((0.51 - g2) * (g2 - 0.5));
        if (id >= 3) g[2] = 0.5 - std::sin(20.0 * kPi * x1);
        return;
    }
    if (id <= 8) {
        double g1, g2;
        lir_shifted(x, n, g1, g2);
        f[0] = x1 + 10.0 * g1 + 0.7057;
        bool sq = (id == 5 || id == 7);
        f[1] = (sq ? 1.0 - std::sqrt(x1) : 1.0 - x1 * x1) + 10.0 * g2 + 0.7057;
        const double th = -0.25 * kPi;
        if (id <= 6) {
            const double p[2] = {id == 5 ? 1.6 : 1.8, id == 5 ? 2.5 : 2.8};
            const double a[2] = {2.0, 2.0};
            const double b[2] = {id == 5 ? 4.0 : 8.0, 8.0};
            for (int k = 0; k < 2; ++k) g[k] = ellipse(f[0], f[1], p[k], p[k], a[k], b[k], 0.1, th);
        } else {
            const double p[3] = {1.2, 2.25, 3.5};
            const double a[3] = {2.0, 2.5, 2.5};
            const double b[3] = {6.0, 12.0, 10.0};
            for (int k = 0; k < 3; ++k) g[k] = ellipse(f[0], f[1], p[k], p[k], a[k], b[k], 0.1, th);
        }
        return;
    }
    if (id <= 12) {
        double g1, g2;
        lir_shifted(x, n, g1, g2);
        f[0] = 1.7057 * x1 * (10.0 * g1 + 1.0);
        bool sq = (id == 10 || id == 11);
        f[1] = 1.7057 * (sq ? 1.0 - std::sqrt(x1) : 1.0 - x1 * x1) * (10.0 * g2 + 1.0);
        const double th = -0.25 * kPi, al = 0.25 * kPi;
        double p, q, a, b, lv;
        switch (id) {
            case 9: p = 1.4; q = 1.4; a = 1.5; b = 6.0; lv = 2.0; break;
            case 10: p = 1.1; q = 1.2; a = 2.0; b = 4.0; lv = 1.0; break;
            case 11: p = 1.2; q = 1.2; a = 1.5; b = 5.0; lv = 2.1; break;
            default: p = 1.6; q = 1.6; a = 1.5; b = 6.0; lv = 2.5; break;
        }
        g[0] = ellipse(f[0], f[1], p, q, a, b, 0.1, th);
        g[1] = lv - (f[0] * std::sin(al) + f[1] * std::cos(al) -
                     std::sin(4.0 * kPi * (f[0] * std::cos(al) - f[1] * std::sin(al))));
        return;
    }
    double gs = 0.0;
    for (int j = 2; j < n; ++j) { double t = x[j] - 0.5; gs += 10.0 * t * t; }
    double rad = 1.7057 + gs;
    f[0] = rad * std::cos(0.5 * kPi * x[0]) * std::cos(0.5 * kPi * x[1]);
    f[1] = rad * std::cos(0.5 * kPi * x[0]) * std::sin(0.5 * kPi * x[1]);
    f[2] = rad * std::sin(0.5 * kPi * x[0]);
    double r2 = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
    g[0] = -((r2 - 9.0) * (r2 - 4.0));
    g[1] = -((r2 - 3.61) * (r2 - 3.24));
    if (id == 14) g[2] = -((r2 - 3.0625) * (r2 - 2.56));
}

// problems.cpp:141-158
double dtlz_g_rast(const double* x, int n, int m) {
    double s = 0.0;
    int k = n - m + 1;
    for (int i = m - 1; i < n; ++i) {
        double t = x[i] - 0.5;
        s += t * t - std::cos(20.0 * kPi * t);
    }
    return 100.0 * (static_cast<double>(k) + s);
}
double dtlz_g_sph(const double* x, int n, int m) {
    double s = 0.0;
    for (int i = m - 1; i < n; ++i) { double t = x[i] - 0.5; s += t * t; }
    return s;
}
// problems.cpp:160-178
void shape_linear(const double* pos, double g, int m, double* f) {
    for (int j = 0; j < m; ++j) {
        double v = 0.5;
        for (int i = 0; i + j + 1 < m; ++i) v *= pos[i];
        if (j > 0) v *= 1.0 - pos[m - 1 - j];
        f[j] = v * (1.0 + g);
    }
}
void shape_sphere(const double* pos, double g, int m, double* f) {
    for (int j = 0; j < m; ++j) {
        double v = 1.0 + g;
        for (int i = 0; i + j + 1 < m; ++i) v *= std::cos(0.5 * kPi * pos[i]);
        if (j > 0) v *= std::sin(0.5 * kPi * pos[m - 1 - j]);
        f[j] = v;
    }
}
// problems.cpp:182-201 (base: 1 linear/rastrigin, 2 sphere/sphere, 3 sphere/rastrigin, 4 DTLZ4)
void dtlz_base(int base, const double* x, int n, int m, double* f) {
    double pos[8];
    for (int i = 0; i < m - 1; ++i) pos[i] = x[i];
    if (base == 1) shape_linear(pos, dtlz_g_rast(x, n, m), m, f);
    else if (base == 2) shape_sphere(pos, dtlz_g_sph(x, n, m), m, f);
    else if (base == 3) shape_sphere(pos, dtlz_g_rast(x, n, m), m, f);
    else {
        for (int i = 0; i < m - 1; ++i) pos[i] = std::pow(pos[i], 100.0);
        shape_sphere(pos, dtlz_g_sph(x, n, m), m, f);
    }
}

// problems.cpp:426-525
void eval_dtlz(int kind, const double* x, int n, int m, double* f, double* g) {
    switch (kind) {
        case C1_DTLZ1: {
            dtlz_base(1, x, n, m, f);
            double s = 0.0;
            for (int i = 0; i + 1 < m; ++i) s += f[i] / 0.5;
            s += f[m - 1] / 0.6;
            g[0] = s - 1.0;
            return;
        }
        case C1_DTLZ3: {
            dtlz_base(3, x, n, m, f);
            double r2 = 0.0;
            for (int i = 0; i < m; ++i) r2 += f[i] * f[i];
            const double r = 9.0;
            g[0] = -((r2 - 16.0) * (r2 - r * r));
            return;
        }
        case C2_DTLZ2: {
            dtlz_base(2, x, n, m, f);
            const double r = 0.4;
            double v1 = std::numeric_limits<double>::infinity();
            for (int i = 0; i < m; ++i) {
                double t = (f[i] - 1.0) * (f[i] - 1.0) - r * r;
                for (int j = 0; j < m; ++j)
                    if (j != i) t += f[j] * f[j];
                v1 = std::min(v1, t);
            }
            double v2 = 0.0;
            const double c = 1.0 / std::sqrt(static_cast<double>(m));
            for (int i = 0; i < m; ++i) v2 += (f[i] - c) * (f[i] - c);
            v2 -= r * r;
            g[0] = std::min(v1, v2);
            return;
        }
        case C3_DTLZ4: {
            dtlz_base(4, x, n, m, f);
            for (int j = 0; j < m; ++j) {
                double s = f[j] * f[j] / 4.0;
                for (int i = 0; i < m; ++i)
                    if (i != j) s += f[i] * f[i];
                g[j] = 1.0 - s;
            }
            return;
        }
        default: break;
    }
    bool linear = (kind == DC1_DTLZ1 || kind == DC2_DTLZ1 || kind == DC3_DTLZ1);
    int base = linear ? 1 : 3;
    dtlz_base(base, x, n, m, f);
    if (kind == DC1_DTLZ1 || kind == DC1_DTLZ3) {
        g[0] = -(std::cos(3.0 * kPi * x[0]) + 0.5);
    } else if (kind == DC2_DTLZ1 || kind == DC2_DTLZ3) {
        double gd = dtlz_g_rast(x, n, m);
        g[0] = 0.9 - std::cos(3.0 * kPi * gd);
        g[1] = 0.9 - std::exp(-gd);
    } else {
        const double a = 3.0;
        for (int j = 0; j + 1 < m; ++j) g[j] = -(std::cos(a * kPi * x[j]) + 0.5);
        double gd = dtlz_g_rast(x, n, m);
        g[m - 1] = -(std::cos(a * kPi * gd) + 0.5);
    }
}

// wta.cpp:51-129 (decode: threshold, stable sort by value desc, capacity cap)
void eval_wta(const Wta& w, const double* x, int n, double* f, double* g) {
    std::vector<int> cand;
    for (int i = 0; i < n; ++i)
        if (x[i] >= 0.5) cand.push_back(i);
    std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) { return x[a] > x[b]; });
    std::vector<uint8_t> a(n, 0);
    std::vector<int> load(w.vehicles, 0);
    for (int gi : cand) {
        int v = gi % w.vehicles;
        if (load[v] < w.cap[v]) { a[gi] = 1; ++load[v]; }
    }
    double f1 = 0.0, f2 = 0.0;
    std::vector<double> lf(w.vehicles, 0.0);
    int base = 0;
    for (int i = 0; i < w.targets; ++i) {
        double surv = 1.0;
        for (int k = 0; k < w.strikes[i]; ++k) {
            double hits = 0.0;
            for (int v = 0; v < w.vehicles; ++v) {
                double xv = a[(base + k) * w.vehicles + v];
                hits += xv;
                lf[v] += xv;
            }
            surv *= 1.0 - w.p[i][k] * hits;
            f2 += hits;
        }
        f1 += 1.0 - surv;
        base += w.strikes[i];
    }
    f[0] = -f1;
    f[1] = f2;
    for (int v = 0; v < w.vehicles; ++v) g[v] = lf[v] - static_cast<double>(w.cap[v]);
    base = 0;
    for (int i = 0; i < w.targets; ++i) {
        double s = 0.0;
        for (int k = 0; k < w.strikes[i]; ++k)
            for (int v = 0; v < w.vehicles; ++v) s += a[(base + k) * w.vehicles + v];
        g[w.vehicles + i] = s - static_cast<double>(w.strikes[i]);
        base += w.strikes[i];
    }
}

// --- MW1-MW14 (NOT in the reference; parity unpinned). Restated from the MW
// suite definitions (Ma & Wang, TEVC 2019; PlatEMO conventions: D = 15,
// M = 2 except MW4/MW8/MW14 with M = 3, x in [0,1]^D except MW14 in
// [0,1.5]^D).  Index j below is 0-based; the paper's index is j+1.
double mw_g_exp(const double* x, int n, int m) {  // MW1/4/5/9/12 distance
    double s = 0.0;
    for (int j = m - 1; j < n; ++j) {
        double t = std::pow(x[j], static_cast<double>(n - m)) - 0.5 -
                   static_cast<double>(j) / (2.0 * n);
        s += 1.0 - std::exp(-10.0 * t * t);
    }
    return s;
}
double mw_g_cos(const double* x, int n, int m) {  // MW2/6/8/10/13 distance
    double s = 0.0;
    for (int j = m - 1; j < n; ++j) {
        double t = x[j] - static_cast<double>(j) / n;
        double z = 1.0 - std::exp(-10.0 * t * t);
        s += 1.5 + (0.1 / n) * z * z - 1.5 * std::cos(2.0 * kPi * z);
    }
    return s;
}
double mw_g_lin(const double* x, int n, int m) {  // MW3/7/11/14 distance
    double s = 0.0;
    for (int j = m - 1; j < n; ++j) {
        double p = x[j - 1] - 0.5;
        double t = x[j] + p * p - 1.0;
        s += 2.0 * t * t;
    }
    return s;
}

// MW objectives and constraints from the position genes x[0 .. m-2] and the
// distance sum gs (the per-kind g above): every MW problem depends on the
// distance genes only through gs, which is what the restated front
// candidates (mw_front_row) scan over.
void eval_mw_level(int id, const double* x, int n, int m, double gs, double* f, double* g) {
    switch (id) {
        case 1: {
            double gg = 1.0 + gs;
            f[0] = x[0];
            f[1] = gg * (1.0 - 0.85 * f[0] / gg);
            double l = std::sqrt(2.0) * f[1] - std::sqrt(2.0) * f[0];
            g[0] = f[0] + f[1] - 1.0 - 0.5 * std::pow(std::sin(2.0 * kPi * l), 8.0);
            return;
        }
        case 2: {
            double gg = 1.0 + gs;
            f[0] = x[0];
            f[1] = gg * (1.0 - f[0] / gg);
            double l = std::sqrt(2.0) * f[1] - std::sqrt(2.0) * f[0];
            g[0] = f[0] + f[1] - 1.0 - 0.5 * std::pow(std::sin(3.0 * kPi * l), 8.0);
            return;
        }
        case 3: {
            double gg = 1.0 + gs;
            f[0] = x[0];
            f[1] = gg * (1.0 - f[0] / gg);
            double l = std::sqrt(2.0) * f[1] - std::sqrt(2.0) * f[0];
            double s = f[0] + f[1];
            g[0] = s - 1.05 - 0.45 * std::pow(std::sin(0.75 * kPi * l), 6.0);
            g[1] = 0.85 - s + 0.3 * std::pow(std::sin(0.75 * kPi * l), 2.0);
            return;
        }
        case 4:
        case 8: {
            double gg = gs;
            // f_k = (1+g) * prod_{i < m-1-k} c(x_i) * (k > 0 ? s(x_{m-1-k}) : 1)
            for (int k = 0; k < m; ++k) {
                double v = 1.0 + gg;
                for (int i = 0; i + k + 1 < m; ++i)
                    v *= id == 4 ? x[i] : std::cos(0.5 * kPi * x[i]);
                if (k > 0) v *= id == 4 ? 1.0 - x[m - 1 - k] : std::sin(0.5 * kPi * x[m - 1 - k]);
                f[k] = v;
            }
            if (id == 4) {
                double l = f[m - 1];
                for (int k = 0; k + 1 < m; ++k) l -= f[k];
                double s = 0.0;
                for (int k = 0; k < m; ++k) s += f[k];
                g[0] = s - (1.0 + 0.4 * std::pow(std::sin(2.5 * kPi * l), 8.0));
            } else {
                double s2 = 0.0;
                for (int k = 0; k < m; ++k) s2 += f[k] * f[k];
                double l = std::asin(f[m - 1] / std::sqrt(s2));
                double t = 1.25 - 0.5 * std::pow(std::sin(6.0 * l), 2.0);
                g[0] = s2 - t * t;
            }
            return;
        }
        case 5: {
            double gg = 1.0 + gs;
            f[0] = gg * x[0];
            double r = f[0] / gg;
            f[1] = gg * std::sqrt(1.0 - r * r);
            double l1 = std::atan(f[1] / f[0]);
            double l2 = 0.5 * kPi - 2.0 * std::fabs(l1 - 0.25 * kPi);
            double q = f[0] * f[0] + f[1] * f[1];
            double a = 1.7 - 0.2 * std::sin(2.0 * l1);
            double b = 1.0 + 0.5 * std::sin(6.0 * l2 * l2 * l2);
            double c = 1.0 - 0.45 * std::sin(6.0 * l2 * l2 * l2);
            g[0] = q - a * a;
            g[1] = b * b - q;
            g[2] = c * c - q;
            return;
        }
        case 6: {
            double gg = 1.0 + gs;
            f[0] = gg * x[0] * 1.0999;
            double r = f[0] / gg;
            f[1] = gg * std::sqrt(1.1 * 1.1 - r * r);
            double l = std::pow(std::cos(6.0 * std::pow(std::atan(f[1] / f[0]), 4.0)), 10.0);
            double a = f[0] / (1.0 + 0.15 * l), b = f[1] / (1.0 + 0.75 * l);
            g[0] = a * a + b * b - 1.0;
            return;
        }
        case 7: {
            double gg = 1.0 + gs;
            f[0] = gg * x[0];
            double r = f[0] / gg;
            f[1] = gg * std::sqrt(1.0 - r * r);
            double l = std::atan(f[1] / f[0]);
            double q = f[0] * f[0] + f[1] * f[1];
            double a = 1.2 + 0.4 * std::pow(std::sin(4.0 * l), 16.0);
            double b = 1.15 - 0.2 * std::pow(std::sin(4.0 * l), 8.0);
            g[0] = q - a * a;
            g[1] = b * b - q;
            return;
        }
        case 9: {
            double gg = 1.0 + gs;
            f[0] = gg * x[0];
            f[1] = gg * (1.0 - std::pow(f[0] / gg, 0.6));
            double f1s = f[0] * f[0];
            double t1 = (1.0 - 0.64 * f1s - f[1]) * (1.0 - 0.36 * f1s - f[1]);
            double a = f[0] + 0.35, b = f[0] + 0.15;
            double t2 = 1.35 * 1.35 - a * a - f[1];
            double t3 = 1.15 * 1.15 - b * b - f[1];
            g[0] = std::min(t1, t2 * t3);
            return;
        }
        case 10: {
            double gg = 1.0 + gs;
            f[0] = gg * std::pow(x[0], static_cast<double>(n));
            double r = f[0] / gg;
            f[1] = gg * (1.0 - r * r);
            double s = f[0] * f[0];
            g[0] = -(2.0 - 4.0 * s - f[1]) * (2.0 - 8.0 * s - f[1]);
            g[1] = (2.0 - 2.0 * s - f[1]) * (2.0 - 16.0 * s - f[1]);
            g[2] = (1.0 - s - f[1]) * (1.2 - 1.2 * s - f[1]);
            return;
        }
        case 11: {
            double gg = 1.0 + gs;
            f[0] = gg * x[0] * std::sqrt(1.9999);
            double r = f[0] / gg;
            f[1] = gg * std::sqrt(2.0 - r * r);
            double s = f[0] * f[0];
            g[0] = -(3.0 - s - f[1]) * (3.0 - 4.0 * s - f[1]);
            g[1] = (3.0 - 0.625 * s - f[1]) * (3.0 - 7.0 * s - f[1]);
            g[2] = -(1.62 - 0.18 * s - f[1]) * (1.125 - 0.125 * s - f[1]);
            g[3] = (2.07 - 0.23 * s - f[1]) * (0.63 - 0.07 * s - f[1]);
            return;
        }
        case 12: {
            double gg = 1.0 + gs;
            f[0] = gg * x[0];
            double r = f[0] / gg;
            f[1] = gg * (0.85 - 0.8 * r - 0.08 * std::fabs(std::sin(3.2 * kPi * r)));
            double a = 1.0 - 0.8 * f[0] - f[1] + 0.08 * std::sin(2.0 * kPi * (f[1] - f[0] / 1.5));
            double b = 1.8 - 1.125 * f[0] - f[1] +
                       0.08 * std::sin(2.0 * kPi * (f[1] / 1.8 - f[0] / 1.6));
            double c = 1.0 - 0.625 * f[0] - f[1] +
                       0.08 * std::sin(2.0 * kPi * (f[1] - f[0] / 1.6));
            double e = 1.4 - 0.875 * f[0] - f[1] +
                       0.08 * std::sin(2.0 * kPi * (f[1] / 1.4 - f[0] / 1.6));
            g[0] = a * b;
            g[1] = -(c * e);
            return;
        }
        case 13: {
            double gg = 1.0 + gs;
            f[0] = gg * x[0] * 1.5;
            double r = f[0] / gg;
            f[1] = gg * (5.0 - std::exp(r) - std::fabs(0.5 * std::sin(3.0 * kPi * r)));
            double s3 = 0.5 * std::sin(3.0 * kPi * f[0]);
            double a = 5.0 - std::exp(f[0]) - s3 - f[1];
            double b = 5.0 - (1.0 + 0.4 * f[0]) - s3 - f[1];
            double c = 5.0 - (1.0 + f[0] + 0.5 * f[0] * f[0]) - s3 - f[1];
            double e = 5.0 - (1.0 + 0.7 * f[0]) - s3 - f[1];
            g[0] = a * b;
            g[1] = -(c * e);
            return;
        }
        case 14: {
            double gg = gs;
            double s = 0.0, sa = 0.0;
            for (int k = 0; k + 1 < m; ++k) {
                f[k] = x[k];
                double q = f[k] * f[k];
                s += 6.0 - std::exp(f[k]) - 1.5 * std::sin(1.1 * kPi * q);
                sa += 6.1 - (1.0 + f[k] + 0.5 * q + 1.5 * std::sin(1.1 * kPi * q));
            }
            f[m - 1] = (1.0 + gg) / (m - 1) * s;
            g[0] = f[m - 1] - 1.0 / (m - 1) * sa;
            return;
        }
        default: break;
    }
}

int mw_kind(int id) {  // 0: exp distance, 1: cos distance, 2: linear distance
    switch (id) {
        case 1: case 4: case 5: case 9: case 12: return 0;
        case 2: case 6: case 8: case 10: case 13: return 1;
        default: return 2;
    }
}

double mw_gsum(int id, const double* x, int n, int m) {
    const int k = mw_kind(id);
    return k == 0 ? mw_g_exp(x, n, m) : (k == 1 ? mw_g_cos(x, n, m) : mw_g_lin(x, n, m));
}

void eval_mw(int id, const double* x, int n, int m, double* f, double* g) {
    eval_mw_level(id, x, n, m, mw_gsum(id, x, n, m), f, g);
}

// --- DAS-CMOP1-9 (NOT in the reference; parity unpinned).  Restated from the
// DAS-CMOP toolkit definitions (Fan et al., Evol. Comput. 28(3), 2020): D = 30,
// x in [0,1]^D, difficulty triplet (eta, zeta, gamma) = (0.5, 0.5, 0.5), so
// a = 20, b = 2 eta - 1 = 0, d = 0.5, e = d - ln(gamma), r = 0.5 zeta.
// Constraints in the reference's "<= 0 feasible" form.
double das_g(int id, const double* x, int n) {
    const bool rast = id == 4 || id == 5 || id == 6 || id == 9;  // multimodal distance
    const int m = id >= 7 ? 3 : 2;
    const double shift = m == 2 ? std::sin(0.5 * kPi * x[0]) : 0.5;
    double s = 0.0;
    for (int j = m - 1; j < n; ++j) {
        double y = x[j] - shift;
        s += rast ? y * y - std::cos(20.0 * kPi * y) : y * y;
    }
    return rast ? static_cast<double>(n - m + 1) + s : s;
}

// objectives and constraints from the position genes and the distance g
void eval_das_level(int id, const double* x, double gg, double* f, double* g) {
    const double a = 20.0, b = 2.0 * 0.5 - 1.0, d = 0.5, e = d - std::log(0.5), r = 0.5 * 0.5;
    const int m = id >= 7 ? 3 : 2;
    const double x1 = x[0];
    g[0] = b - std::sin(a * kPi * x1);  // type I (diversity)
    if (m == 2) {
        f[0] = x1 + gg;
        if (id == 1 || id == 4)
            f[1] = 1.0 - x1 * x1 + gg;
        else if (id == 2 || id == 5)
            f[1] = 1.0 - std::sqrt(x1) + gg;
        else
            f[1] = 1.0 - std::sqrt(x1) + 0.5 * std::fabs(std::sin(5.0 * kPi * x1)) + gg;
        g[1] = -((e - gg) * (gg - d));  // type II (convergence)
        // type III (feasibility): nine rotated ellipses
        const double p[9] = {0.0, 1.0, 0.0, 1.0, 2.0, 0.0, 1.0, 2.0, 3.0};
        const double q[9] = {1.5, 0.5, 2.5, 1.5, 0.5, 3.5, 2.5, 1.5, 0.5};
        const double ea = 0.3, eb = 1.2, th = -0.25 * kPi;
        for (int k = 0; k < 9; ++k) {
            double u = (f[0] - p[k]) * std::cos(th) - (f[1] - q[k]) * std::sin(th);
            double v = (f[0] - p[k]) * std::sin(th) + (f[1] - q[k]) * std::cos(th);
            g[2 + k] = r - (u * u / (ea * ea) + v * v / (eb * eb));
        }
        return;
    }
    const double x2 = x[1];
    if (id == 7) {
        f[0] = x1 * x2 + gg;
        f[1] = x2 * (1.0 - x1) + gg;
        f[2] = 1.0 - x2 + gg;
    } else {
        f[0] = std::cos(0.5 * kPi * x1) * std::cos(0.5 * kPi * x2) + gg;
        f[1] = std::cos(0.5 * kPi * x1) * std::sin(0.5 * kPi * x2) + gg;
        f[2] = std::sin(0.5 * kPi * x1) + gg;
    }
    g[1] = b - std::cos(a * kPi * x2);
    g[2] = -((e - gg) * (gg - d));
    // four spheres: the three axis points and the centroid direction
    const double t = 1.0 / std::sqrt(3.0);
    const double P[4][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}, {t, t, t}};
    for (int k = 0; k < 4; ++k) {
        double s2 = 0.0;
        for (int i = 0; i < 3; ++i) s2 += (f[i] - P[k][i]) * (f[i] - P[k][i]);
        g[3 + k] = r * r - s2;
    }
}

void eval_das(int id, const double* x, int n, double* f, double* g) {
    eval_das_level(id, x, das_g(id, x, n), f, g);
}

int mw_ncon(int id) {
    switch (id) {
        case 3: case 7: case 12: case 13: return 2;
        case 5: case 10: return 3;
        case 11: return 4;
        default: return 1;
    }
}

Problem make_problem(const std::string& name) {
    Problem p;
    p.name = name;
    if (name.rfind("LIRCMOP", 0) == 0) {
        int id = std::stoi(name.substr(7));
        if (id < 1 || id > 14) throw std::invalid_argument("unknown problem: " + name);
        p.fam = FAM_LIR;
        p.id = id;
        p.d = 30;
        p.m = id >= 13 ? 3 : 2;
        p.nin = (id == 3 || id == 4 || id == 7 || id == 8 || id == 14) ? 3 : 2;
        p.lo.assign(p.d, 0.0);
        p.hi.assign(p.d, 1.0);
        return p;
    }
    if (name.rfind("MW", 0) == 0) {
        int id = std::stoi(name.substr(2));
        if (id < 1 || id > 14) throw std::invalid_argument("unknown problem: " + name);
        p.fam = FAM_MW;
        p.id = id;
        p.d = 15;
        p.m = (id == 4 || id == 8 || id == 14) ? 3 : 2;
        p.nin = mw_ncon(id);
        p.lo.assign(p.d, 0.0);
        p.hi.assign(p.d, id == 14 ? 1.5 : 1.0);
        return p;
    }
    if (name.rfind("DASCMOP", 0) == 0 || name.rfind("DAS-CMOP", 0) == 0) {
        int id = std::stoi(name.substr(name[3] == '-' ? 8 : 7));
        if (id < 1 || id > 9) throw std::invalid_argument("unknown problem: " + name);
        p.fam = FAM_DAS;
        p.id = id;
        p.d = 30;
        p.m = id >= 7 ? 3 : 2;
        p.nin = id >= 7 ? 7 : 11;
        p.lo.assign(p.d, 0.0);
        p.hi.assign(p.d, 1.0);
        return p;
    }
    if (name.rfind("WTA-", 0) == 0) {
        // custom scenarios (load_wta files, the synthetic instances past P10)
        std::lock_guard<std::mutex> lk(g_wta_mu);
        auto it = g_wta_custom.find(name.substr(4));
        if (it != g_wta_custom.end()) {
            p.fam = FAM_WTA;
            p.w = it->second;
            int slots = 0;
            for (int s : p.w.strikes) slots += s;
            p.d = slots * p.w.vehicles;
            p.m = 2;
            p.nin = p.w.vehicles + p.w.targets;
            p.lo.assign(p.d, 0.0);
            p.hi.assign(p.d, 1.0);
            return p;
        }
    }
    if (name.rfind("WTA-P", 0) == 0) {
        int num = std::stoi(name.substr(5));
        if (num < 1 || num > 10) throw std::invalid_argument("unknown WTA scenario: " + name.substr(4));
        p.fam = FAM_WTA;
        p.id = num;
        p.w = wta_scenario(num);
        int slots = 0;
        for (int s : p.w.strikes) slots += s;
        p.d = slots * p.w.vehicles;
        p.m = 2;
        p.nin = p.w.vehicles + p.w.targets;
        p.lo.assign(p.d, 0.0);
        p.hi.assign(p.d, 1.0);
        return p;
    }
    static const char* kDtlz[] = {"C1-DTLZ1", "C1-DTLZ3", "C2-DTLZ2", "C3-DTLZ4", "DC1-DTLZ1",
                                  "DC1-DTLZ3", "DC2-DTLZ1", "DC2-DTLZ3", "DC3-DTLZ1", "DC3-DTLZ3"};
    for (int k = 0; k < 10; ++k)
        if (name == kDtlz[k]) {
            p.fam = FAM_DTLZ;
            p.id = k + 1;
            p.m = 3;
            bool d7 = (p.id == C1_DTLZ1 || p.id == DC1_DTLZ1 || p.id == DC2_DTLZ1 || p.id == DC3_DTLZ1);
            p.d = d7 ? 7 : 12;
            if (p.id == C3_DTLZ4) p.nin = 3;
            else if (p.id == DC2_DTLZ1 || p.id == DC2_DTLZ3) p.nin = 2;
            else if (p.id == DC3_DTLZ1 || p.id == DC3_DTLZ3) p.nin = p.m;
            else p.nin = 1;
            p.lo.assign(p.d, 0.0);
            p.hi.assign(p.d, 1.0);
            return p;
        }
    throw std::invalid_argument("unknown problem: " + name);
}

void eval_row(const Problem& p, const double* x, double* f, double* g) {
    switch (p.fam) {
        case FAM_LIR: eval_lircmop(p.id, x, p.d, f, g); break;
        case FAM_DTLZ: eval_dtlz(p.id, x, p.d, p.m, f, g); break;
        case FAM_WTA: eval_wta(p.w, x, p.d, f, g); break;
        case FAM_MW: eval_mw(p.id, x, p.d, p.m, f, g); break;
        case FAM_DAS: eval_das(p.id, x, p.d, f, g); break;
    }
}

// --- restated reference-front candidates for MW / DAS-CMOP (no reference
// counterpart: the reference's front_candidates exist only for its own
// suites, problems.cpp:203-393).  Every MW / DAS-CMOP objective vector is a
// function of the position genes x_0 .. x_{m-2} and one distance value (MW:
// the distance sum gs, DAS-CMOP: g), nondecreasing in that distance for a fixed
// position, so a position's best feasible point is at its smallest feasible
// distance.  That distance is located on kLevels steps of [0, kLevelMax],
// refined by bisection, nudged 1e-9 into the feasible side and realised in
// decision space (equal per-gene shares); pf_reference (fronts.cpp:54-79)
// then evaluates, filters and subsamples the rows as for any problem.
constexpr int kLevels = 600;
constexpr double kLevelMax = 3.0;

bool restated_front(const Problem& p) { return p.fam == FAM_MW || p.fam == FAM_DAS; }

void eval_level(const Problem& p, const double* pos, double lvl, double* f, double* g) {
    if (p.fam == FAM_MW)
        eval_mw_level(p.id, pos, p.d, p.m, lvl, f, g);
    else
        eval_das_level(p.id, pos, lvl, f, g);
}

bool level_feasible(const Problem& p, const double* pos, double lvl) {
    double f[3], g[16];
    eval_level(p, pos, lvl, f, g);
    for (int k = 0; k < p.nin + p.neq; ++k)
        if (!(g[k] <= 0.0)) return false;
    return true;
}

// smallest feasible distance at this position; -1 when none on the grid
double min_feasible_level(const Problem& p, const double* pos) {
    for (int k = 0; k <= kLevels; ++k) {
        const double lvl = kLevelMax * k / kLevels;
        if (!level_feasible(p, pos, lvl)) continue;
        if (k == 0) return 0.0;
        double lo = kLevelMax * (k - 1) / kLevels, hi = lvl;
        for (int it = 0; it < 60; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (level_feasible(p, pos, mid))
                hi = mid;
            else
                lo = mid;
        }
        return hi * (1.0 + 1e-9);
    }
    return -1.0;
}

// bisection for the increasing per-gene term t(v) = tau on [a, b]
template <class T>
double solve_term(T t, double tau, double a, double b) {
    if (tau <= 0.0) return a;
    if (t(b) <= tau) return b;
    for (int it = 0; it < 80; ++it) {
        const double mid = 0.5 * (a + b);
        if (t(mid) < tau)
            a = mid;
        else
            b = mid;
    }
    return 0.5 * (a + b);
}

// decision row at position pos whose distance value is lvl
void realize_level(const Problem& p, const double* pos, double lvl, double* x) {
    const int n = p.d, m = p.m, nd = n - m + 1;
    for (int k = 0; k + 1 < m; ++k) x[k] = pos[k];
    const double tau = std::max(lvl, 0.0) / nd;
    if (p.fam == FAM_DAS) {
        const bool rast = p.id == 4 || p.id == 5 || p.id == 6 || p.id == 9;
        const double shift = m == 2 ? std::sin(0.5 * kPi * pos[0]) : 0.5;
        const double y = rast ? solve_term([](double v) { return v * v + 1.0 - std::cos(20.0 * kPi * v); }, tau,
                                           0.0, 0.05)
                              : std::sqrt(tau);
        for (int j = m - 1; j < n; ++j) x[j] = shift + y <= 1.0 ? shift + y : shift - y;
        return;
    }
    const double lo = p.lo[0], hi = p.hi[0];
    switch (mw_kind(p.id)) {
        case 0: {  // 1 - exp(-10 t^2), t = x^(n-m) - c_j
            const double e = static_cast<double>(n - m);
            const double t = std::sqrt(-std::log(1.0 - std::min(tau, 0.999)) / 10.0);
            for (int j = m - 1; j < n; ++j) {
                const double c = 0.5 + static_cast<double>(j) / (2.0 * n);
                const double v = c - t >= 0.0 ? c - t : c + t;
                x[j] = std::min(std::pow(v, 1.0 / e), hi);
            }
            return;
        }
        case 1: {  // 1.5 + (0.1/n) z^2 - 1.5 cos(2 pi z), z = 1 - exp(-10 t^2), t = x - j/n
            const double z = solve_term(
                [n](double v) { return 1.5 + (0.1 / n) * v * v - 1.5 * std::cos(2.0 * kPi * v); }, tau, 0.0, 0.5);
            const double t = std::sqrt(-std::log(1.0 - z) / 10.0);
            for (int j = m - 1; j < n; ++j) {
                const double b = static_cast<double>(j) / n;
                x[j] = b + t <= hi ? b + t : b - t;
            }
            return;
        }
        default: {  // 2 t^2, t = x_j + (x_{j-1} - 0.5)^2 - 1
            const double u = std::sqrt(tau / 2.0);
            for (int j = m - 1; j < n; ++j) {
                const double q = x[j - 1] - 0.5;
                const double v = 1.0 - q * q - u;
                x[j] = v >= lo ? v : std::min(1.0 - q * q + u, hi);
            }
            return;
        }
    }
}

// front_candidates(n_samples): m = 2 positions x_0 on n_samples even steps of
// the first gene's range; m = 3 a side x side grid (side^2 >= n_samples)
int64_t restated_front_rows(const Problem& p, int64_t n_samples) {
    if (p.m == 2) return n_samples;
    int64_t side = 1;
    while (side * side < n_samples) ++side;
    return side * side;
}

void restated_front_candidates(const Problem& p, int64_t n_samples, double* out) {
    const int64_t rows = restated_front_rows(p, n_samples);
    int64_t side = 1;
    while (side * side < n_samples) ++side;
    for (int64_t r = 0; r < rows; ++r) {
        double pos[2] = {0.0, 0.0};
        if (p.m == 2) {
            const double t = n_samples == 1 ? 0.0 : static_cast<double>(r) / static_cast<double>(n_samples - 1);
            pos[0] = p.lo[0] + (p.hi[0] - p.lo[0]) * t;
        } else {
            const double s1 = side == 1 ? 0.0 : static_cast<double>(r / side) / static_cast<double>(side - 1);
            const double s2 = side == 1 ? 0.0 : static_cast<double>(r % side) / static_cast<double>(side - 1);
            pos[0] = p.lo[0] + (p.hi[0] - p.lo[0]) * s1;
            pos[1] = p.lo[1] + (p.hi[1] - p.lo[1]) * s2;
        }
        const double lvl = min_feasible_level(p, pos);
        realize_level(p, pos, lvl < 0.0 ? 0.0 : lvl, out + r * p.d);
    }
}

// ---------------------------------------------------------------------------
// scalarization (reference: proj/src/scalarize.cpp, proj/src/kernels.cpp)

// kernels.cpp:56-67: four lane accumulators over the blocked prefix, lanes
// combined left to right, tail in order
double relu_sum(const double* a, int n) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int blocked = n / 4 * 4;
    for (int i = 0; i < blocked; ++i) acc[i % 4] += a[i] > 0.0 ? a[i] : 0.0;
    double s = ((acc[0] + acc[1]) + acc[2]) + acc[3];
    for (int i = blocked; i < n; ++i) s += a[i] > 0.0 ? a[i] : 0.0;
    return s;
}

// scalarize.cpp:39-49
double cv_raw(const double* raw, int nin, int neq) {
    if (neq == 0) return relu_sum(raw, nin);
    double s = relu_sum(raw, nin);
    for (int j = nin; j < nin + neq; ++j) {
        double v = std::fabs(raw[j]) - 1e-6;
        s += v > 0.0 ? v : 0.0;
    }
    return s;
}

// scalarize.cpp:72-89
double pbi(const double* f, const double* w, const double* z, int m, double theta) {
    double wn2 = 0.0;
    for (int i = 0; i < m; ++i) wn2 += w[i] * w[i];
    if (wn2 == 0.0) throw std::invalid_argument("pbi: zero-norm reference vector");
    double wn = std::sqrt(wn2);
    double proj = 0.0;
    for (int i = 0; i < m; ++i) proj += (f[i] - z[i]) * w[i];
    double d1 = std::fabs(proj) / wn;
    double d2sq = 0.0;
    for (int i = 0; i < m; ++i) {
        double r = (f[i] - z[i]) - d1 * (w[i] / wn);
        d2sq += r * r;
    }
    return d1 + theta * std::sqrt(d2sq);
}

// scalarize.cpp:91-96
bool fpr_better(double ga, double cva, double gb, double cvb) {
    if (cva < 0.0 || cvb < 0.0)
        throw std::invalid_argument("fpr_better: negative constraint violation");
    if (cva == cvb) return ga < gb;
    return cva < cvb;
}

// ---------------------------------------------------------------------------
// lattice + neighbourhoods (reference: proj/src/gmpea.cpp:27-100)

size_t lattice_size(size_t m, size_t H) {
    size_t n = 1;
    for (size_t i = 1; i < m; ++i) n = n * (H + i) / i;
    return n;
}

void compositions(size_t m, size_t H, std::vector<size_t>& cur, std::vector<double>& out) {
    size_t used = 0;
    for (size_t v : cur) used += v;
    if (cur.size() + 1 == m) {
        for (size_t v : cur) out.push_back(static_cast<double>(v) / H);
        out.push_back(static_cast<double>(H - used) / H);
        return;
    }
    for (size_t v = 0; v + used <= H; ++v) {
        cur.push_back(v);
        compositions(m, H, cur, out);
        cur.pop_back();
    }
}

std::vector<double> reference_vectors(size_t m, size_t n) {
    size_t H = 1;
    while (lattice_size(m, H) < n) ++H;
    std::vector<double> flat;
    std::vector<size_t> cur;
    compositions(m, H, cur, flat);
    flat.resize(n * m);
    return flat;
}

// brute-force t-NN with the (d2, j) sort order of gmpea.cpp:84-97
void knn(const double* W, size_t n, size_t m, size_t t, uint32_t* out) {
    std::vector<std::pair<double, uint32_t>> d(n);
    for (size_t i = 0; i < n; ++i) {
        for (size_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (size_t c = 0; c < m; ++c) {
                double v = W[i * m + c] - W[j * m + c];
                s += v * v;
            }
            d[j] = {s, static_cast<uint32_t>(j)};
        }
        std::partial_sort(d.begin(), d.begin() + static_cast<std::ptrdiff_t>(t), d.end());
        for (size_t k = 0; k < t; ++k) out[i * t + k] = d[k].second;
    }
}

// the brute-force t-NN rows `rows` only (a sample of a large population),
// same arithmetic and (d2, j) order as knn(); rows split over threads
void knn_rows(const double* W, size_t n, size_t m, size_t t, const int64_t* rows, size_t nrows, uint32_t* out,
              unsigned threads) {
    auto work = [&](size_t r0, size_t r1) {
        std::vector<std::pair<double, uint32_t>> d(n);
        for (size_t r = r0; r < r1; ++r) {
            const size_t i = static_cast<size_t>(rows[r]);
            for (size_t j = 0; j < n; ++j) {
                double s = 0.0;
                for (size_t c = 0; c < m; ++c) {
                    double v = W[i * m + c] - W[j * m + c];
                    s += v * v;
                }
                d[j] = {s, static_cast<uint32_t>(j)};
            }
            std::partial_sort(d.begin(), d.begin() + static_cast<std::ptrdiff_t>(t), d.end());
            for (size_t k = 0; k < t; ++k) out[r * t + k] = d[k].second;
        }
    };
    threads = std::max(1u, threads);
    std::vector<std::thread> th;
    for (unsigned k = 0; k < threads; ++k) th.emplace_back(work, nrows * k / threads, nrows * (k + 1) / threads);
    for (auto& x : th) x.join();
}

// windowed t-NN on the Das-Dennis lattice, same (d2, j) order as
// gmpea.cpp:84-97: candidates within +-R lattice steps, accepted only when
// every point outside the window is provably farther than the t-th one
// (else the window doubles).  Lets the CPU baseline build topologies at N
// where the reference's O(N^2 log N) build_neighborhoods is impractical.
void lattice_knn(size_t m, size_t n, size_t t1, size_t t2, uint32_t* B1, uint32_t* B2, unsigned threads) {
    size_t H = 1;
    if (m == 2) H = n > 1 ? n - 1 : 1;
    else
        while (lattice_size(m, H) < n) ++H;
    std::vector<double> W = reference_vectors(m, n);
    auto start3 = [&](long long a) { return a * (long long)(H + 1) - a * (a - 1) / 2; };
    auto unrank = [&](long long i, long long& a, long long& b) {
        if (m == 2) { a = i; b = (long long)H - i; return; }
        long long lo = 0, hi = (long long)H;
        while (lo < hi) {
            long long mid = (lo + hi + 1) / 2;
            if (start3(mid) <= i) lo = mid; else hi = mid - 1;
        }
        a = lo;
        b = i - start3(lo);
    };
    auto work = [&](size_t r0, size_t r1) {
        std::vector<std::pair<double, uint32_t>> cand;
        for (size_t i = r0; i < r1; ++i) {
            long long a, b;
            unrank((long long)i, a, b);
            for (long long R = 6;; R *= 2) {
                cand.clear();
                auto push = [&](long long j) {
                    double s2 = 0.0;
                    for (size_t c = 0; c < m; ++c) {
                        double d = W[i * m + c] - W[(size_t)j * m + c];
                        s2 += d * d;
                    }
                    cand.emplace_back(s2, (uint32_t)j);
                };
                bool all;
                if (m == 2) {
                    long long lo = std::max(0ll, (long long)i - R), hi = std::min((long long)n - 1, (long long)i + R);
                    for (long long j = lo; j <= hi; ++j) push(j);
                    all = lo == 0 && hi == (long long)n - 1;
                } else {
                    for (long long aa = a - R; aa <= a + R; ++aa) {
                        if (aa < 0 || aa > (long long)H) continue;
                        for (long long bb = b - R; bb <= b + R; ++bb) {
                            if (bb < 0 || aa + bb > (long long)H) continue;
                            long long j = start3(aa) + bb;
                            if (j < (long long)n) push(j);
                        }
                    }
                    all = (a - R <= 0) && (a + R >= (long long)H) && (b - R <= 0) && (b + R >= (long long)H);
                }
                size_t t = std::max(t1, t2);
                if (cand.size() < t && !all) continue;
                std::partial_sort(cand.begin(), cand.begin() + (std::ptrdiff_t)t, cand.end());
                if (!all) {
                    double step = (double)(R + 1) / (double)H;
                    double bound = (m == 2 ? 2.0 : 1.0) * step * step * (1.0 - 1e-9);
                    if (!(cand[t - 1].first < bound)) continue;
                }
                for (size_t k = 0; k < t1; ++k) B1[i * t1 + k] = cand[k].second;
                for (size_t k = 0; k < t2; ++k) B2[i * t2 + k] = cand[k].second;
                break;
            }
        }
    };
    threads = std::max(1u, threads);
    std::vector<std::thread> th;
    for (unsigned k = 0; k < threads; ++k)
        th.emplace_back(work, n * k / threads, n * (k + 1) / threads);
    for (auto& x : th) x.join();
}

// ---------------------------------------------------------------------------
// environmental selection (reference: proj/src/gmpea.cpp:248-399)
//
// Works on (F, cv) only: X and C ride along with the winning row, so the
// outcome is fully described by a source code per parent slot:
//   -1 = parent kept, c in [0,N) = off1 row c, N + c = off2 row c.
// OP1 is represented without a physical swap: eff_k[i] names the row stream k
// holds after cooperation.

struct SelIn {
    int n, m;
    const double *F1, *cv1, *F2, *cv2;     // parents
    const double *Fo1, *cvo1, *Fo2, *cvo2; // offspring
    const double *W, *z;
    double theta;
    int t1, t2;
    const uint32_t *B1, *B2;
    int agg = 0;  // 0: PBI (the reference's), 1: Tchebycheff (engine extension)
};

// weighted Tchebycheff aggregation (no reference counterpart; the engine's
// GMPEA_AGG_TCH): max_k max(w_k, 1e-6) |f_k - z_k|
double tchebycheff(const double* f, const double* w, const double* z, int m) {
    double g = 0.0;
    for (int i = 0; i < m; ++i) {
        double v = std::max(w[i], 1e-6) * std::fabs(f[i] - z[i]);
        if (std::isnan(v)) return v;
        g = std::max(g, v);
    }
    return g;
}

void selection(const SelIn& s, int32_t* src1, int32_t* src2, uint8_t* marks1, uint8_t* marks2) {
    const int n = s.n, m = s.m;
    auto key = [&](const double* f, const double* w) {
        return s.agg == 1 ? tchebycheff(f, w, s.z, m) : pbi(f, w, s.z, m, s.theta);
    };
    // OP1 (gmpea.cpp:248-279)
    std::vector<int32_t> eff1(n), eff2(n);
    for (int i = 0; i < n; ++i) {
        double g1 = key(s.Fo1 + i * m, s.W + i * m);
        double g2 = key(s.Fo2 + i * m, s.W + i * m);
        double c1 = s.cvo1[i], c2 = s.cvo2[i];
        // the reference builds these through Heaviside masks on differences,
        // which reject non-finite values (batch.cpp:10-16)
        if (!std::isfinite(c1 - c2) || !std::isfinite(g1 - g2))
            throw std::invalid_argument("non-finite mask source");
        bool s1 = c2 < c1 || (c1 == c2 && g1 > g2);
        bool s2 = g2 > g1;
        eff1[i] = s1 ? n + i : i;
        eff2[i] = s2 ? i : n + i;
    }
    auto Fof = [&](int32_t code) { return code < n ? s.Fo1 + code * m : s.Fo2 + (code - n) * m; };
    auto cvof = [&](int32_t code) { return code < n ? s.cvo1[code] : s.cvo2[code - n]; };
    for (int pop = 1; pop <= 2; ++pop) {
        const int t = pop == 1 ? s.t1 : s.t2;
        const uint32_t* B = pop == 1 ? s.B1 : s.B2;
        const double* Fp = pop == 1 ? s.F1 : s.F2;
        const double* cvp = pop == 1 ? s.cv1 : s.cv2;
        const std::vector<int32_t>& eff = pop == 1 ? eff1 : eff2;
        int32_t* src = pop == 1 ? src1 : src2;
        uint8_t* marks = pop == 1 ? marks1 : marks2;
        // OP2 (gmpea.cpp:283-303): marks; claims bucketed in ascending i (:318-327)
        std::vector<std::vector<int>> claims(n);
        for (int i = 0; i < n; ++i)
            for (int l = 0; l < t; ++l) {
                int j = static_cast<int>(B[i * t + l]);
                double go = key(Fof(eff[i]), s.W + j * m);
                double gp = key(Fp + j * m, s.W + j * m);
                bool rep = pop == 1 ? fpr_better(go, cvof(eff[i]), gp, cvp[j]) : go < gp;
                if (marks) marks[i * t + l] = rep ? 1 : 0;
                if (rep) claims[j].push_back(i);
            }
        // OP3 (gmpea.cpp:333-380)
        for (int j = 0; j < n; ++j) {
            src[j] = -1;
            const auto& cl = claims[j];
            if (cl.empty()) continue;
            int u = 0;
            for (int c : cl) {
                if (c != u) break;
                ++u;
            }
            double bcv = cvp[j];
            double bg = key(Fp + j * m, s.W + j * m);
            int bidx = u;
            int best = -1;
            for (int c : cl) {
                double g = key(Fof(eff[c]), s.W + j * m);
                double cv = cvof(eff[c]);
                bool wins;
                if (pop == 1)
                    wins = cv < bcv || (cv == bcv && g < bg) || (cv == bcv && g == bg && c < bidx);
                else
                    wins = g < bg || (g == bg && c < bidx);
                if (wins) { bcv = cv; bg = g; bidx = c; best = c; }
            }
            if (best >= 0) src[j] = eff[best];
        }
    }
}

// ---------------------------------------------------------------------------
// variation with Philox draws (structure of proj/src/gmpea.cpp:113-206)

struct Keyed {
    uint32_t key[2];
    uint32_t slot, gen, pop;
    uint32_t out[4];
    void draw(uint32_t stream, uint32_t index) {
        uint32_t ctr[4] = {slot, gen, orc_tag(pop, stream), index};
        orc_philox4x32_10(ctr, key, out);
    }
    // PICK stream: a sequence of 32-bit words, four per counter (the picks a,
    // b with the b == a redraw, DE's jrand and SBX's per-child coin, in order)
    uint32_t q = 0;
    uint32_t pick_cache[4];
    uint32_t pick32() {
        if (q % 4 == 0) {
            draw(ORC_STREAM_PICK, q / 4);
            for (int k = 0; k < 4; ++k) pick_cache[k] = out[k];
        }
        return pick_cache[q++ % 4];
    }
    // rng.hpp:23-30 rejection semantics, on 32-bit words
    uint64_t index(uint64_t n) {
        const uint64_t limit = (1ull << 32) - (1ull << 32) % n;
        uint64_t v;
        do { v = pick32(); } while (v >= limit);
        return v % n;
    }
    // SBX per-child coin u <= pc (gmpea.cpp:117): the next PICK word w, taken
    // iff w < ceil(pc 2^32)
    bool child_coin(double pc) {
        const double t = std::ceil(pc * 4294967296.0);
        return static_cast<double>(pick32()) < t;
    }
    // 32-bit coin of gene j with an exact threshold (DE's CR coin, CR < 1):
    // head = 16-bit half j % 8 of index j / 8 of the coin stream, tail = low
    // 16 bits of index j of the refinement stream
    double coin(uint32_t stream, uint32_t ref_stream, uint32_t j) {
        draw(stream, j / 8);
        uint32_t word = out[(j % 8) / 2];
        uint32_t head = (j % 2) ? (word >> 16) : (word & 0xffffu);
        draw(ref_stream, j);
        uint32_t tail = out[0] & 0xffffu;
        return static_cast<double>((head << 16) | tail) * 0x1.0p-32;
    }
    // SBX per-gene crossover coin (gmpea.cpp:119, u <= 0.5): one bit per gene,
    // bit j % 32 of word (j % 128) / 32 of index j / 128 of XCOIN; crosses iff 1
    bool xbit(uint32_t j) {
        draw(ORC_STREAM_XCOIN, j / 128);
        return (out[(j % 128) / 32] >> (j % 32)) & 1u;
    }
    // four genes per counter: gene j is word j % 4 of index j / 4
    double word(uint32_t stream, uint32_t j) {
        draw(stream, j / 4);
        return static_cast<double>(out[j % 4]) * 0x1.0p-32;
    }
    double mu(uint32_t j) {
        draw(ORC_STREAM_MU, j);
        return static_cast<double>(out[0]) * 0x1.0p-32;
    }
};

// Polynomial mutation's per-gene coin (gmpea.cpp:139: skip gene iff U > pm).
// The DE operator draws one 32-bit coin per gene (MCOIN head + MREF tail, as
// Keyed::coin).  The SBX operator draws it as gaps: the genes between two mutated ones are Geometric(pm); word t
// of MSKIP (index t / 4, word t % 4) gives gap t = the largest k in [0, d]
// with w <= T[k], T[k] = ceil((1 - pm)^k 2^32) - 1, so P(gap >= k) =
// (1 - pm)^k up to 2^-32 and every gene mutates independently with
// probability pm.  The engine builds the identical table (host.cuh).
std::vector<int64_t> pm_gap_table(double pm, int d) {
    std::vector<int64_t> T(static_cast<size_t>(d) + 1);
    T[0] = 0xffffffffll;
    double v = 1.0;
    for (int k = 1; k <= d; ++k) {
        v *= 1.0 - pm;
        T[k] = static_cast<int64_t>(std::ceil(v * 4294967296.0)) - 1;
    }
    return T;
}

std::vector<uint8_t> pm_mutated(Keyed& kd, const std::vector<int64_t>& T, int d) {
    std::vector<uint8_t> mut(static_cast<size_t>(d), 0);
    int64_t pos = -1;
    for (uint32_t t = 0;; ++t) {
        uint32_t ctr[4] = {kd.slot, kd.gen, orc_tag(kd.pop, ORC_STREAM_MSKIP), t / 4};
        uint32_t o[4];
        orc_philox4x32_10(ctr, kd.key, o);
        const int64_t w = o[t % 4];
        int gap = 0;
        while (gap < d && w <= T[gap + 1]) ++gap;
        pos += gap + 1;
        if (pos >= d) break;
        mut[pos] = 1;
    }
    return mut;
}

struct OpParams {
    double sbx_prob, sbx_eta, pm_eta, de_cr, de_f, pm_prob;  // pm_prob < 0: 1/d
};

// gmpea.cpp:135-160 for one gene the gap draws selected (pm_mutated); the
// direction uniform from MU (drawn only for mutated genes)
void pm_gene(double& x, double lo, double hi, double eta, Keyed& k, uint32_t j) {
    double span = hi - lo;
    if (span <= 0.0) return;
    double u = k.mu(j), dq;
    if (u < 0.5) {
        double d1 = (x - lo) / span;
        dq = std::pow(2.0 * u + (1.0 - 2.0 * u) * std::pow(1.0 - d1, eta + 1.0), 1.0 / (eta + 1.0)) - 1.0;
    } else {
        double d2 = (hi - x) / span;
        dq = 1.0 - std::pow(2.0 * (1.0 - u) + 2.0 * (u - 0.5) * std::pow(1.0 - d2, eta + 1.0),
                            1.0 / (eta + 1.0));
    }
    x += dq * span;
}

// std::clamp semantics: NaN passes through (gmpea.cpp:162-165)
double clamp_ref(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

void reproduce(const Problem& p, const double* X, size_t n, const uint32_t* nb, size_t t, int op,
               const OpParams& prm, uint64_t seed, uint32_t gen, uint32_t pop, double* off,
               int32_t* picks, uint32_t slot_base = 0) {
    const int d = p.d;
    const double pm = prm.pm_prob >= 0.0 ? prm.pm_prob : 1.0 / static_cast<double>(d);
    const std::vector<int64_t> gapT = pm_gap_table(pm, d);
    for (size_t i = 0; i < n; ++i) {
        Keyed k;
        k.key[0] = static_cast<uint32_t>(seed);
        k.key[1] = static_cast<uint32_t>(seed >> 32);
        k.slot = slot_base + static_cast<uint32_t>(i);  // Philox keys use global slots
        k.gen = gen;
        k.pop = pop;
        size_t a = k.index(t);
        size_t b = k.index(t);
        while (t > 1 && b == a) b = k.index(t);
        const double* xa = X + static_cast<size_t>(nb[i * t + a]) * d;
        const double* xb = X + static_cast<size_t>(nb[i * t + b]) * d;
        double* child = off + i * d;
        size_t jrand = 0;
        bool cross = true;
        if (op == 0) {
            cross = k.child_coin(prm.sbx_prob);
        } else {
            jrand = k.index(static_cast<uint64_t>(d));
        }
        if (picks) {
            picks[i * 3 + 0] = static_cast<int32_t>(a);
            picks[i * 3 + 1] = static_cast<int32_t>(b);
            picks[i * 3 + 2] = op == 0 ? (cross ? 1 : 0) : static_cast<int32_t>(jrand);
        }
        // PM genes: the SBX kernels draw gaps, the DE kernels one coin per gene
        const std::vector<uint8_t> mut = op == 0 ? pm_mutated(k, gapT, d) : std::vector<uint8_t>();
        const double* base = X + i * d;
        for (int j = 0; j < d; ++j) {
            const uint32_t uj = static_cast<uint32_t>(j);
            double c;
            if (op == 0) {
                if (!cross) {
                    c = xa[j];
                } else if (k.xbit(uj)) {
                    double u = k.word(ORC_STREAM_XU, uj);
                    double beta = u <= 0.5 ? std::pow(2.0 * u, 1.0 / (prm.sbx_eta + 1.0))
                                           : std::pow(1.0 / (2.0 * (1.0 - u)), 1.0 / (prm.sbx_eta + 1.0));
                    c = 0.5 * ((1.0 + beta) * xa[j] + (1.0 - beta) * xb[j]);
                } else {
                    c = xa[j];
                }
            } else {
                // CR >= 1 decides the coin without drawing it (u < 1 <= CR)
                bool take = static_cast<size_t>(j) == jrand || prm.de_cr >= 1.0 ||
                            k.coin(ORC_STREAM_XCOIN, ORC_STREAM_XREF, uj) < prm.de_cr;
                c = take ? base[j] + prm.de_f * (xa[j] - xb[j]) : base[j];
            }
            const bool mutate = op == 0 ? mut[j] != 0
                                        : pm > 0.0 && k.coin(ORC_STREAM_MCOIN, ORC_STREAM_MREF, uj) <= pm;
            if (mutate) pm_gene(c, p.lo[j], p.hi[j], prm.pm_eta, k, uj);
            child[j] = clamp_ref(c, p.lo[j], p.hi[j]);
        }
    }
}

// ---------------------------------------------------------------------------
// metrics (reference: proj/src/metrics.cpp)

bool dominates(const double* a, const double* b, int m) {
    bool strict = false;
    for (int i = 0; i < m; ++i) {
        if (a[i] > b[i]) return false;
        if (a[i] < b[i]) strict = true;
    }
    return strict;
}

// metrics.cpp:15-37
double igd(const double* A, size_t na, const double* R, size_t nr, int m) {
    if (nr == 0) throw std::invalid_argument("igd: empty reference front");
    if (na == 0) return std::numeric_limits<double>::infinity();
    double total = 0.0;
    for (size_t r = 0; r < nr; ++r) {
        double best = std::numeric_limits<double>::infinity();
        for (size_t a = 0; a < na; ++a) {
            double s = 0.0;
            for (int c = 0; c < m; ++c) {
                double d = A[a * m + c] - R[r * m + c];
                s += d * d;
            }
            best = std::min(best, s);
        }
        total += std::sqrt(best);
    }
    return total / static_cast<double>(nr);
}

// metrics.cpp:155-175 — feasible, dedup (first kept), nondominated rows
std::vector<size_t> metric_front(const double* F, const double* cv, size_t n, int m) {
    std::vector<size_t> feas;
    for (size_t i = 0; i < n; ++i)
        if (cv[i] == 0.0) feas.push_back(i);
    std::vector<size_t> keep;
    for (size_t a = 0; a < feas.size(); ++a) {
        const double* fa = F + feas[a] * m;
        bool skip = false;
        for (size_t b = 0; b < feas.size() && !skip; ++b) {
            if (a == b) continue;
            const double* fb = F + feas[b] * m;
            if (dominates(fb, fa, m)) skip = true;
            if (b < a && std::equal(fa, fa + m, fb)) skip = true;
        }
        if (!skip) keep.push_back(feas[a]);
    }
    return keep;
}

// metrics.cpp:42-121
std::vector<size_t> hv_relevant(const double* P, size_t n, int m, const double* ref) {
    std::vector<size_t> keep;
    for (size_t i = 0; i < n; ++i) {
        const double* pi = P + i * m;
        bool inside = true;
        for (int c = 0; c < m; ++c)
            if (!(pi[c] < ref[c])) inside = false;
        if (!inside) continue;
        bool skip = false;
        for (size_t j = 0; j < n && !skip; ++j) {
            if (j == i) continue;
            if (dominates(P + j * m, pi, m)) skip = true;
            if (j < i && std::equal(pi, pi + m, P + j * m)) skip = true;
        }
        if (!skip) keep.push_back(i);
    }
    return keep;
}
double hv2(std::vector<std::pair<double, double>> pts, double r0, double r1) {
    if (pts.empty()) return 0.0;
    std::sort(pts.begin(), pts.end());
    double vol = 0.0, prev = r1;
    for (auto [x, y] : pts)
        if (y < prev) { vol += (r0 - x) * (prev - y); prev = y; }
    return vol;
}
double hypervolume(const double* P, size_t n, int m, const double* ref) {
    std::vector<size_t> keep = hv_relevant(P, n, m, ref);
    if (keep.empty()) return 0.0;
    if (m == 2) {
        std::vector<std::pair<double, double>> pts;
        for (size_t i : keep) pts.emplace_back(P[i * 2], P[i * 2 + 1]);
        return hv2(std::move(pts), ref[0], ref[1]);
    }
    if (m == 3) {
        std::vector<size_t> order = keep;
        std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return P[a * 3 + 2] < P[b * 3 + 2]; });
        double vol = 0.0;
        for (size_t k = 0; k < order.size(); ++k) {
            double z0 = P[order[k] * 3 + 2];
            double z1 = k + 1 < order.size() ? P[order[k + 1] * 3 + 2] : ref[2];
            if (z1 <= z0) continue;
            std::vector<std::pair<double, double>> slab;
            for (size_t t = 0; t <= k; ++t) slab.emplace_back(P[order[t] * 3], P[order[t] * 3 + 1]);
            vol += (z1 - z0) * hv2(std::move(slab), ref[0], ref[1]);
        }
        return vol;
    }
    // m > 3: Monte-Carlo estimate, metrics.cpp:95-121 — 10^6 samples of
    // mt19937_64(0x48563D), uniform(lo, ref) = lo + (ref - lo) * (e() >> 11) * 2^-53
    std::vector<double> lo(m, std::numeric_limits<double>::infinity());
    for (size_t i : keep)
        for (int c = 0; c < m; ++c) lo[c] = std::min(lo[c], P[i * m + c]);
    double box = 1.0;
    for (int c = 0; c < m; ++c) box *= ref[c] - lo[c];
    if (box <= 0.0) return 0.0;
    std::mt19937_64 e(0x48563D);
    const size_t samples = 1000000;
    size_t hits = 0;
    std::vector<double> x(m);
    for (size_t s = 0; s < samples; ++s) {
        for (int c = 0; c < m; ++c) x[c] = lo[c] + (ref[c] - lo[c]) * ((double)(e() >> 11) * 0x1.0p-53);
        for (size_t i : keep) {
            bool dom = true;
            for (int c = 0; c < m && dom; ++c)
                if (P[i * m + c] > x[c]) dom = false;
            if (dom) {
                ++hits;
                break;
            }
        }
    }
    return box * (double)hits / (double)samples;
}

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

}  // namespace

// ===========================================================================
extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    orc_philox4x32_10(ctr, key, out);
}

int orc_problem_info(const char* name, int32_t* d, int32_t* m, int32_t* nin, int32_t* neq,
                     double* lo, double* hi) {
    return guarded([&] {
        Problem p = make_problem(name);
        *d = p.d; *m = p.m; *nin = p.nin; *neq = p.neq;
        if (lo) std::copy(p.lo.begin(), p.lo.end(), lo);
        if (hi) std::copy(p.hi.begin(), p.hi.end(), hi);
    });
}

// problems.cpp:552-573 + gmpea.cpp:15-23 (evaluate + cv)
int orc_evaluate(const char* name, const double* X, int64_t n, double* F, double* G, double* cv) {
    return guarded([&] {
        Problem p = make_problem(name);
        std::string bad;
        for (int64_t r = 0; r < n; ++r)
            for (int c = 0; c < p.d; ++c)
                if (!(X[r * p.d + c] >= p.lo[c] && X[r * p.d + c] <= p.hi[c])) {
                    bad += " " + std::to_string(r);
                    break;
                }
        if (!bad.empty()) throw std::invalid_argument("evaluate: out-of-bounds rows:" + bad);
        int nc = p.nin + p.neq;
        for (int64_t r = 0; r < n; ++r) {
            eval_row(p, X + r * p.d, F + r * p.m, G + r * nc);
            if (cv) cv[r] = cv_raw(G + r * nc, p.nin, p.neq);
        }
    });
}

// opaque problem handle for hot loops (used by the reference-loop baseline to
// wrap the restated MW evaluators as reference ProblemDefs)
void* orc_problem_new(const char* name) {
    try {
        return new Problem(make_problem(name));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void orc_problem_free(void* h) { delete static_cast<Problem*>(h); }
// restated front candidates by name (MW / DAS-CMOP): rows, or -1
int64_t orc_front_candidates(const char* name, int64_t n_samples, double* out, int64_t cap) {
    try {
        Problem p = make_problem(name);
        if (!restated_front(p)) throw std::invalid_argument("no restated front for " + p.name);
        const int64_t rows = restated_front_rows(p, n_samples);
        if (out) {
            if (rows * p.d > cap) throw std::invalid_argument("front_candidates: cap too small");
            restated_front_candidates(p, n_samples, out);
        }
        return rows;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int64_t orc_problem_front_rows(const void* h, int64_t n_samples) {
    const Problem& p = *static_cast<const Problem*>(h);
    return restated_front(p) ? restated_front_rows(p, n_samples) : -1;
}
void orc_problem_front_candidates(const void* h, int64_t n_samples, double* out) {
    restated_front_candidates(*static_cast<const Problem*>(h), n_samples, out);
}
void orc_problem_eval_row(const void* h, const double* x, double* f, double* g) {
    eval_row(*static_cast<const Problem*>(h), x, f, g);
}

// registers a scenario (as loaded by load_wta) under "WTA-<scenario>"
int orc_wta_register(const char* scenario, int32_t targets, int32_t vehicles, const int32_t* strikes,
                     const int32_t* cap, const double* p) {
    return guarded([&] {
        Wta w;
        w.targets = targets;
        w.vehicles = vehicles;
        w.strikes.assign(strikes, strikes + targets);
        w.cap.assign(cap, cap + vehicles);
        size_t o = 0;
        w.p.resize(targets);
        for (int i = 0; i < targets; ++i)
            for (int k = 0; k < w.strikes[i]; ++k) w.p[i].push_back(p[o++]);
        std::lock_guard<std::mutex> lk(g_wta_mu);
        g_wta_custom[scenario] = w;
    });
}

int orc_wta_scenario(int32_t num, int32_t* targets, int32_t* vehicles, int32_t* strikes,
                     int32_t* cap, double* p) {
    return guarded([&] {
        if (num < 1 || num > 123) throw std::invalid_argument("unknown WTA scenario");
        Wta w = wta_scenario(num);
        *targets = w.targets;
        *vehicles = w.vehicles;
        size_t o = 0;
        for (int i = 0; i < w.targets; ++i) {
            if (strikes) strikes[i] = w.strikes[i];
            for (int k = 0; k < w.strikes[i]; ++k, ++o)
                if (p) p[o] = w.p[i][k];
        }
        if (cap)
            for (int v = 0; v < w.vehicles; ++v) cap[v] = w.cap[v];
    });
}

double orc_pbi(const double* f, const double* w, const double* z, int32_t m, double theta) {
    return pbi(f, w, z, m, theta);
}

double orc_cv(const double* raw, int32_t nin, int32_t neq) { return cv_raw(raw, nin, neq); }

int orc_reference_vectors(int32_t m, int64_t n, double* W) {
    return guarded([&] {
        if (n <= 0) throw std::invalid_argument("reference_vectors: target_n must be positive");
        auto v = reference_vectors(static_cast<size_t>(m), static_cast<size_t>(n));
        std::copy(v.begin(), v.end(), W);
    });
}

int orc_knn(const double* W, int64_t n, int32_t m, int32_t t, uint32_t* out) {
    return guarded([&] {
        if (t > n) throw std::invalid_argument("build_neighborhoods: neighborhood exceeds population");
        knn(W, static_cast<size_t>(n), static_cast<size_t>(m), static_cast<size_t>(t), out);
    });
}

int orc_knn_rows(const double* W, int64_t n, int32_t m, int32_t t, const int64_t* rows, int64_t nrows,
                 uint32_t* out, int32_t threads) {
    return guarded([&] {
        if (t > n) throw std::invalid_argument("build_neighborhoods: neighborhood exceeds population");
        for (int64_t r = 0; r < nrows; ++r)
            if (rows[r] < 0 || rows[r] >= n) throw std::invalid_argument("knn_rows: row out of range");
        knn_rows(W, (size_t)n, (size_t)m, (size_t)t, rows, (size_t)nrows, out, (unsigned)threads);
    });
}

int orc_lattice_knn(int32_t m, int64_t n, int32_t t1, int32_t t2, uint32_t* B1, uint32_t* B2, int32_t threads) {
    return guarded([&] {
        if (t1 > n || t2 > n) throw std::invalid_argument("build_neighborhoods: neighborhood exceeds population");
        lattice_knn((size_t)m, (size_t)n, (size_t)t1, (size_t)t2, B1, B2, (unsigned)threads);
    });
}

int orc_selection_ex(int32_t n, int32_t m, const double* F1, const double* cv1, const double* F2,
                     const double* cv2, const double* Fo1, const double* cvo1, const double* Fo2,
                     const double* cvo2, const double* W, const double* z, double theta, int32_t agg, int32_t t1,
                     const uint32_t* B1, int32_t t2, const uint32_t* B2, int32_t* src1, int32_t* src2,
                     uint8_t* marks1, uint8_t* marks2);

int orc_selection(int32_t n, int32_t m, const double* F1, const double* cv1, const double* F2,
                  const double* cv2, const double* Fo1, const double* cvo1, const double* Fo2,
                  const double* cvo2, const double* W, const double* z, double theta, int32_t t1,
                  const uint32_t* B1, int32_t t2, const uint32_t* B2, int32_t* src1, int32_t* src2,
                  uint8_t* marks1, uint8_t* marks2) {
    return orc_selection_ex(n, m, F1, cv1, F2, cv2, Fo1, cvo1, Fo2, cvo2, W, z, theta, 0, t1, B1, t2, B2, src1,
                            src2, marks1, marks2);
}

int orc_selection_ex(int32_t n, int32_t m, const double* F1, const double* cv1, const double* F2,
                     const double* cv2, const double* Fo1, const double* cvo1, const double* Fo2,
                     const double* cvo2, const double* W, const double* z, double theta, int32_t agg, int32_t t1,
                     const uint32_t* B1, int32_t t2, const uint32_t* B2, int32_t* src1, int32_t* src2,
                     uint8_t* marks1, uint8_t* marks2) {
    return guarded([&] {
        SelIn s{n, m, F1, cv1, F2, cv2, Fo1, cvo1, Fo2, cvo2, W, z, theta, t1, t2, B1, B2, agg};
        selection(s, src1, src2, marks1, marks2);
    });
}

int orc_reproduce(const char* name, const double* X, int64_t n, const uint32_t* nb, int32_t t,
                  int32_t op, const double* params5, double pm_prob, uint64_t seed, uint32_t gen,
                  uint32_t pop, double* off, int32_t* picks, uint32_t slot_base) {
    return guarded([&] {
        Problem p = make_problem(name);
        OpParams prm{params5[0], params5[1], params5[2], params5[3], params5[4], pm_prob};
        reproduce(p, X, static_cast<size_t>(n), nb, static_cast<size_t>(t), op, prm, seed, gen, pop,
                  off, picks, slot_base);
    });
}

// The whole loop of run_gmpea (gmpea.cpp:421-493, k_max semantics) in f64
// with the engine's Philox draws: init (INIT stream) -> per generation
// reproduce x2 (B1 / B2) -> evaluate x2 -> update_ideal -> OP1/OP2/OP3.
// fp32 != 0 rounds the stored state (X, F, C, cv) to fp32 after every step,
// as the engine stores it, so the three arms reference (mt19937, f64) /
// oracle (Philox, f64) / oracle (Philox, fp32 storage) separate the draw
// schema from the arithmetic (the LIRCMOP1 statistics).
int orc_run_gmpea(const char* name, int64_t n64, int64_t k_max, uint64_t seed, int32_t op, int32_t fp32,
                  double* Xout, double* Fout, double* cvout) {
    return guarded([&] {
        const Problem p = make_problem(name);
        const size_t n = static_cast<size_t>(n64), d = p.d, m = p.m, nc = p.nin + p.neq;
        const size_t t1 = std::min<size_t>(5, n), t2 = std::min<size_t>(20, n);
        std::vector<double> W = reference_vectors(m, n);
        std::vector<uint32_t> B1(n * t1), B2(n * t2);
        lattice_knn(m, n, t1, t2, B1.data(), B2.data(), 1);
        auto rnd = [&](std::vector<double>& v) {
            if (fp32)
                for (double& x : v) x = static_cast<double>(static_cast<float>(x));
        };
        struct Pop { std::vector<double> X, F, G, cv; };
        auto eval = [&](Pop& P) {
            P.F.assign(n * m, 0.0);
            P.G.assign(n * nc, 0.0);
            P.cv.assign(n, 0.0);
            for (size_t r = 0; r < n; ++r) {
                for (size_t c = 0; c < d; ++c)
                    if (!(P.X[r * d + c] >= p.lo[c] && P.X[r * d + c] <= p.hi[c]))
                        throw std::runtime_error("run_gmpea: evaluation failed: out-of-bounds row " +
                                                 std::to_string(r));
                eval_row(p, P.X.data() + r * d, P.F.data() + r * m, P.G.data() + r * nc);
                P.cv[r] = cv_raw(P.G.data() + r * nc, p.nin, p.neq);
            }
            rnd(P.F);
            rnd(P.G);
            rnd(P.cv);
        };
        Pop pop[2];
        const uint32_t key[2] = {static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)};
        for (int q = 0; q < 2; ++q) {
            pop[q].X.resize(n * d);
            for (size_t r = 0; r < n; ++r)
                for (size_t c = 0; c < d; ++c) {
                    uint32_t ctr[4] = {static_cast<uint32_t>(r), 0u, orc_tag(q + 1, ORC_STREAM_INIT),
                                       static_cast<uint32_t>(c / 2)};
                    uint32_t o[4];
                    orc_philox4x32_10(ctr, key, o);
                    uint64_t v = (c % 2 == 0) ? ((uint64_t)o[1] << 32 | o[0]) : ((uint64_t)o[3] << 32 | o[2]);
                    pop[q].X[r * d + c] = p.lo[c] + (p.hi[c] - p.lo[c]) * (static_cast<double>(v >> 11) * 0x1.0p-53);
                }
            rnd(pop[q].X);
            eval(pop[q]);
        }
        std::vector<double> z(m, std::numeric_limits<double>::infinity());
        auto upd = [&](const Pop& P) {
            for (size_t r = 0; r < n; ++r)
                for (size_t c = 0; c < m; ++c) z[c] = std::min(z[c], P.F[r * m + c]);
        };
        upd(pop[0]);
        upd(pop[1]);
        const OpParams prm{1.0, 20.0, 20.0, 1.0, 0.5, -1.0};
        for (int64_t gen = 1; gen <= k_max; ++gen) {
            Pop off[2];
            for (int q = 0; q < 2; ++q) {
                off[q].X.assign(n * d, 0.0);
                reproduce(p, pop[q].X.data(), n, q ? B2.data() : B1.data(), q ? t2 : t1, op, prm, seed,
                          static_cast<uint32_t>(gen), q + 1, off[q].X.data(), nullptr);
                rnd(off[q].X);
                eval(off[q]);
            }
            upd(off[0]);
            upd(off[1]);
            SelIn s{static_cast<int>(n), static_cast<int>(m), pop[0].F.data(), pop[0].cv.data(), pop[1].F.data(),
                    pop[1].cv.data(), off[0].F.data(), off[0].cv.data(), off[1].F.data(), off[1].cv.data(),
                    W.data(), z.data(), 5.0, static_cast<int>(t1), static_cast<int>(t2), B1.data(), B2.data()};
            std::vector<int32_t> src[2] = {std::vector<int32_t>(n), std::vector<int32_t>(n)};
            selection(s, src[0].data(), src[1].data(), nullptr, nullptr);
            for (int q = 0; q < 2; ++q) {
                Pop next = pop[q];
                for (size_t j = 0; j < n; ++j) {
                    const int32_t c = src[q][j];
                    if (c < 0) continue;
                    const Pop& o = off[c < static_cast<int32_t>(n) ? 0 : 1];
                    const size_t r = static_cast<size_t>(c) % n;
                    std::copy(o.X.begin() + r * d, o.X.begin() + (r + 1) * d, next.X.begin() + j * d);
                    std::copy(o.F.begin() + r * m, o.F.begin() + (r + 1) * m, next.F.begin() + j * m);
                    std::copy(o.G.begin() + r * nc, o.G.begin() + (r + 1) * nc, next.G.begin() + j * nc);
                    next.cv[j] = o.cv[r];
                }
                pop[q] = std::move(next);
            }
        }
        std::copy(pop[0].X.begin(), pop[0].X.end(), Xout);
        std::copy(pop[0].F.begin(), pop[0].F.end(), Fout);
        std::copy(pop[0].cv.begin(), pop[0].cv.end(), cvout);
    });
}

// initial population draws (INIT stream): X[r][c] = lo + (hi - lo) * u53
int orc_init_population(const char* name, int64_t n, uint64_t seed, uint32_t pop, double* X) {
    return guarded([&] {
        Problem p = make_problem(name);
        uint32_t key[2] = {static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)};
        for (int64_t r = 0; r < n; ++r)
            for (int c = 0; c < p.d; ++c) {
                uint32_t ctr[4] = {static_cast<uint32_t>(r), 0u, orc_tag(pop, ORC_STREAM_INIT),
                                   static_cast<uint32_t>(c / 2)};
                uint32_t o[4];
                orc_philox4x32_10(ctr, key, o);
                uint64_t v = (c % 2 == 0) ? ((uint64_t)o[1] << 32 | o[0]) : ((uint64_t)o[3] << 32 | o[2]);
                double u = static_cast<double>(v >> 11) * 0x1.0p-53;
                X[r * p.d + c] = p.lo[c] + (p.hi[c] - p.lo[c]) * u;
            }
    });
}

int orc_igd(const double* A, int64_t na, const double* R, int64_t nr, int32_t m, double* out) {
    return guarded([&] { *out = igd(A, static_cast<size_t>(na), R, static_cast<size_t>(nr), m); });
}

int orc_metric_front(const double* F, const double* cv, int64_t n, int32_t m, int64_t* idx,
                     int64_t* count) {
    return guarded([&] {
        auto k = metric_front(F, cv, static_cast<size_t>(n), m);
        for (size_t i = 0; i < k.size(); ++i) idx[i] = static_cast<int64_t>(k[i]);
        *count = static_cast<int64_t>(k.size());
    });
}

int orc_hypervolume(const double* P, int64_t n, int32_t m, const double* ref, double* out) {
    return guarded([&] { *out = hypervolume(P, static_cast<size_t>(n), m, ref); });
}

}  // extern "C"
