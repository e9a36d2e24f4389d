// Reference-front construction on device: pf_reference (proj/src/fronts.cpp:54-84).
//
// One thread per candidate decision row: the analytic front candidates of the
// problem (problems.cpp:203-393: simplex_weights, dtlz1_front_rows,
// sphere_front_rows, lircmop_front_rows, including the per-row bisections of
// LIRCMOP7-12) are built in fp64 in registers/local memory and evaluated in
// fp64 by the same device evaluators the generation kernel streams fp32 genes
// through (Ev::gene<double>).  The host side (engine.cu) keeps the feasible
// rows, filters them with the nondominated filter of fronts.cpp:15-42 and
// subsamples with subsample_front (fronts.cpp:86-103).
#pragma once
#include "common.cuh"
#include "kernels.cuh"
#include "problems.cuh"

namespace gmpea_b200 {

constexpr int kPfMaxD = 64;
constexpr double kPfPi = 3.141592653589793;

enum : int { PF_LIR = 1, PF_DTLZ1 = 2, PF_SPHERE = 3, PF_LEVEL = 4 };

struct PfParams {
    ProbDev P;
    int kind;             // PF_*
    long long n_samples;  // requested candidates (front_candidates(n))
    long long h;          // simplex_weights grid: (h + 1)(h + 2) / 2 rows; PF_LEVEL m = 3: grid side
    long long rows;       // candidate rows generated
    double alpha, rnum, rden;  // sphere_front_rows parameters
    double* F;            // rows x m
    unsigned char* feas;  // cv == 0
    int* n_oob;           // rows outside the bounds (evaluate rejects them)
};

// simplex_weights (problems.cpp:205-218): row r of the triangular grid,
// i outer (0..h), j inner (0..h - i)
__device__ __forceinline__ void simplex_row(long long r, long long h, double w[3]) {
    long long lo = 0, hi = h;
    auto start = [&](long long i) { return i * (h + 1) - i * (i - 1) / 2; };
    while (lo < hi) {
        const long long mid = (lo + hi + 1) / 2;
        if (start(mid) <= r)
            lo = mid;
        else
            hi = mid - 1;
    }
    const long long i = lo, j = r - start(lo);
    w[0] = (double)i / (double)h;
    w[1] = (double)j / (double)h;
    w[2] = (double)(h - i - j) / (double)h;
}

// ellipse_raw (problems.cpp:54-59) with theta = -pi/4 (cos/sin from the host)
__device__ __forceinline__ double pf_ellipse(const ProbDev& P, double f1, double f2, double p, double q,
                                             double a, double b, double r) {
    const double u = (f1 - p) * P.cth - (f2 - q) * P.sth;
    const double v = (f1 - p) * P.sth + (f2 - q) * P.cth;
    return r - u * u / (a * a) - v * v / (b * b);
}

// lircmop_front_rows (problems.cpp:267-369) for one row
__device__ void lir_front_row(const ProbDev& P, int id, int d, long long r, long long n_samples, double* x) {
    const double n = (double)d;
    if (id <= 12) {
        const double x1 = n_samples == 1 ? 0.0 : (double)r / (double)(n_samples - 1);
        x[0] = x1;
        double g1t = 0.0, g2t = 0.0;
        if (id <= 4) {
            g1t = g2t = 0.5 * (1.0 + 1e-9);
        } else if (id >= 9) {
            const bool sqrt_shape = (id == 10 || id == 11);
            double p, q, a, b, level;
            switch (id) {
                case 9: p = 1.4; q = 1.4; a = 1.5; b = 6.0; level = 2.0; break;
                case 10: p = 1.1; q = 1.2; a = 2.0; b = 4.0; level = 1.0; break;
                case 11: p = 1.2; q = 1.2; a = 1.5; b = 5.0; level = 2.1; break;
                default: p = 1.6; q = 1.6; a = 1.5; b = 6.0; level = 2.5; break;
            }
            auto clear_at = [&](double s) {
                const double f1 = 1.7057 * x1 * s;
                const double f2 = 1.7057 * (sqrt_shape ? 1.0 - sqrt(x1) : 1.0 - x1 * x1) * s;
                if (pf_ellipse(P, f1, f2, p, q, a, b, 0.1) > 0.0) return false;
                return level - (f1 * P.sal + f2 * P.cal - sin(4.0 * kPfPi * (f1 * P.cal - f2 * P.sal))) <= 0.0;
            };
            double s = 1.0;
            if (!clear_at(1.0)) {
                double lo = 1.0, hi = 1.002;
                while (hi < 64.0 && !clear_at(hi)) {
                    lo = hi;
                    hi *= 1.002;
                }
                for (int it = 0; it < 60; ++it) {
                    const double mid = 0.5 * (lo + hi);
                    if (clear_at(mid))
                        hi = mid;
                    else
                        lo = mid;
                }
                s = hi;
            }
            s *= 1.0005;
            g1t = g2t = (s - 1.0) / 10.0;
        } else if (id >= 7) {
            const double f1b = x1 + 0.7057;
            const double f2b = (id == 7 ? 1.0 - sqrt(x1) : 1.0 - x1 * x1) + 0.7057;
            const double pp[3] = {1.2, 2.25, 3.5};
            const double aa[3] = {2.0, 2.5, 2.5};
            const double bb[3] = {6.0, 12.0, 10.0};
            auto clear_at = [&](double u) {
                for (int k = 0; k < 3; ++k)
                    if (pf_ellipse(P, f1b + u, f2b + u, pp[k], pp[k], aa[k], bb[k], 0.1) > 0.0) return false;
                return true;
            };
            double u = 0.0;
            if (!clear_at(0.0)) {
                double lo = 0.0, hi = 0.05;
                while (hi < 16.0 && !clear_at(hi)) {
                    lo = hi;
                    hi += 0.05;
                }
                for (int it = 0; it < 80; ++it) {
                    const double mid = 0.5 * (lo + hi);
                    if (clear_at(mid))
                        hi = mid;
                    else
                        lo = mid;
                }
                u = hi;
            }
            u += 1e-6;
            g1t = g2t = u / 10.0;
        }
        int len1 = 0, len2 = 0;
        for (int j = 2; j < d; j += 2) ++len1;
        for (int j = 1; j < d; j += 2) ++len2;
        const double d1 = len1 ? sqrt(g1t / (double)len1) : 0.0;
        const double d2 = len2 ? sqrt(g2t / (double)len2) : 0.0;
        for (int j = 2; j < d; j += 2) {
            const double base = id <= 4 ? sin(0.5 * kPfPi * x1) : sin(0.5 * (double)(j + 1) * kPfPi * x1 / n);
            x[j] = base <= 0.5 ? base + d1 : base - d1;
        }
        for (int j = 1; j < d; j += 2) {
            const double base = id <= 4 ? cos(0.5 * kPfPi * x1) : cos(0.5 * (double)(j + 1) * kPfPi * x1 / n);
            x[j] = base <= 0.5 ? base + d2 : base - d2;
        }
        return;
    }
    // LIRCMOP13/14: sphere front at the innermost feasible radius
    // (the simplex row is supplied by the caller through x[0..2])
}

// ---- restated fronts of MW / DAS-CMOP (no reference counterpart; mirrors
// oracle/gmpea_oracle.cpp restated_front_candidates).  The objectives depend on
// the position genes and one distance value and are nondecreasing in it, so a
// position's front point is at its smallest feasible distance: located on
// kPfLevels steps of [0, kPfLevelMax], bisected, nudged 1e-9 into the
// feasible side and realised in decision space with equal per-gene shares.
constexpr int kPfLevels = 600;
constexpr double kPfLevelMax = 3.0;

template <class Ev>
__device__ bool pf_level_feasible(const ProbDev& P, const double* pos, double lvl) {
    Ev ev;
    ev.set_level(P, pos, lvl);
    double f[kMaxM];
    bool ok = true;
    ev.finish(P, f, [&](int, double g) { ok = ok && g <= 0.0; });
    return ok;
}

template <class Ev>
__device__ double pf_min_level(const ProbDev& P, const double* pos) {
    for (int k = 0; k <= kPfLevels; ++k) {
        const double lvl = kPfLevelMax * k / kPfLevels;
        if (!pf_level_feasible<Ev>(P, pos, lvl)) continue;
        if (k == 0) return 0.0;
        double lo = kPfLevelMax * (k - 1) / kPfLevels, hi = lvl;
        for (int it = 0; it < 60; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (pf_level_feasible<Ev>(P, pos, mid))
                hi = mid;
            else
                lo = mid;
        }
        return hi * (1.0 + 1e-9);
    }
    return -1.0;
}

template <class T>
__device__ double pf_solve_term(T t, double tau, double a, double b) {
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

__device__ void pf_realize_level(const ProbDev& P, const double* pos, double lvl, double* x) {
    const int n = P.d, m = P.m, nd = n - m + 1;
    for (int k = 0; k + 1 < m; ++k) x[k] = pos[k];
    const double tau = fmax(lvl, 0.0) / nd;
    if (P.fam == FAM_DAS) {
        const bool rast = P.id == 4 || P.id == 5 || P.id == 6 || P.id == 9;
        const double shift = m == 2 ? sin(0.5 * kPfPi * pos[0]) : 0.5;
        const double y = rast ? pf_solve_term([](double v) { return v * v + 1.0 - cos(20.0 * kPfPi * v); }, tau,
                                              0.0, 0.05)
                              : sqrt(tau);
        for (int j = m - 1; j < n; ++j) x[j] = shift + y <= 1.0 ? shift + y : shift - y;
        return;
    }
    const double lo = P.lob(0), hi = P.hib(0);
    const int kd = EvalMw::kind(P.id);
    if (kd == 0) {
        const double e = (double)(n - m);
        const double t = sqrt(-log(1.0 - fmin(tau, 0.999)) / 10.0);
        for (int j = m - 1; j < n; ++j) {
            const double c = 0.5 + (double)j / (2.0 * n);
            const double v = c - t >= 0.0 ? c - t : c + t;
            x[j] = fmin(pow(v, 1.0 / e), hi);
        }
    } else if (kd == 1) {
        const double z = pf_solve_term(
            [n](double v) { return 1.5 + (0.1 / n) * v * v - 1.5 * cos(2.0 * kPfPi * v); }, tau, 0.0, 0.5);
        const double t = sqrt(-log(1.0 - z) / 10.0);
        for (int j = m - 1; j < n; ++j) {
            const double b = (double)j / n;
            x[j] = b + t <= hi ? b + t : b - t;
        }
    } else {
        const double u = sqrt(tau / 2.0);
        for (int j = m - 1; j < n; ++j) {
            const double q = x[j - 1] - 0.5;
            const double v = 1.0 - q * q - u;
            x[j] = v >= lo ? v : fmin(1.0 - q * q + u, hi);
        }
    }
}

__device__ void pf_level_row(const PfParams& p, long long r, double* x) {
    const ProbDev& P = p.P;
    double pos[2] = {0.0, 0.0};
    if (P.m == 2) {
        const double t = p.n_samples == 1 ? 0.0 : (double)r / (double)(p.n_samples - 1);
        pos[0] = (double)P.lob(0) + ((double)P.hib(0) - (double)P.lob(0)) * t;
    } else {
        const long long side = p.h;
        const double s1 = side == 1 ? 0.0 : (double)(r / side) / (double)(side - 1);
        const double s2 = side == 1 ? 0.0 : (double)(r % side) / (double)(side - 1);
        pos[0] = (double)P.lob(0) + ((double)P.hib(0) - (double)P.lob(0)) * s1;
        pos[1] = (double)P.lob(1) + ((double)P.hib(1) - (double)P.lob(1)) * s2;
    }
    const double lvl = P.fam == FAM_MW ? pf_min_level<EvalMw>(P, pos) : pf_min_level<EvalDas>(P, pos);
    pf_realize_level(P, pos, lvl < 0.0 ? 0.0 : lvl, x);
}

__global__ void pf_candidates_kernel(PfParams p) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.rows) return;
    const ProbDev& P = p.P;
    const int d = P.d, m = P.m;
    double x[kPfMaxD];
    for (int j = 0; j < d; ++j) x[j] = 0.5;
    if (p.kind == PF_LIR && P.id <= 12) {
        lir_front_row(P, P.id, d, r, p.n_samples, x);
    } else if (p.kind == PF_LEVEL) {
        pf_level_row(p, r, x);
    } else {
        double w[3];
        simplex_row(r, p.h, w);
        if (p.kind == PF_DTLZ1) {  // dtlz1_front_rows (problems.cpp:221-233)
            const double x1 = w[0] + w[1];
            x[0] = x1;
            x[1] = x1 > 0.0 ? w[0] / x1 : 0.0;
        } else {
            double n2 = 0.0;
            for (int c = 0; c < 3; ++c) n2 += w[c] * w[c];
            const double nrm = sqrt(n2);
            const double v1 = w[0] / nrm, v2 = w[1] / nrm, v3 = w[2] / nrm;
            double x1 = asin(fmin(1.0, v3)) / (0.5 * kPfPi);
            double x2 = (v1 == 0.0 && v2 == 0.0) ? 0.0 : atan2(v2, v1) / (0.5 * kPfPi);
            if (p.kind == PF_LIR) {  // LIRCMOP13/14 (problems.cpp:371-392)
                const double radius = P.id == 13 ? 1.7057 : 1.75 * (1.0 + 1e-9);
                const double g = radius - 1.7057;
                const double off = g > 0.0 ? sqrt(g / (10.0 * (double)(d - 2))) : 0.0;
                x[0] = x1;
                x[1] = x2;
                for (int c = 2; c < d; ++c) x[c] = 0.5 + off;
            } else {  // sphere_front_rows (problems.cpp:237-264)
                if (p.alpha != 1.0) {
                    x1 = pow(x1, 1.0 / p.alpha);
                    x2 = pow(x2, 1.0 / p.alpha);
                }
                x[0] = fmin(fmax(x1, 0.0), 1.0);
                x[1] = fmin(fmax(x2, 0.0), 1.0);
                double t = p.rnum;
                if (p.rden != 0.0) {
                    const double mx = fmax(fmax(v1, v2), v3);
                    t = (1.0 + 1e-9) / sqrt(1.0 - 0.75 * mx * mx);
                }
                const double g = t - 1.0;
                if (g > 0.0) {
                    const double off = sqrt(g / (double)(d - 2));
                    for (int c = 2; c < d; ++c) x[c] = 0.5 + off;
                }
            }
        }
    }
    // evaluate (problems.cpp:552-573) in fp64; out-of-bounds rows are counted
    // (the reference's evaluate would reject them)
    bool oob = false;
    for (int j = 0; j < d; ++j)
        if (!(x[j] >= P.lob(j) && x[j] <= P.hib(j))) oob = true;
    if (oob) atomicAdd(p.n_oob, 1);
    double f[kMaxM] = {0.0, 0.0, 0.0};
    Emitter em{nullptr, {}, 0.0, false};
    em.cv.init(P.nin);
    if (P.fam == FAM_LIR) {
        EvalLir ev;
        ev.begin(P);
        for (int j = 0; j < d; ++j) ev.gene(P, j, x[j]);
        ev.finish(P, f, em);
    } else if (P.fam == FAM_MW) {
        EvalMw ev;
        ev.begin(P);
        for (int j = 0; j < d; ++j) ev.gene(P, j, x[j]);
        ev.finish(P, f, em);
    } else if (P.fam == FAM_DAS) {
        EvalDas ev;
        ev.begin(P);
        for (int j = 0; j < d; ++j) ev.gene(P, j, x[j]);
        ev.finish(P, f, em);
    } else {
        EvalDtlz ev;
        ev.begin(P);
        for (int j = 0; j < d; ++j) ev.gene(P, j, x[j]);
        ev.finish(P, f, em);
    }
    for (int c = 0; c < m; ++c) p.F[r * m + c] = f[c];
    p.feas[r] = !oob && em.result() == 0.0;
}

// subsample_front picks (fronts.cpp:98-101): out[r] = rows[order[r (n - 1) / (k - 1)]]
__global__ void pf_pick_kernel(const double* F, const long long* order, long long n, long long k, int m,
                               double* out) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= k) return;
    const long long pick = r * (n - 1) / (k - 1 == 0 ? 1 : k - 1);
    const long long a = order[pick];
    for (int c = 0; c < m; ++c) out[r * m + c] = F[a * m + c];
}

}  // namespace gmpea_b200
