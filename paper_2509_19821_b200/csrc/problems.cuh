// Batched CMOP evaluation on device, streamed gene by gene.
//
// A child is produced one gene at a time by the variation loop and handed to
// Eval::gene(j, x) in ascending j, so no problem needs the whole decision row
// in registers (D = 252 for WTA-P10).  Eval::finish() forms the objectives and
// raw constraints (<= 0 feasible) exactly as the reference does:
//   LIRCMOP1-14    proj/src/problems.cpp:22-137
//   C-/DC-DTLZ     proj/src/problems.cpp:141-201,426-525
//   WTA P1-P10     proj/src/wta.cpp:51-129 (decode = per-vehicle top-capacity,
//                  which equals the reference's global stable sort because the
//                  vehicles are independent)
//   MW1-MW14       not in the reference; restated from the MW
//                  suite (Ma & Wang 2019, PlatEMO conventions), parity
//                  unpinned, mirrored by oracle/gmpea_oracle.cpp eval_mw.
//   DASCMOP1-9     not in the reference either; restated from Fan et al. 2020
//                  (difficulty triplet (0.5, 0.5, 0.5)), parity unpinned,
//                  mirrored by oracle/gmpea_oracle.cpp eval_das.
// Precision policy: inputs are fp32; sums, products and the
// per-individual transcendental terms are evaluated in fp64 (B200 runs fp64
// at half the fp32 rate), the per-gene trigonometric terms of LIRCMOP5-12 in
// fp32 (argument < pi/2, error < 2e-7).  Outputs are rounded to fp32.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace gmpea_b200 {

enum : int { FAM_LIR = 1, FAM_DTLZ = 2, FAM_WTA = 3, FAM_MW = 4, FAM_DAS = 5 };
enum : int {
    C1_DTLZ1 = 1, C1_DTLZ3, C2_DTLZ2, C3_DTLZ4, DC1_DTLZ1, DC1_DTLZ3,
    DC2_DTLZ1, DC2_DTLZ3, DC3_DTLZ1, DC3_DTLZ3
};

// WTA limits: scenarios past P10 and reference-valid
// files (load_wta, wta.cpp:148-192) of up to 64 vehicles and 4096 strike slots.
// Slots <= kWtaNarrowSlots use 32-bit decode keys (slot in 8 bits), larger
// scenarios 64-bit keys (EvalWtaT<true>).  A vehicle's capacity is unlimited:
// it can never take more than one assignment per slot, so its kept list holds
// min(capacity, slots) keys.
constexpr int kWtaMaxVehicles = 64;
constexpr int kWtaMaxSlots = 4096;
constexpr int kWtaNarrowSlots = 256;

struct ProbDev {
    int fam, id, d, m, nin, neq;
    const float* lo;  // d lower bounds
    const float* hi;  // d upper bounds
    int uniform;      // all genes share [ulo, uhi] (every registered suite)
    float ulo, uhi;
    __device__ __forceinline__ float lob(int j) const { return uniform ? ulo : lo[j]; }
    __device__ __forceinline__ float hib(int j) const { return uniform ? uhi : hi[j]; }
    // host-computed constants (glibc values, identical to the reference's)
    double cth, sth;  // cos/sin(-pi/4)  (LIRCMOP5-12 ellipse rotation)
    double cal, sal;  // cos/sin(pi/4)   (LIRCMOP9-12 alpha)
    // WTA scenario tables (wta.hpp:17-28)
    int wta_targets, wta_vehicles, wta_slots;
    const int* wta_cap;          // per vehicle
    const int* wta_strikes;      // per target
    const int* wta_slot_target;  // per strike slot
    const double* wta_p;         // per strike slot
    // streaming decode state (EvalWta): per-vehicle capacity and the offset
    // of its candidate list in the per-thread scratch; total scratch words
    int wta_capv[kWtaMaxVehicles];
    int wta_base[kWtaMaxVehicles];
    int wta_ncap, wta_n32, wta_n8;  // scratch: 32-bit words, and 8-byte units for sizing
};

// c·pi·x trigonometry.  The generation path uses the exact-pi forms
// (sinpi/cospi).  fp64 front candidates (pf_reference) round c·pi·x first, as
// problems.cpp does, so that e.g. cos(pi/2) is 6.1e-17 as with glibc:
// subsample_front orders the front lexicographically by those values.
constexpr double kPiD = 3.141592653589793;
__device__ __forceinline__ double trig_sin(bool ref, double c, double x) { return ref ? sin(c * kPiD * x) : sinpi(c * x); }
__device__ __forceinline__ double trig_cos(bool ref, double c, double x) { return ref ? cos(c * kPiD * x) : cospi(c * x); }

// ---------------------------------------------------------------- LIRCMOP
// SUB > 0 fixes the sub-family at compile time (1: LIRCMOP1-4, 5: 5-8,
// 9: 9-12, 13: 13-14) so the per-gene code carries no problem dispatch.
template <int SUB = 0>
struct EvalLirT {
    static constexpr bool kStream = false;
    __device__ __forceinline__ void bind(void*, int, int) {}
    double g1, g2, x0, x1, s0, c0;
    float x0f;
    bool ref;  // fp64 candidate rows: reference-rounded trigonometry
    __device__ __forceinline__ void begin(const ProbDev&) {
        g1 = g2 = 0.0;
        ref = false;
    }
    __device__ __forceinline__ static int sub_of(int id) {
        return SUB ? SUB : (id <= 4 ? 1 : (id <= 8 ? 5 : (id <= 12 ? 9 : 13)));
    }
    // T = float: generation rows (fp32); T = double: reference-front
    // candidates (pf_reference), evaluated fully in fp64
    template <class T>
    __device__ __forceinline__ void gene(const ProbDev& P, int j, T xf) {
        const double x = xf;
        const int sub = sub_of(P.id);
        ref = std::is_same<T, double>::value;
        if (j == 0) {
            x0 = x;
            x0f = (float)xf;
            if (sub == 1) {  // problems.cpp:23-24
                if (ref) {
                    s0 = trig_sin(true, 0.5, x);
                    c0 = trig_cos(true, 0.5, x);
                } else {
                    sincospi(0.5 * x, &s0, &c0);
                }
            }
            return;
        }
        if (sub == 13) {  // problems.cpp:124-128
            if (j == 1) {
                x1 = x;
                return;
            }
            double t = x - 0.5;
            g1 += 10.0 * t * t;
            return;
        }
        double track;
        if (sub == 1) {
            track = (j & 1) ? c0 : s0;
        } else if (std::is_same<T, double>::value) {  // problems.cpp:43-50 in fp64
            const double a = 0.5 * (double)(j + 1) * kPiD * x0 / (double)P.d;
            track = (j & 1) ? cos(a) : sin(a);
        } else {  // problems.cpp:43-50: sin/cos(0.5 (j+1) pi x1 / n)
            float a = __fdiv_rn(0.5f * (float)(j + 1) * x0f, (float)P.d);
            track = (j & 1) ? (double)cospif(a) : (double)sinpif(a);
        }
        double t = x - track;
        if (j & 1)
            g2 += t * t;
        else
            g1 += t * t;
    }
    __device__ static double ellipse(const ProbDev& P, double f1, double f2, double p, double q,
                                     double a, double b) {
        double u = (f1 - p) * P.cth - (f2 - q) * P.sth;
        double v = (f1 - p) * P.sth + (f2 - q) * P.cth;
        return 0.1 - u * u / (a * a) - v * v / (b * b);
    }
    template <class G>
    __device__ __forceinline__ void finish(const ProbDev& P, double* f, G&& emit) {
        const int id = P.id;
        const int sub = sub_of(id);
        if (sub == 1) {
            f[0] = x0 + g1;
            f[1] = (id == 1 || id == 3) ? 1.0 - x0 * x0 + g2 : 1.0 - sqrt(x0) + g2;
            emit(0, -((0.51 - g1) * (g1 - 0.5)));
            emit(1, -((0.51 - g2) * (g2 - 0.5)));
            if (id >= 3) emit(2, 0.5 - trig_sin(ref, 20.0, x0));
            return;
        }
        if (sub == 5) {
            f[0] = x0 + 10.0 * g1 + 0.7057;
            bool sq = (id == 5 || id == 7);
            f[1] = (sq ? 1.0 - sqrt(x0) : 1.0 - x0 * x0) + 10.0 * g2 + 0.7057;
            if (id <= 6) {
                double p0 = id == 5 ? 1.6 : 1.8, p1 = id == 5 ? 2.5 : 2.8;
                double b0 = id == 5 ? 4.0 : 8.0;
                emit(0, ellipse(P, f[0], f[1], p0, p0, 2.0, b0));
                emit(1, ellipse(P, f[0], f[1], p1, p1, 2.0, 8.0));
            } else {
                emit(0, ellipse(P, f[0], f[1], 1.2, 1.2, 2.0, 6.0));
                emit(1, ellipse(P, f[0], f[1], 2.25, 2.25, 2.5, 12.0));
                emit(2, ellipse(P, f[0], f[1], 3.5, 3.5, 2.5, 10.0));
            }
            return;
        }
        if (sub == 9) {
            f[0] = 1.7057 * x0 * (10.0 * g1 + 1.0);
            bool sq = (id == 10 || id == 11);
            f[1] = 1.7057 * (sq ? 1.0 - sqrt(x0) : 1.0 - x0 * x0) * (10.0 * g2 + 1.0);
            double p, q, a, b, lv;
            switch (id) {
                case 9: p = 1.4; q = 1.4; a = 1.5; b = 6.0; lv = 2.0; break;
                case 10: p = 1.1; q = 1.2; a = 2.0; b = 4.0; lv = 1.0; break;
                case 11: p = 1.2; q = 1.2; a = 1.5; b = 5.0; lv = 2.1; break;
                default: p = 1.6; q = 1.6; a = 1.5; b = 6.0; lv = 2.5; break;
            }
            emit(0, ellipse(P, f[0], f[1], p, q, a, b));
            emit(1, lv - (f[0] * P.sal + f[1] * P.cal - trig_sin(ref, 4.0, f[0] * P.cal - f[1] * P.sal)));
            return;
        }
        double rad = 1.7057 + g1;
        double s1, c1;
        if (ref) {
            s0 = trig_sin(true, 0.5, x0);
            c0 = trig_cos(true, 0.5, x0);
            s1 = trig_sin(true, 0.5, x1);
            c1 = trig_cos(true, 0.5, x1);
        } else {
            sincospi(0.5 * x0, &s0, &c0);
            sincospi(0.5 * x1, &s1, &c1);
        }
        f[0] = rad * c0 * c1;
        f[1] = rad * c0 * s1;
        f[2] = rad * s0;
        double r2 = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
        emit(0, -((r2 - 9.0) * (r2 - 4.0)));
        emit(1, -((r2 - 3.61) * (r2 - 3.24)));
        if (id == 14) emit(2, -((r2 - 3.0625) * (r2 - 2.56)));
    }
};
using EvalLir = EvalLirT<0>;

// ---------------------------------------------------------------- C/DC-DTLZ
// ID > 0 fixes the C/DC-DTLZ problem at compile time (per-problem generation kernels)
template <int ID = 0>
struct EvalDtlzT {
    static constexpr bool kStream = false;
    __device__ __forceinline__ void bind(void*, int, int) {}
    double pos[2];
    double rast, sph;
    bool ref;  // fp64 candidate rows: reference-rounded trigonometry
    __device__ __forceinline__ void begin(const ProbDev&) {
        rast = sph = 0.0;
        ref = false;
    }
    template <class T>
    __device__ __forceinline__ void gene(const ProbDev& P, int j, T xf) {
        const double x = xf;
        ref = std::is_same<T, double>::value;
        if (j < P.m - 1) {  // static indices keep pos[] in registers
            if (j == 0)
                pos[0] = x;
            else
                pos[1] = x;
            return;
        }
        double t = x - 0.5;  // problems.cpp:144-147, 153-155
        // (fp64 cosine: DC2/DC3-DTLZ feed 100 g into cos(3 pi .), which turns
        // an fp32 cosine's 1e-7 per term into 1e-4 in the constraints)
        rast += t * t - trig_cos(ref, 20.0, t);
        sph += t * t;
    }
    __device__ static void shape(int base, const double* pos, double g, double* f, bool ref) {
        // m = 3 (problems.cpp:160-178)
        if (base == 1) {
            f[0] = 0.5 * pos[0] * pos[1] * (1.0 + g);
            f[1] = 0.5 * pos[0] * (1.0 - pos[1]) * (1.0 + g);
            f[2] = 0.5 * (1.0 - pos[0]) * (1.0 + g);
        } else {
            double s0, c0, s1, c1;
            if (ref) {
                s0 = trig_sin(true, 0.5, pos[0]);
                c0 = trig_cos(true, 0.5, pos[0]);
                s1 = trig_sin(true, 0.5, pos[1]);
                c1 = trig_cos(true, 0.5, pos[1]);
            } else {
                sincospi(0.5 * pos[0], &s0, &c0);
                sincospi(0.5 * pos[1], &s1, &c1);
            }
            f[0] = (1.0 + g) * c0 * c1;
            f[1] = (1.0 + g) * c0 * s1;
            f[2] = (1.0 + g) * s0;
        }
    }
    template <class G>
    __device__ __forceinline__ void finish(const ProbDev& P, double* f, G&& emit) {
        const int k = (ID ? ID : P.id);
        const int m = P.m;
        const double gr = 100.0 * ((double)(P.d - m + 1) + rast);
        switch (k) {
            case C1_DTLZ1: {
                shape(1, pos, gr, f, ref);
                emit(0, f[0] / 0.5 + f[1] / 0.5 + f[2] / 0.6 - 1.0);
                return;
            }
            case C1_DTLZ3: {
                shape(2, pos, gr, f, ref);
                double r2 = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
                emit(0, -((r2 - 16.0) * (r2 - 81.0)));
                return;
            }
            case C2_DTLZ2: {
                shape(2, pos, sph, f, ref);
                const double r = 0.4;
                double v1 = 1.0 / 0.0;
                for (int i = 0; i < 3; ++i) {
                    double t = (f[i] - 1.0) * (f[i] - 1.0) - r * r;
                    for (int j = 0; j < 3; ++j)
                        if (j != i) t += f[j] * f[j];
                    v1 = fmin(v1, t);
                }
                const double c = 1.0 / sqrt(3.0);  // correctly rounded, as glibc
                double v2 = 0.0;
                for (int i = 0; i < 3; ++i) v2 += (f[i] - c) * (f[i] - c);
                v2 -= r * r;
                emit(0, fmin(v1, v2));
                return;
            }
            case C3_DTLZ4: {
                double pp[2] = {pow(pos[0], 100.0), pow(pos[1], 100.0)};
                shape(2, pp, sph, f, ref);
                for (int j = 0; j < 3; ++j) {
                    double s = f[j] * f[j] / 4.0;
                    for (int i = 0; i < 3; ++i)
                        if (i != j) s += f[i] * f[i];
                    emit(j, 1.0 - s);
                }
                return;
            }
            default: break;
        }
        bool linear = (k == DC1_DTLZ1 || k == DC2_DTLZ1 || k == DC3_DTLZ1);
        shape(linear ? 1 : 2, pos, gr, f, ref);
        if (k == DC1_DTLZ1 || k == DC1_DTLZ3) {
            emit(0, -(trig_cos(ref, 3.0, pos[0]) + 0.5));
        } else if (k == DC2_DTLZ1 || k == DC2_DTLZ3) {
            emit(0, 0.9 - trig_cos(ref, 3.0, gr));
            emit(1, 0.9 - exp(-gr));
        } else {
            emit(0, -(trig_cos(ref, 3.0, pos[0]) + 0.5));
            emit(1, -(trig_cos(ref, 3.0, pos[1]) + 0.5));
            emit(2, -(trig_cos(ref, 3.0, gr) + 0.5));
        }
    }
};
using EvalDtlz = EvalDtlzT<0>;
template <class Ev>
struct is_dtlz : std::false_type {};
template <int ID>
struct is_dtlz<EvalDtlzT<ID>> : std::true_type {};

// ---------------------------------------------------------------- MW (unpinned)
__device__ __forceinline__ double ipow(double x, int e) {
    double r = 1.0;
    if (e >= 0 && e < 32) {  // square-and-multiply, unrolled (same product order)
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            if (e & (1 << k)) r *= x;
            x *= x;
        }
        return r;
    }
    while (e) {
        if (e & 1) r *= x;
        x *= x;
        e >>= 1;
    }
    return r;
}

// ID > 0 fixes the MW problem at compile time (the generation kernels at
// d = 15: one kernel per problem, no problem dispatch in the hot code)
template <int ID = 0>
struct EvalMwT {
    static constexpr bool kStream = false;
    __device__ __forceinline__ void bind(void*, int, int) {}
    double xs[2];
    double prev;
    double gs;
    int kd;
    bool ref;  // fp64 front candidates: reference-rounded trigonometry (trig_sin)
    __device__ __forceinline__ void begin(const ProbDev& P) {
        gs = 0.0;
        kd = kind(ID ? ID : P.id);
        ref = false;
    }
    __device__ __forceinline__ static int kind(int id) {
        // 0: exp distance (MW1/4/5/9/12), 1: cos distance (2/6/8/10/13), 2: linear (3/7/11/14)
        switch (id) {
            case 1: case 4: case 5: case 9: case 12: return 0;
            case 2: case 6: case 8: case 10: case 13: return 1;
            default: return 2;
        }
    }
    // front candidates (pf_reference): the distance value itself
    __device__ __forceinline__ void set_level(const ProbDev& P, const double* pos, double lvl) {
        xs[0] = pos[0];
        xs[1] = pos[1];
        gs = lvl;
        kd = kind(P.id);
        ref = true;
    }
    // T = float: generation rows (fp32 per-gene terms); T = double: front
    // candidates, evaluated fully in fp64
    template <class T>
    __device__ __forceinline__ void gene(const ProbDev& P, int j, T xf) {
        const double x = xf;
        const int n = P.d, m = P.m;
        ref = std::is_same<T, double>::value;
        if (j < m - 1) {  // static indices keep xs[] in registers
            if (j == 0)
                xs[0] = x;
            else
                xs[1] = x;
            prev = x;
            return;
        }
        // per-gene terms: argument in fp64, the exponential / cosine in fp32
        // (each term < 1e-7 off; the sum accumulates in fp64)
        // (MUFU exp2 for the exponential: argument in [-25, 0], ~2 ulp)
        if (std::is_same<T, double>::value) {  // oracle form (mw_g_exp / _cos / _lin)
            if (kd == 0) {
                double t = pow(x, (double)(n - m)) - 0.5 - (double)j / (2.0 * n);
                gs += 1.0 - exp(-10.0 * t * t);
            } else if (kd == 1) {
                double t = x - (double)j / n;
                double z = 1.0 - exp(-10.0 * t * t);
                gs += 1.5 + (0.1 / n) * z * z - 1.5 * trig_cos(true, 2.0, z);
            } else {
                double q = prev - 0.5;
                double t = x + q * q - 1.0;
                gs += 2.0 * t * t;
            }
            prev = x;
            return;
        }
        if (kd == 0) {
            const int e = n - m;  // 13 or 12 for the registered D = 15
            const double x2 = x * x, x4 = x2 * x2, x8 = x4 * x4;
            const double xe = e == 13 ? x8 * x4 * x : (e == 12 ? x8 * x4 : ipow(x, e));
            double t = xe - 0.5 - (double)j * (0.5 / n);
            gs += 1.0 - (double)__expf((float)(-10.0 * t * t));
        } else if (kd == 1) {
            double t = x - (double)j * (1.0 / n);
            double z = 1.0 - (double)__expf((float)(-10.0 * t * t));
            gs += 1.5 + (0.1 / n) * z * z - 1.5 * (double)cospif((float)(2.0 * z));
        } else {
            double p = prev - 0.5;
            double t = x + p * p - 1.0;
            gs += 2.0 * t * t;
        }
        prev = x;
    }
    template <class G>
    __device__ __forceinline__ void finish(const ProbDev& P, double* f, G&& emit) {
        const int id = ID ? ID : P.id, n = P.d;
        const double r2 = sqrt(2.0);
        switch (id) {
            case 1: case 2: {
                double g = 1.0 + gs;
                f[0] = xs[0];
                f[1] = id == 1 ? g * (1.0 - 0.85 * f[0] / g) : g * (1.0 - f[0] / g);
                double l = r2 * f[1] - r2 * f[0];
                emit(0, f[0] + f[1] - 1.0 - 0.5 * ipow(trig_sin(ref, id == 1 ? 2.0 : 3.0, l), 8));
                return;
            }
            case 3: {
                double g = 1.0 + gs;
                f[0] = xs[0];
                f[1] = g * (1.0 - f[0] / g);
                double l = r2 * f[1] - r2 * f[0];
                double s = f[0] + f[1];
                double sn = trig_sin(ref, 0.75, l);
                emit(0, s - 1.05 - 0.45 * ipow(sn, 6));
                emit(1, 0.85 - s + 0.3 * sn * sn);
                return;
            }
            case 4: case 8: {
                double g = gs;
                // registered with m = 3: f = (1+g)(c0 c1, c0 s1, s0)
                double c[2], s[2];
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    if (id == 4) {
                        c[i] = xs[i];
                        s[i] = 1.0 - xs[i];
                    } else {
                        if (ref) {
                            s[i] = trig_sin(true, 0.5, xs[i]);
                            c[i] = trig_cos(true, 0.5, xs[i]);
                        } else {
                            sincospi(0.5 * xs[i], &s[i], &c[i]);
                        }
                    }
                }
                f[0] = (1.0 + g) * c[0] * c[1];
                f[1] = (1.0 + g) * c[0] * s[1];
                f[2] = (1.0 + g) * s[0];
                if (id == 4) {
                    double l = f[2] - f[0] - f[1];
                    double sum = f[0] + f[1] + f[2];
                    emit(0, sum - (1.0 + 0.4 * ipow(trig_sin(ref, 2.5, l), 8)));
                } else {
                    double q = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
                    double l = asin(f[2] / sqrt(q));
                    double sn = sin(6.0 * l);
                    double t = 1.25 - 0.5 * sn * sn;
                    emit(0, q - t * t);
                }
                return;
            }
            case 5: {
                double g = 1.0 + gs;
                f[0] = g * xs[0];
                double r = f[0] / g;
                f[1] = g * sqrt(1.0 - r * r);
                double l1 = atan(f[1] / f[0]);
                double l2 = 0.5 * 3.141592653589793 - 2.0 * fabs(l1 - 0.25 * 3.141592653589793);
                double q = f[0] * f[0] + f[1] * f[1];
                double a = 1.7 - 0.2 * sin(2.0 * l1);
                double s6 = sin(6.0 * l2 * l2 * l2);
                double b = 1.0 + 0.5 * s6, c = 1.0 - 0.45 * s6;
                emit(0, q - a * a);
                emit(1, b * b - q);
                emit(2, c * c - q);
                return;
            }
            case 6: {
                double g = 1.0 + gs;
                f[0] = g * xs[0] * 1.0999;
                double r = f[0] / g;
                f[1] = g * sqrt(1.1 * 1.1 - r * r);
                double l = ipow(cos(6.0 * ipow(atan(f[1] / f[0]), 4)), 10);
                double a = f[0] / (1.0 + 0.15 * l), b = f[1] / (1.0 + 0.75 * l);
                emit(0, a * a + b * b - 1.0);
                return;
            }
            case 7: {
                double g = 1.0 + gs;
                f[0] = g * xs[0];
                double r = f[0] / g;
                f[1] = g * sqrt(1.0 - r * r);
                double q = f[0] * f[0] + f[1] * f[1];
                double sn;
                if (ref) {  // front candidates: the reference's own rounding
                    sn = sin(4.0 * atan(f[1] / f[0]));
                } else {
                    // sin(4 atan(y / x)) = 4 x y (x^2 - y^2) / (x^2 + y^2)^2 for x, y >= 0
                    // (double-angle identities; no fp64 atan / sin on the generation path)
                    sn = 4.0 * f[0] * f[1] * (f[0] * f[0] - f[1] * f[1]) / (q * q);
                }
                double a = 1.2 + 0.4 * ipow(sn, 16);
                double b = 1.15 - 0.2 * ipow(sn, 8);
                emit(0, q - a * a);
                emit(1, b * b - q);
                return;
            }
            case 9: {
                double g = 1.0 + gs;
                f[0] = g * xs[0];
                f[1] = g * (1.0 - pow(f[0] / g, 0.6));
                double s = f[0] * f[0];
                double t1 = (1.0 - 0.64 * s - f[1]) * (1.0 - 0.36 * s - f[1]);
                double a = f[0] + 0.35, b = f[0] + 0.15;
                // uncontracted (the reference is built -ffp-contract=off): t2 is
                // exactly 0 on the front's end point x1 = 1, g = 1
                double t2 = __dsub_rn(__dsub_rn(__dmul_rn(1.35, 1.35), __dmul_rn(a, a)), f[1]);
                double t3 = __dsub_rn(__dsub_rn(__dmul_rn(1.15, 1.15), __dmul_rn(b, b)), f[1]);
                emit(0, fmin(t1, t2 * t3));
                return;
            }
            case 10: {
                double g = 1.0 + gs;
                f[0] = g * ipow(xs[0], n);
                double r = f[0] / g;
                f[1] = g * (1.0 - r * r);
                double s = f[0] * f[0];
                emit(0, -(2.0 - 4.0 * s - f[1]) * (2.0 - 8.0 * s - f[1]));
                emit(1, (2.0 - 2.0 * s - f[1]) * (2.0 - 16.0 * s - f[1]));
                emit(2, (1.0 - s - f[1]) * (1.2 - 1.2 * s - f[1]));
                return;
            }
            case 11: {
                double g = 1.0 + gs;
                f[0] = g * xs[0] * sqrt(1.9999);
                double r = f[0] / g;
                f[1] = g * sqrt(2.0 - r * r);
                double s = f[0] * f[0];
                emit(0, -(3.0 - s - f[1]) * (3.0 - 4.0 * s - f[1]));
                emit(1, (3.0 - 0.625 * s - f[1]) * (3.0 - 7.0 * s - f[1]));
                emit(2, -(1.62 - 0.18 * s - f[1]) * (1.125 - 0.125 * s - f[1]));
                emit(3, (2.07 - 0.23 * s - f[1]) * (0.63 - 0.07 * s - f[1]));
                return;
            }
            case 12: {
                double g = 1.0 + gs;
                f[0] = g * xs[0];
                double r = f[0] / g;
                f[1] = g * (0.85 - 0.8 * r - 0.08 * fabs(trig_sin(ref, 3.2, r)));
                double a = 1.0 - 0.8 * f[0] - f[1] + 0.08 * trig_sin(ref, 2.0, (f[1] - f[0] / 1.5));
                double b = 1.8 - 1.125 * f[0] - f[1] + 0.08 * trig_sin(ref, 2.0, (f[1] / 1.8 - f[0] / 1.6));
                double c = 1.0 - 0.625 * f[0] - f[1] + 0.08 * trig_sin(ref, 2.0, (f[1] - f[0] / 1.6));
                double e = 1.4 - 0.875 * f[0] - f[1] + 0.08 * trig_sin(ref, 2.0, (f[1] / 1.4 - f[0] / 1.6));
                emit(0, a * b);
                emit(1, -(c * e));
                return;
            }
            case 13: {
                double g = 1.0 + gs;
                f[0] = g * xs[0] * 1.5;
                double r = f[0] / g;
                f[1] = g * (5.0 - exp(r) - fabs(0.5 * trig_sin(ref, 3.0, r)));
                double s3 = 0.5 * trig_sin(ref, 3.0, f[0]);
                double a = 5.0 - exp(f[0]) - s3 - f[1];
                double b = 5.0 - (1.0 + 0.4 * f[0]) - s3 - f[1];
                double c = 5.0 - (1.0 + f[0] + 0.5 * f[0] * f[0]) - s3 - f[1];
                double e = 5.0 - (1.0 + 0.7 * f[0]) - s3 - f[1];
                emit(0, a * b);
                emit(1, -(c * e));
                return;
            }
            default: {  // 14, registered with m = 3
                double g = gs;
                double s = 0.0, sa = 0.0;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    f[k] = xs[k];
                    double q = f[k] * f[k];
                    double sn = trig_sin(ref, 1.1, q);
                    s += 6.0 - exp(f[k]) - 1.5 * sn;
                    sa += 6.1 - (1.0 + f[k] + 0.5 * q + 1.5 * sn);
                }
                f[2] = (1.0 + g) / 2.0 * s;
                emit(0, f[2] - 1.0 / 2.0 * sa);
                return;
            }
        }
    }
};
using EvalMw = EvalMwT<0>;
template <class Ev>
struct is_mw : std::false_type {};
template <int ID>
struct is_mw<EvalMwT<ID>> : std::true_type {};

// ---------------------------------------------------------------- DAS-CMOP (unpinned)
// DAS-CMOP1-9 (Fan et al., Evol. Comput. 28(3), 2020; D = 30, x in [0,1]^D),
// difficulty triplet (eta, zeta, gamma) = (0.5, 0.5, 0.5).  Not in the
// reference; restated from the published definitions and
// mirrored by oracle/gmpea_oracle.cpp eval_das.  Constraints are written in the
// reference's "<= 0 feasible" form:
//   type I   (diversity):    b - sin(a pi x1)  [DAS7-9 also b - cos(a pi x2)], a = 20, b = 2 eta - 1
//   type II  (convergence):  -(e - g)(g - d),  d = 0.5, e = d - ln gamma
//   type III (feasibility):  r - ellipse_k(f)  (DAS1-6, 9 ellipses, r = 0.5 zeta)
//                            r^2 - |f - P_k|^2 (DAS7-9, 4 spheres)
// The per-gene distance terms are fp64 (the DAS4-6/9 Rastrigin cosine has a
// 20 pi argument: fp32 would lose 1e-5 relative in g).
// DAS-CMOP4-6/9 distance terms on generation rows: cos(20 pi y) in fp32 on an
// exactly reduced argument (A/B switch)
#ifndef GMPEA_DAS_COS32
#define GMPEA_DAS_COS32 1
#endif

struct DasConst {
    static constexpr double a = 20.0, b = 0.0;      // b = 2*0.5 - 1
    static constexpr double d = 0.5;
    static constexpr double e = 1.1931471805599454;  // 0.5 - ln(0.5)
    static constexpr double r = 0.25;               // 0.5 * 0.5
    static constexpr double ea = 0.3, eb = 1.2;     // ellipse semi-axes (DAS1-6)
};

// ID > 0 fixes the DAS-CMOP problem at compile time (per-problem generation kernels)
template <int ID = 0>
struct EvalDasT {
    static constexpr bool kStream = false;
    __device__ __forceinline__ void bind(void*, int, int) {}
    double xs[2];
    double sh;  // sin(0.5 pi x1): the position shift of DAS1-6's distance genes
    double gs;
    bool rast;
    bool ref;  // fp64 front candidates: reference-rounded trigonometry (trig_sin)
    __device__ __forceinline__ void begin(const ProbDev& P) {
        gs = 0.0;
        sh = 0.5;
        rast = (ID ? ID : P.id) == 4 || (ID ? ID : P.id) == 5 || (ID ? ID : P.id) == 6 || (ID ? ID : P.id) == 9;
        ref = false;
    }
    // front candidates (pf_reference): g itself
    __device__ __forceinline__ void set_level(const ProbDev& P, const double* pos, double lvl) {
        begin(P);
        xs[0] = pos[0];
        xs[1] = pos[1];
        gs = rast ? lvl - (double)(P.d - P.m + 1) : lvl;
        ref = true;
    }
    template <class T>
    __device__ __forceinline__ void gene(const ProbDev& P, int j, T xf) {
        const double x = xf;
        ref = std::is_same<T, double>::value;
        if (j < P.m - 1) {
            if (j == 0) {
                xs[0] = x;
                if (P.m == 2) sh = trig_sin(ref, 0.5, x);
            } else {
                xs[1] = x;
            }
            return;
        }
        const double y = x - sh;
        if (!rast) {
            gs += y * y;
        } else if (std::is_same<T, double>::value || !GMPEA_DAS_COS32) {
            gs += y * y - trig_cos(ref, 20.0, y);
        } else {
            // generation rows: the cosine in fp32 on an exactly reduced argument
            // (20 y - 2 round(10 y) in [-1, 1], exact in fp64; < 1.2e-7 off per
            // term), the sum in fp64 -- as the MW terms (EvalMwT::gene)
            const double t = 20.0 * y;
            const double r = fma(-2.0, rint(0.5 * t), t);
            gs += y * y - (double)cospif((float)r);
        }
    }
    template <class G>
    __device__ __forceinline__ void finish(const ProbDev& P, double* f, G&& emit) {
        using K = DasConst;
        const int id = (ID ? ID : P.id);
        const double g = rast ? (double)(P.d - P.m + 1) + gs : gs;
        const double x1 = xs[0];
        emit(0, K::b - trig_sin(ref, K::a, x1));
        if (id <= 6) {
            f[0] = x1 + g;
            const int shape = (id - 1) % 3;  // 0: 1 - x^2, 1: 1 - sqrt x, 2: + 0.5|sin 5 pi x|
            f[1] = (shape == 0 ? 1.0 - x1 * x1 : 1.0 - sqrt(x1)) + (shape == 2 ? 0.5 * fabs(trig_sin(ref, 5.0, x1)) : 0.0) + g;
            emit(1, -((K::e - g) * (g - K::d)));
            const double c = 0.7071067811865476, s = -0.7071067811865476;  // cos, sin(-pi/4)
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const double p = k == 0 || k == 2 || k == 5 ? 0.0 : (k == 1 || k == 3 || k == 6 ? 1.0 : (k == 8 ? 3.0 : 2.0));
                const double q = k == 0 || k == 3 || k == 7 ? 1.5 : (k == 1 || k == 4 || k == 8 ? 0.5 : (k == 2 || k == 6 ? 2.5 : 3.5));
                const double u = (f[0] - p) * c - (f[1] - q) * s;
                const double v = (f[0] - p) * s + (f[1] - q) * c;
                emit(2 + k, K::r - (u * u / (K::ea * K::ea) + v * v / (K::eb * K::eb)));
            }
            return;
        }
        const double x2 = xs[1];
        if (id == 7) {
            f[0] = x1 * x2 + g;
            f[1] = x2 * (1.0 - x1) + g;
            f[2] = 1.0 - x2 + g;
        } else {
            double s0, c0, s1, c1;
            if (ref) {
                s0 = trig_sin(true, 0.5, x1);
                c0 = trig_cos(true, 0.5, x1);
                s1 = trig_sin(true, 0.5, x2);
                c1 = trig_cos(true, 0.5, x2);
            } else {
                sincospi(0.5 * x1, &s0, &c0);
                sincospi(0.5 * x2, &s1, &c1);
            }
            f[0] = c0 * c1 + g;
            f[1] = c0 * s1 + g;
            f[2] = s0 + g;
        }
        emit(1, K::b - trig_cos(ref, K::a, x2));
        emit(2, -((K::e - g) * (g - K::d)));
        const double t = 0.5773502691896258;  // 1/sqrt(3)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double px = k == 0 ? 1.0 : (k == 3 ? t : 0.0);
            const double py = k == 1 ? 1.0 : (k == 3 ? t : 0.0);
            const double pz = k == 2 ? 1.0 : (k == 3 ? t : 0.0);
            const double a = f[0] - px, b = f[1] - py, cc = f[2] - pz;
            emit(3 + k, K::r * K::r - (a * a + b * b + cc * cc));
        }
    }
};
using EvalDas = EvalDasT<0>;
template <class Ev>
struct is_das : std::false_type {};
template <int ID>
struct is_das<EvalDasT<ID>> : std::true_type {};

// ---------------------------------------------------------------- WTA
// decode_wta (wta.cpp:51-72): genes >= 0.5 are candidates, taken in
// descending value (ties to the lower flat index) while the vehicle has
// capacity.  Vehicle v = g % vehicles and vehicles are independent, so vehicle
// v keeps exactly its first cap[v] candidates in that order: it selects every
// candidate at or above its cap[v]-th one.  The evaluator works on the whole
// child row (staged in shared memory by the generation kernel): one selection
// pass per capacity unit finds each vehicle's threshold, then one pass over
// the strike slots forms hits, objectives and constraints (wta.cpp:74-110)
// in the reference's order.  No per-thread arrays (no local memory).
// WTA (wta.cpp:51-129), streamed gene by gene.  decode_wta keeps, per vehicle
// v = j mod V, the first cap_v candidates (x_j >= 0.5) in (value desc, index
// asc) order; only that set matters, so each thread keeps per vehicle the
// cap_v best keys seen so far (key = value bits << 32 | ~j: larger = earlier
// in the stable order) and the current minimum, replacing it when a better
// candidate arrives.  finish() turns the kept sets into a selection bitmask,
// counts hits per strike slot and forms f and g in the reference's order.
// The state lives in shared memory as 64-bit words with stride S (one column
// per thread): [lists | counts (V) | minima (V) | mask (ceil(D / 64))].
template <bool WIDE = false>
struct EvalWtaT {
    static constexpr bool kStream = true;
    // decode key: (value rank desc, slot asc) as one unsigned integer
    using Key = typename std::conditional<WIDE, unsigned long long, unsigned>::type;
    static constexpr int KW = WIDE ? 2 : 1;  // 32-bit words per key
    // 32-bit scratch words in shared memory, one column per thread (stride S):
    // [lists (ncap keys) | counts (V) | minima (V keys) | selection mask ((d + 31) / 32)]
    unsigned* L;
    int S;
    int v, slot;  // vehicle and strike slot of the next gene (j = slot V + v)
    __device__ __forceinline__ void bind(void* smem, int tid, int nthreads) {
        L = reinterpret_cast<unsigned*>(smem) + tid;
        S = nthreads;
    }
    __device__ __forceinline__ unsigned& at(int k) const { return L[k * S]; }
    __device__ __forceinline__ Key kget(int k) const {
        if (WIDE) return ((unsigned long long)at(k + 1) << 32) | at(k);
        return (Key)at(k);
    }
    __device__ __forceinline__ void kput(int k, Key key) const {
        at(k) = (unsigned)key;
        if (WIDE) at(k + 1) = (unsigned)((unsigned long long)key >> 32);
    }
    __device__ __forceinline__ static int counts_at(const ProbDev& P) { return P.wta_ncap * KW; }
    __device__ __forceinline__ static int minima_at(const ProbDev& P) { return P.wta_ncap * KW + P.wta_vehicles; }
    __device__ __forceinline__ static int mask_at(const ProbDev& P) {
        return P.wta_ncap * KW + P.wta_vehicles * (1 + KW);
    }
    __device__ __forceinline__ void begin(const ProbDev& P) {
        v = 0;
        slot = 0;
        for (int k = counts_at(P); k < mask_at(P); ++k) at(k) = 0u;  // counts, minima (finish clears the mask)
    }
    // A vehicle's candidates are ranked by (value desc, slot asc), i.e. the
    // reference's stable order restricted to one vehicle (its genes are
    // j = slot V + v).  Candidates lie in [0.5, 1]: the fp32 bit pattern minus
    // that of 0.5 orders them in 24 bits; the slot takes the low byte (narrow)
    // or the low word (WIDE).
    // keeps key among vehicle u's cap_u best (the keys of one vehicle are
    // distinct, so the kept set does not depend on the arrival order)
    __device__ __forceinline__ void insert(const ProbDev& P, int u, Key key) {
        const int cap = P.wta_capv[u], base = P.wta_base[u] * KW;
        const int kc = counts_at(P) + u, km = minima_at(P) + u * KW;
        const int c = (int)at(kc);
        if (c < cap) {
            kput(base + c * KW, key);
            at(kc) = (unsigned)(c + 1);
            if (c + 1 == cap) {
                Key mn = key;
                for (int e = 0; e < c; ++e) mn = min(mn, kget(base + e * KW));
                kput(km, mn);
            }
        } else if (cap > 0 && key > kget(km)) {
            const Key old = kget(km);
            Key mn = key;
            for (int e = 0; e < cap; ++e) {
                Key k2 = kget(base + e * KW);
                if (k2 == old) {
                    kput(base + e * KW, key);
                    k2 = key;
                }
                mn = min(mn, k2);
            }
            kput(km, mn);
        }
    }
    __device__ __forceinline__ static bool candidate(float x) { return x >= 0.5f; }
    __device__ __forceinline__ Key key(float x, int s) const {
        const unsigned rank = __float_as_uint(x) - 0x3F000000u;
        if (WIDE) return ((unsigned long long)rank << 32) | (0xffffffffu - (unsigned)s);
        return (Key)((rank << 8) | (255u - (unsigned)s));
    }
    __device__ __forceinline__ static int slot_of(Key k) {
        return WIDE ? (int)(0xffffffffu - (unsigned)(k & 0xffffffffull)) : (int)(255u - (unsigned)(k & 0xffu));
    }
    // the next ng genes at once (the generation kernel's gene groups): only the
    // candidates (bit k of cand: gene k of the group is >= 0.5, value sel(k))
    // are visited, then the (vehicle, slot) cursor moves on by ng
    template <class Sel>
    __device__ __forceinline__ void group(const ProbDev& P, int ng, unsigned cand, Sel&& sel) {
        const int V = P.wta_vehicles;
        while (cand) {
            const int k = __ffs(cand) - 1;
            cand &= cand - 1u;
            int u = v + k, s = slot;
            while (u >= V) {
                u -= V;
                ++s;
            }
            insert(P, u, key(sel(k), s));
        }
        v += ng;
        while (v >= V) {
            v -= V;
            ++slot;
        }
    }
    __device__ __forceinline__ void gene(const ProbDev& P, int, float x) {
        const int V = P.wta_vehicles;
        if (candidate(x)) insert(P, v, key(x, slot));
        if (++v == V) {
            v = 0;
            ++slot;
        }
    }
    template <class G>
    __device__ __forceinline__ void finish(const ProbDev& P, double* f, G&& emit) {
        const int V = P.wta_vehicles, T = P.wta_targets;
        const int k0 = mask_at(P);  // mask words
        for (int w = 0, nw = (P.d + 31) / 32; w < nw; ++w) at(k0 + w) = 0u;
        for (int u = 0; u < V; ++u) {
            const int c = (int)at(counts_at(P) + u);
            for (int e = 0; e < c; ++e) {
                const unsigned j = (unsigned)slot_of(kget((P.wta_base[u] + e) * KW)) * (unsigned)V + (unsigned)u;
                at(k0 + (int)(j >> 5)) |= 1u << (j & 31);
            }
            emit(u, (double)c - (double)P.wta_cap[u]);  // per-vehicle capacity (wta.cpp:99-100)
        }
        double f1 = 0.0, f2 = 0.0;
        int s = 0;
        for (int i = 0; i < T; ++i) {
            double surv = 1.0, strikes = 0.0;
            for (int k = 0; k < P.wta_strikes[i]; ++k, ++s) {
                // vehicles of slot s: mask bits [s V, s V + V)
                int hits = 0;
                for (int b = s * V, e = b + V; b < e;) {
                    const int w = b >> 5, o = b & 31, take = min(32 - o, e - b);
                    const unsigned bits = at(k0 + w) >> o;
                    hits += __popc(take == 32 ? bits : bits & ((1u << take) - 1u));
                    b += take;
                }
                const double hd = (double)hits;
                surv *= 1.0 - P.wta_p[s] * hd;
                f2 += hd;
                strikes += hd;
            }
            f1 += 1.0 - surv;
            emit(V + i, strikes - (double)P.wta_strikes[i]);  // per-target strikes (wta.cpp:101-109)
        }
        f[0] = -f1;  // wta.cpp:126 (solvers minimise)
        f[1] = f2;
    }
};
using EvalWta = EvalWtaT<false>;

}  // namespace gmpea_b200
