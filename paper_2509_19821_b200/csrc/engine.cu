// GMPEA-B200 engine: host runtime (C++) + C ABI (include/gmpea_b200.h).
//
// The host side owns every device buffer, builds the setup (reference
// vectors, neighbourhoods, reverse lists, initial populations) with kernels,
// captures one generation (vary_eval -> op1 -> select -> end_gen [-> restore])
// as a CUDA graph and replays it.  It mirrors run_gmpea (gmpea.cpp:421-493):
// k_max / eval-budget / time-budget semantics, the discarded crossing
// generation, per-generation GenRecords and the returned pop1.
#include <algorithm>
#include <chrono>
#include <numeric>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gmpea_b200.h"
#include "baselines.cuh"
#include "common.cuh"
#include "fronts.cuh"
#include "kernels.cuh"
#include "metrics.cuh"
#include "problems.cuh"
#include "topology.cuh"

using namespace gmpea_b200;

namespace {

thread_local std::string g_err;

struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(expr)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            throw cuda_error(std::string(#expr) + ": " + cudaGetErrorString(e_));            \
    } while (0)

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return GMPEA_OK;
    } catch (const cuda_error& e) {
        g_err = e.what();
        return GMPEA_ECUDA;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return GMPEA_EINVAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return GMPEA_ERUNTIME;
    }
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t count) {
        if (p) cudaFree(p);
        p = nullptr;
        n = count;
        if (count) CK(cudaMalloc(&p, count * sizeof(T)));
    }
    void zero(cudaStream_t s) {
        if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
};

inline int blocks_for(long long n, int bs) { return (int)((n + bs - 1) / bs); }

void require_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw cuda_error("no CUDA device available (the engine has no CPU fallback)");
}

// ---------------------------------------------------------------- problems
constexpr double kPi = 3.141592653589793;

struct WtaHost {
    std::string scenario;
    int targets = 0, vehicles = 0;
    std::vector<int> strikes, cap;
    std::vector<double> p;  // per strike slot, target-major
};

// wta_scenario (wta.cpp:23-49): sizes grow with the index, tables from the
// reference's seeded mt19937_64 draws (rng.hpp:18-30)
WtaHost wta_scenario(int num) {
    WtaHost w;
    w.scenario = "P" + std::to_string(num);
    w.targets = 4 + 2 * (num - 1);
    w.vehicles = 3 + (num - 1) / 2;
    std::mt19937_64 e(0x57A0000ull + (uint64_t)num);
    auto index = [&](uint64_t n) {
        uint64_t limit = UINT64_MAX - UINT64_MAX % n, v;
        do {
            v = e();
        } while (v >= limit);
        return v % n;
    };
    for (int i = 0; i < w.targets; ++i) w.strikes.push_back(1 + (int)index(3));
    for (int v = 0; v < w.vehicles; ++v) w.cap.push_back(2 + (int)index(3));
    for (int i = 0; i < w.targets; ++i)
        for (int k = 0; k < w.strikes[i]; ++k) w.p.push_back(0.35 + 0.6 * ((double)(e() >> 11) * 0x1.0p-53));
    return w;
}

int mw_ncon(int id) {
    switch (id) {
        case 3: case 7: case 12: case 13: return 2;
        case 5: case 10: return 3;
        case 11: return 4;
        default: return 1;
    }
}

// packs R into int16 offsets for select (pack_reverse_kernel); false when an
// offset does not fit or GMPEA_NO_RPACK is set (select then reads R)
bool device_pack_reverse(cudaStream_t s, int n, int maxdeg, const DevBuf<int>& R, long long ld,
                         const DevBuf<int>& deg, DevBuf<uint2>& Rp) {
    const char* off = getenv("GMPEA_NO_RPACK");
    if (off && *off && *off != '0') return false;
    const int nq = (std::max(maxdeg, 1) + 3) / 4;
    Rp.alloc((size_t)nq * ld);
    DevBuf<int> overflow(1);
    overflow.zero(s);
    pack_reverse_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, deg.p, R.p, ld, nq, Rp.p, overflow.p);
    CK(cudaGetLastError());
    int h = 0;
    CK(cudaMemcpyAsync(&h, overflow.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return h == 0;
}

}  // namespace

struct gmpea_problem {
    std::string name;
    int fam = 0, id = 0, d = 0, m = 0, nin = 0, neq = 0;
    std::vector<double> lo, hi;
    WtaHost wta;
    int device = 0;
    // device copies
    DevBuf<float> dlo, dhi;
    DevBuf<double> dlo64, dhi64;
    DevBuf<int> dcap, dstrikes, dslot_target;
    DevBuf<double> dp;
    ProbDev dev{};

    void upload() {
        require_device();
        CK(cudaGetDevice(&device));
        std::vector<float> lf(lo.begin(), lo.end()), hf(hi.begin(), hi.end());
        dlo.alloc(d);
        dhi.alloc(d);
        dlo64.alloc(d);
        dhi64.alloc(d);
        CK(cudaMemcpy(dlo.p, lf.data(), d * sizeof(float), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dhi.p, hf.data(), d * sizeof(float), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dlo64.p, lo.data(), d * sizeof(double), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dhi64.p, hi.data(), d * sizeof(double), cudaMemcpyHostToDevice));
        dev = ProbDev{};
        dev.fam = fam;
        dev.id = id;
        dev.d = d;
        dev.m = m;
        dev.nin = nin;
        dev.neq = neq;
        dev.lo = dlo.p;
        dev.hi = dhi.p;
        dev.uniform = 1;
        for (int j = 0; j < d; ++j)
            if (lo[j] != lo[0] || hi[j] != hi[0]) dev.uniform = 0;
        dev.ulo = d ? (float)lo[0] : 0.0f;
        dev.uhi = d ? (float)hi[0] : 0.0f;
        // the reference evaluates these with glibc at run time; volatile keeps
        // the host compiler from folding them with a different rounding
        volatile double th = -0.25 * kPi, al = 0.25 * kPi;
        dev.cth = std::cos(th);
        dev.sth = std::sin(th);
        dev.cal = std::cos(al);
        dev.sal = std::sin(al);
        if (fam == FAM_WTA) {
            std::vector<int> st;
            for (int i = 0; i < wta.targets; ++i)
                for (int k = 0; k < wta.strikes[i]; ++k) st.push_back(i);
            dcap.alloc(wta.vehicles);
            dstrikes.alloc(wta.targets);
            dslot_target.alloc(st.size());
            dp.alloc(wta.p.size());
            CK(cudaMemcpy(dcap.p, wta.cap.data(), wta.vehicles * sizeof(int), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dstrikes.p, wta.strikes.data(), wta.targets * sizeof(int), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dslot_target.p, st.data(), st.size() * sizeof(int), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dp.p, wta.p.data(), wta.p.size() * sizeof(double), cudaMemcpyHostToDevice));
            dev.wta_targets = wta.targets;
            dev.wta_vehicles = wta.vehicles;
            dev.wta_slots = (int)st.size();
            dev.wta_cap = dcap.p;
            dev.wta_strikes = dstrikes.p;
            dev.wta_slot_target = dslot_target.p;
            dev.wta_p = dp.p;
            if (wta.vehicles > kWtaMaxVehicles) throw std::invalid_argument("wta: too many vehicles");
            int base = 0;
            for (int v = 0; v < wta.vehicles; ++v) {
                dev.wta_capv[v] = wta.cap[v];
                dev.wta_base[v] = base;
                base += wta.cap[v];
            }
            dev.wta_ncap = base;
            // EvalWta scratch (32-bit words; its keys hold the slot in 8 bits:
            // kWtaMaxSlots <= 256)
            dev.wta_n32 = base + 2 * wta.vehicles + (d + 31) / 32;
            dev.wta_n8 = (dev.wta_n32 + 1) / 2;
        }
    }
};

namespace {

void make_wta(gmpea_problem& p, const WtaHost& w) {
    if (w.targets <= 0 || w.vehicles <= 0) throw std::invalid_argument("WTA: empty scenario");
    if (w.vehicles > kWtaMaxVehicles)
        throw std::invalid_argument("WTA: at most " + std::to_string(kWtaMaxVehicles) + " vehicles");
    int slots = 0;
    for (int s : w.strikes) slots += s;
    if (slots > kWtaMaxSlots) throw std::invalid_argument("WTA: too many strike slots");
    for (int c : w.cap)
        if (c < 0 || c > kWtaMaxCap)
            throw std::invalid_argument("WTA: vehicle capacity above " + std::to_string(kWtaMaxCap));
    p.fam = FAM_WTA;
    p.wta = w;
    p.name = "WTA-" + w.scenario;
    p.d = slots * w.vehicles;
    p.m = 2;
    p.nin = w.vehicles + w.targets;
    p.lo.assign(p.d, 0.0);
    p.hi.assign(p.d, 1.0);
}

std::unique_ptr<gmpea_problem> make_problem(const std::string& name) {
    auto p = std::make_unique<gmpea_problem>();
    p->name = name;
    auto num = [&](size_t pos) {
        try {
            size_t used = 0;
            int v = std::stoi(name.substr(pos), &used);
            if (used != name.size() - pos) return -1;
            return v;
        } catch (...) {
            return -1;
        }
    };
    if (name.rfind("LIRCMOP", 0) == 0) {
        int id = num(7);
        if (id >= 1 && id <= 14) {
            p->fam = FAM_LIR;
            p->id = id;
            p->d = 30;
            p->m = id >= 13 ? 3 : 2;
            p->nin = (id == 3 || id == 4 || id == 7 || id == 8 || id == 14) ? 3 : 2;
            p->lo.assign(p->d, 0.0);
            p->hi.assign(p->d, 1.0);
            return p;
        }
    }
    if (name.rfind("MW", 0) == 0) {
        int id = num(2);
        if (id >= 1 && id <= 14) {
            p->fam = FAM_MW;
            p->id = id;
            p->d = 15;
            p->m = (id == 4 || id == 8 || id == 14) ? 3 : 2;
            p->nin = mw_ncon(id);
            p->lo.assign(p->d, 0.0);
            p->hi.assign(p->d, id == 14 ? 1.5 : 1.0);
            return p;
        }
    }
    if (name.rfind("DASCMOP", 0) == 0 || name.rfind("DAS-CMOP", 0) == 0) {
        int id = num(name[3] == '-' ? 8 : 7);
        if (id >= 1 && id <= 9) {
            p->fam = FAM_DAS;
            p->id = id;
            p->d = 30;
            p->m = id >= 7 ? 3 : 2;
            p->nin = id >= 7 ? 7 : 11;
            p->lo.assign(p->d, 0.0);
            p->hi.assign(p->d, 1.0);
            return p;
        }
    }
    if (name.rfind("WTA-", 0) == 0) {
        std::string sc = name.substr(4);
        int v = sc.size() >= 2 && sc[0] == 'P' ? num(5) : -1;
        if (v < 1 || v > 10) throw std::invalid_argument("unknown WTA scenario: " + sc);
        make_wta(*p, wta_scenario(v));
        p->id = v;
        return p;
    }
    static const char* kDtlz[] = {"C1-DTLZ1", "C1-DTLZ3", "C2-DTLZ2", "C3-DTLZ4", "DC1-DTLZ1",
                                  "DC1-DTLZ3", "DC2-DTLZ1", "DC2-DTLZ3", "DC3-DTLZ1", "DC3-DTLZ3"};
    for (int k = 0; k < 10; ++k)
        if (name == kDtlz[k]) {
            p->fam = FAM_DTLZ;
            p->id = k + 1;
            p->m = 3;
            bool d7 = p->id == C1_DTLZ1 || p->id == DC1_DTLZ1 || p->id == DC2_DTLZ1 || p->id == DC3_DTLZ1;
            p->d = d7 ? 7 : 12;
            if (p->id == C3_DTLZ4)
                p->nin = 3;
            else if (p->id == DC2_DTLZ1 || p->id == DC2_DTLZ3)
                p->nin = 2;
            else if (p->id == DC3_DTLZ1 || p->id == DC3_DTLZ3)
                p->nin = 3;
            else
                p->nin = 1;
            p->lo.assign(p->d, 0.0);
            p->hi.assign(p->d, 1.0);
            return p;
        }
    throw std::invalid_argument("unknown problem: " + name);
}

// ---------------------------------------------------------------- layout helpers
// row-major f64 (n x k) -> columns [0, k) of fp32 rows (stride rs floats),
// with the reference's f64 bounds check (problems.cpp:554-568)
__global__ void to_rows_kernel(const double* in, long long n, int k, float* out, int rs, const double* lo,
                               const double* hi, int* bad, int* nbad) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * k) return;
    const long long r = e / k;
    const int c = (int)(e % k);
    const double v = in[e];
    out[r * rs + c] = (float)v;
    if (lo && !(v >= lo[c] && v <= hi[c])) {
        // one entry per offending row: the first failing column claims it
        bool first = true;
        for (int cc = 0; cc < c; ++cc) {
            double w = in[r * k + cc];
            if (!(w >= lo[cc] && w <= hi[cc])) {
                first = false;
                break;
            }
        }
        if (first) bad[atomicAdd(nbad, 1)] = (int)r;
    }
}

// columns [col0, col0 + k) of fp32 rows -> row-major f64 (n x k)
__global__ void from_rows_kernel(const float* in, int rs, long long n, int col0, int k, double* out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * k) return;
    const long long r = e / k;
    const int c = (int)(e % k);
    out[e] = (double)in[r * rs + col0 + c];
}

__global__ void fcv_from_rows_kernel(const double* F, const double* cv, long long n, int m, float4* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 o = make_float4((float)F[i * m], (float)F[i * m + 1], m > 2 ? (float)F[i * m + 2] : 0.0f,
                           (float)cv[i]);
    out[i] = o;
}

__global__ void fcv_to_rows_kernel(const float4* in, long long n, int m, double* F, double* cv) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 v = in[i];
    F[i * m] = v.x;
    F[i * m + 1] = v.y;
    if (m > 2) F[i * m + 2] = v.z;
    if (cv) cv[i] = v.w;
}

__global__ void u32_to_i32_kernel(const unsigned* in, long long n, int* out, int lim, int* err) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    unsigned v = in[e];
    if (v >= (unsigned)lim) atomicExch(err, 1);
    out[e] = (int)v;
}

__global__ void init_state_kernel(DevState* st, int m) {
    for (int k = 0; k < 4; ++k) st->zbits[k] = k < m ? 0xffffffffu : float_to_ordered(0.0f);
}

__global__ void set_z_kernel(DevState* st, int m, float z0, float z1, float z2) {
    st->zbits[0] = float_to_ordered(z0);
    st->zbits[1] = float_to_ordered(z1);
    st->zbits[2] = m > 2 ? float_to_ordered(z2) : float_to_ordered(0.0f);
}

__global__ void z_of_kernel(const float4* Fcv, long long n, int m, DevState* st) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 v = Fcv[i];
    atomicMin(&st->zbits[0], float_to_ordered(v.x));
    atomicMin(&st->zbits[1], float_to_ordered(v.y));
    if (m > 2) atomicMin(&st->zbits[2], float_to_ordered(v.z));
}

// max |B[i][l] - i| over all rows (the neighbourhood reach)
__global__ void reach_kernel(const int* B, long long n, int t, int* out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * t) return;
    int dlt = B[e] - (int)(e / t);
    atomicMax(out, dlt < 0 ? -dlt : dlt);
}

// rows [r0, r1) of the global table, re-indexed to the local window [e0, ...);
// other local rows point at themselves (never used: variation runs on [r0, r1))
__global__ void slice_topology_kernel(const int* Bg, int t, long long e0, long long nloc, long long r0,
                                      long long r1, int* Bl) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nloc * t) return;
    const long long i = e / t;
    const long long g = e0 + i;
    Bl[e] = (g >= r0 && g < r1) ? (int)(Bg[g * t + e % t] - e0) : (int)i;
}

// individuals as padded fp32 rows [x | g | pad] plus packed keys
struct RowGeom {
    int rs4;   // row stride, float4
    int srs4;  // shared-memory row stride (odd float4 count)
    int bs;    // vary_eval block size
    int stream8;
    size_t smem;
};

// stream8 > 0: a streaming evaluator (no staged row) with that many 64-bit
// shared words per thread
RowGeom row_geom(int d, int nc, int stream8 = 0) {
    RowGeom g;
    g.rs4 = (d + nc + 3) / 4;
    g.srs4 = stream8 > 0 ? 0 : g.rs4 | 1;
    g.stream8 = stream8;
    const int per = stream8 > 0 ? stream8 * 8 : g.srs4 * 16;
    g.bs = per * 128 <= 40 * 1024 ? 128 : (per * 64 <= 40 * 1024 ? 64 : 32);
    g.smem = (size_t)g.bs * per;
    if (g.smem > 48 * 1024) throw std::invalid_argument("problem rows too wide for the engine");
    return g;
}

struct PopBuf {
    DevBuf<float4> X;  // n rows of rs4 float4
    DevBuf<float4> Fcv;
    void alloc(long long n, int rs4, long long ld) {
        X.alloc((size_t)n * rs4);
        Fcv.alloc(ld);
    }
};

// ---------------------------------------------------------------- kernel dispatch
using VaryKernel = void (*)(VaryParams);

// the dimension-specialised generation kernels also assume uniform bounds
// (true of every registered suite; checked by the caller)
template <class Ev, int DC = 0, bool VARY_ONLY = false, bool UBF = false>
VaryKernel pick_vary(int mode, int op, bool tour = false) {
    if (tour) {  // the comparison algorithms: SBX children of tournament parents
        constexpr bool UBT = DC > 0 || UBF;
        return vary_eval_kernel<Ev, MODE_VARY, OP_SBX, DC, UBT, true>;
    }
    if (!VARY_ONLY) {
        if (mode == MODE_EVAL) return vary_eval_kernel<Ev, MODE_EVAL, OP_SBX>;
        if (mode == MODE_INIT) return vary_eval_kernel<Ev, MODE_INIT, OP_SBX>;
    }
    constexpr bool UB = DC > 0 || UBF;  // UBF: uniform bounds at a run-time dimension
    return op == OP_DE ? vary_eval_kernel<Ev, MODE_VARY, OP_DE, DC, UB> : vary_eval_kernel<Ev, MODE_VARY, OP_SBX, DC, UB>;
}

// the generation kernel is compiled for the registered suites' dimension
VaryKernel vary_kernel_for(int fam, int mode, int op, int d = 0, int id = 0, bool tour = false) {
    tour = tour && mode == MODE_VARY;
    switch (fam) {
        case FAM_LIR:
            if (d != 30 || mode != MODE_VARY) return pick_vary<EvalLir>(mode, op, tour);
            return id <= 4 ? pick_vary<EvalLirT<1>, 30, true>(mode, op, tour)
                           : (id <= 8 ? pick_vary<EvalLirT<5>, 30, true>(mode, op, tour)
                                      : (id <= 12 ? pick_vary<EvalLirT<9>, 30, true>(mode, op, tour)
                                                  : pick_vary<EvalLirT<13>, 30, true>(mode, op, tour)));
        case FAM_DTLZ:
            return d == 7 ? pick_vary<EvalDtlz, 7>(mode, op, tour)
                          : (d == 12 ? pick_vary<EvalDtlz, 12>(mode, op, tour) : pick_vary<EvalDtlz>(mode, op, tour));
        case FAM_WTA:
            return d > 0 && mode == MODE_VARY ? pick_vary<EvalWta, 0, true, true>(mode, op, tour)
                                              : pick_vary<EvalWta>(mode, op, tour);
        case FAM_DAS:
            return d == 30 ? pick_vary<EvalDas, 30>(mode, op, tour) : pick_vary<EvalDas>(mode, op, tour);
        default: return d == 15 ? pick_vary<EvalMw, 15>(mode, op, tour) : pick_vary<EvalMw>(mode, op, tour);
    }
}

void launch_vary(VaryKernel k, const VaryParams& vp, int npops, cudaStream_t s) {
    const RowGeom g = [&] {
        RowGeom r;
        r.rs4 = vp.rs4;
        r.srs4 = vp.srs4;
        const int per = vp.scratch8 > 0 ? vp.scratch8 * 8 : r.srs4 * 16;
        r.bs = per * 128 <= 40 * 1024 ? 128 : (per * 64 <= 40 * 1024 ? 64 : 32);
        r.smem = (size_t)r.bs * per;
        return r;
    }();
    k<<<dim3(blocks_for(vp.row_end - vp.row0, g.bs), npops), g.bs, g.smem, s>>>(vp);
}

void fill_op_params(VaryParams& vp, const gmpea_operator_params& prm, int d) {
    vp.sbx_prob = prm.sbx_prob;
    vp.sbx_e = (float)(1.0 / (prm.sbx_eta + 1.0));
    vp.pm_e1 = (float)(prm.pm_eta + 1.0);
    vp.pm_einv = (float)(1.0 / (prm.pm_eta + 1.0));
    const double pm = prm.pm_prob >= 0.0 ? prm.pm_prob : 1.0 / (double)d;
    // PM: skip iff u > pm with u = w 2^-32  <=>  mutate iff w <= floor(pm 2^32)
    const double T = pm * 4294967296.0;
    vp.pm_T = pm < 0.0 ? -1 : (long long)std::min(std::floor(T), 4294967295.0);
    // DE: take iff u < CR  <=>  w < ceil(CR 2^32)  <=>  w <= ceil(CR 2^32) - 1
    const double C = prm.de_cr * 4294967296.0;
    vp.de_T = prm.de_cr >= 1.0 ? 0xffffffffll : (prm.de_cr <= 0.0 ? -1ll : (long long)std::ceil(C) - 1);
    vp.uid = make_uidx((unsigned long long)d);
    vp.de_f = (float)prm.de_f;
}

std::string rows_message(std::vector<int> rows) {
    std::sort(rows.begin(), rows.end());
    std::ostringstream os;
    os << "evaluate: out-of-bounds rows:";
    for (int r : rows) os << ' ' << r;
    return os.str();
}

long long lattice_H(int m, long long n) {
    // reference_vectors: smallest H with C(H + m - 1, m - 1) >= n (gmpea.cpp:62-66)
    auto size = [&](long long H) {
        long long s = 1;
        for (long long i = 1; i < m; ++i) s = s * (H + i) / i;
        return s;
    };
    long long H = 1;
    if (m == 2) return std::max<long long>(1, n - 1);
    while (size(H) < n) ++H;
    return H;
}

// neighbourhoods on device: B1/B2 as int32 (n x t)
void device_knn(cudaStream_t s, int n, int m, int t1, int t2, const double* dW, bool lattice, long long H,
                int* B1, int* B2) {
    if (t1 > n || t2 > n)
        throw std::invalid_argument("build_neighborhoods: neighborhood exceeds population");
    if (t1 < 1 || t2 < 1) throw std::invalid_argument("build_neighborhoods: empty neighbourhood");
    if (std::max(t1, t2) <= kMaxT) {
        const int tmax = std::max(t1, t2);
        // the insertion list keeps the first t1 of the sorted top-tmax
        int* Bbig = t2 >= t1 ? B2 : B1;
        int* Bsmall = t2 >= t1 ? B1 : B2;
        int tsmall = std::min(t1, t2);
        if (lattice && n > 4096) {
            DevBuf<int> retry(1);
            for (int R = 6;; R *= 2) {
                retry.zero(s);
                knn_lattice_kernel<<<blocks_for(n, 128), 128, 0, s>>>(n, m, H, tsmall, tmax, R, dW, Bsmall,
                                                                       Bbig, retry.p);
                CK(cudaGetLastError());
                int flag = 0;
                CK(cudaMemcpyAsync(&flag, retry.p, sizeof(int), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                if (!flag) return;
                if (R > 4096) break;
            }
        }
        knn_brute_kernel<<<blocks_for(n, 128), 128, 0, s>>>(n, m, tsmall, tmax, dW, Bsmall, Bbig);
        CK(cudaGetLastError());
        return;
    }
    knn_select_kernel<<<blocks_for(n, 128), 128, 0, s>>>(n, m, t1, dW, B1);
    knn_select_kernel<<<blocks_for(n, 128), 128, 0, s>>>(n, m, t2, dW, B2);
    CK(cudaGetLastError());
}

// reverse neighbourhood (padded SoA, ascending); returns max in-degree
int device_reverse(cudaStream_t s, int n, int t, const int* B, long long ld, DevBuf<int>& deg,
                   DevBuf<int>& R, int r0 = 0, int r1 = -1) {
    // claimants are the rows [r0, r1) of B (default: all n)
    if (r1 < 0) r1 = n;
    deg.alloc(std::max<long long>(ld, 1));
    deg.zero(s);
    const long long E = (long long)(r1 - r0) * t;
    const int* Bs = B + (long long)r0 * t;
    indegree_kernel<<<blocks_for(E, 256), 256, 0, s>>>(r1 - r0, t, Bs, deg.p);
    CK(cudaGetLastError());
    std::vector<int> h(n);
    CK(cudaMemcpyAsync(h.data(), deg.p, n * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int maxdeg = 0;
    for (int v : h) maxdeg = std::max(maxdeg, v);
    R.alloc((size_t)std::max(maxdeg, 1) * ld);
    DevBuf<int> fill(std::max(n, 1));
    fill.zero(s);
    reverse_fill_kernel<<<blocks_for(E, 256), 256, 0, s>>>(r1 - r0, t, Bs, r0, fill.p, R.p, ld);
    reverse_sort_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, deg.p, R.p, ld);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    return maxdeg;
}

}  // namespace

// ====================================================================== engine
struct gmpea_engine {
    const gmpea_problem* prob = nullptr;
    gmpea_run_config cfg{};
    int n = 0, d = 0, m = 0, nc = 0, t1 = 0, t2 = 0;  // n: local rows
    // shard geometry (global slot indices; unsharded: all equal [0, N))
    long long N = 0, e0 = 0, e1 = 0, v0 = 0, v1 = 0, own0 = 0, own1 = 0, reach = 0;
    bool sharded = false;
    long long ld = 0, H = 0;
    RowGeom geo{};
    cudaStream_t s = nullptr;
    bool own_stream = false;
    bool time_mode = false;

    DevBuf<DevState> st;
    DevBuf<DevRecord> rec;
    long long rec_cap = 0;
    DevBuf<float4> U;
    DevBuf<int> B[2], R[2], Rdeg[2];
    DevBuf<uint2> Rp[2];
    bool rpack = false;  // select reads the int16-packed reverse neighbourhood
    int maxdeg[2] = {0, 0};
    PopBuf pop[2], off[2], undo[2];
    DevBuf<float4> eff[2];
    DevBuf<unsigned char> srcbits;
    DevBuf<int> ustamp[2];
    DevBuf<int> bad[2];
    int* host_flag = nullptr;
    DevBuf<unsigned> done_ctr;
    DevBuf<double> staging;  // f64 row-major staging for population transfers
    DevBuf<int> rowsbuf;
    DevBuf<int> nbad_buf;
    int* host_flag_dev = nullptr;

    VaryParams vp{};
    Op1Params op1p{};
    SelParams sp{};
    RestoreParams rp{};
    VaryKernel vary = nullptr;
    cudaGraphExec_t graph = nullptr;
    cudaGraphExec_t graph_first = nullptr;

    long long gens_enqueued = 0;  // generations launched (host view)
    long long gen_limit = 0;      // max generations allowed by k_max / eval budget (-1 = inf)
    bool finished = false;

    ~gmpea_engine() {
        if (graph) cudaGraphExecDestroy(graph);
        if (graph_first) cudaGraphExecDestroy(graph_first);
        if (host_flag) cudaFreeHost(host_flag);
        if (own_stream && s) cudaStreamDestroy(s);
    }

    void setup(const gmpea_problem* p, const gmpea_run_config& c) {
        prob = p;
        cfg = c;
        if (c.n <= 0) throw std::invalid_argument("reference_vectors: target_n must be positive");
        if (c.n > (1ll << 30)) throw std::invalid_argument("engine: n too large");
        if (p->m > kMaxM || p->m < 2) throw std::invalid_argument("engine: objectives must be 2 or 3");
        CK(cudaSetDevice(c.device));
        if (c.stream) {
            s = (cudaStream_t)(uintptr_t)c.stream;
        } else {
            CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            own_stream = true;
        }
        N = c.n;
        d = p->d;
        m = p->m;
        nc = p->nin + p->neq;
        geo = row_geom(d, nc, p->fam == FAM_WTA ? p->dev.wta_n8 : 0);
        t1 = (int)std::min<long long>(c.t1, N);
        t2 = (int)std::min<long long>(c.t2, N);
        time_mode = c.time_budget_s > 0.0;
        H = lattice_H(m, N);
        own0 = 0;
        own1 = N;
        if (c.shard_end > c.shard_begin) {
            if (c.shard_begin < 0 || c.shard_end > N)
                throw std::invalid_argument("engine: shard range outside [0, n)");
            own0 = c.shard_begin;
            own1 = c.shard_end;
            sharded = own0 > 0 || own1 < N;
        }
        if (sharded && time_mode)
            throw std::invalid_argument("engine: a sharded run takes k_max / eval budgets (the deadline would differ per rank)");

        st.alloc(1);
        st.zero(s);
        init_state_kernel<<<1, 1, 0, s>>>(st.p, m);
        // generation limit (gmpea.cpp:456-459)
        bool unbounded = c.k_max == 0 && (time_mode || c.eval_budget > 0);
        long long lim = c.k_max > 0 ? c.k_max : (unbounded ? -1 : 0);
        if (c.eval_budget > 0) {
            long long e = c.eval_budget / (2ll * N) - 1;  // gens with evals + 2n <= budget
            if (e < 0) e = 0;
            lim = lim < 0 ? e : std::min(lim, e);
        }
        gen_limit = lim;
        rec_cap = (lim >= 0 ? lim : (1ll << 22)) + 2;
        rec.alloc(rec_cap);
        rec.zero(s);

        // reference vectors + neighbourhoods (gmpea.cpp:424-428), global
        {
            DevBuf<double> Wg((size_t)N * m);
            DevBuf<float4> Ug(round_up(N, 32));
            lattice_kernel<<<blocks_for(N, 256), 256, 0, s>>>((int)N, m, H, Wg.p, Ug.p);
            CK(cudaGetLastError());
            DevBuf<int> Bg[2];
            Bg[0].alloc((size_t)N * t1);
            Bg[1].alloc((size_t)N * t2);
            device_knn(s, (int)N, m, t1, t2, Wg.p, true, H, Bg[0].p, Bg[1].p);
            // shard window: own [own0, own1); offspring regenerated on
            // [own0 - r, own1 + r); parent rows kept on [own0 - 2r, own1 + 2r)
            if (sharded) {
                DevBuf<int> r(1);
                r.zero(s);
                for (int q = 0; q < 2; ++q)
                    reach_kernel<<<blocks_for(N * (q ? t2 : t1), 256), 256, 0, s>>>(Bg[q].p, N, q ? t2 : t1, r.p);
                int hr = 0;
                CK(cudaMemcpyAsync(&hr, r.p, sizeof(int), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                reach = hr;
                if (own1 - own0 < 2 * reach)
                    throw std::invalid_argument("engine: shard narrower than twice the neighbourhood reach (" +
                                                std::to_string(2 * reach) + " slots)");
            }
            e0 = std::max(0ll, own0 - 2 * reach);
            e1 = std::min(N, own1 + 2 * reach);
            v0 = std::max(0ll, own0 - reach);
            v1 = std::min(N, own1 + reach);
            n = (int)(e1 - e0);
            ld = round_up(n, 32);
            U.alloc(ld);
            U.zero(s);
            CK(cudaMemcpyAsync(U.p, Ug.p + e0, (size_t)n * sizeof(float4), cudaMemcpyDeviceToDevice, s));
            for (int q = 0; q < 2; ++q) {
                const int t = q ? t2 : t1;
                B[q].alloc((size_t)n * t);
                slice_topology_kernel<<<blocks_for((long long)n * t, 256), 256, 0, s>>>(Bg[q].p, t, e0, n, v0, v1,
                                                                                         B[q].p);
            }
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(s));
        }
        maxdeg[0] = device_reverse(s, n, t1, B[0].p, ld, Rdeg[0], R[0], (int)(v0 - e0), (int)(v1 - e0));
        maxdeg[1] = device_reverse(s, n, t2, B[1].p, ld, Rdeg[1], R[1], (int)(v0 - e0), (int)(v1 - e0));
        rpack = device_pack_reverse(s, n, maxdeg[0], R[0], ld, Rdeg[0], Rp[0]) &&
                device_pack_reverse(s, n, maxdeg[1], R[1], ld, Rdeg[1], Rp[1]);

        for (int q = 0; q < 2; ++q) {
            pop[q].alloc(n, geo.rs4, ld);
            off[q].alloc(n, geo.rs4, ld);
            eff[q].alloc(ld);
            bad[q].alloc(kMaxBadRows);
            pop[q].Fcv.zero(s);
            off[q].Fcv.zero(s);
            if (time_mode) {
                undo[q].alloc(n, geo.rs4, ld);
                ustamp[q].alloc(ld);
                CK(cudaMemsetAsync(ustamp[q].p, 0xff, ld * sizeof(int), s));
            }
        }
        srcbits.alloc(ld);
        CK(cudaHostAlloc(&host_flag, sizeof(int), cudaHostAllocMapped));
        *host_flag = 0;
        CK(cudaHostGetDevicePointer((void**)&host_flag_dev, host_flag, 0));

        // kernel parameter blocks
        vp = VaryParams{};
        vp.n = n;
        vp.row0 = 0;
        vp.row_end = n;
        vp.rs4 = geo.rs4;
        vp.srs4 = geo.srs4;
        vp.scratch8 = geo.stream8;
        vp.slot_base = (int)e0;  // Philox keys use global slots
        vp.pop_id[0] = 1;
        vp.pop_id[1] = 2;
        vp.P = p->dev;
        vp.t[0] = t1;
        vp.t[1] = t2;
        vp.ui[0] = make_uidx((unsigned long long)t1);
        vp.ui[1] = make_uidx((unsigned long long)t2);
        vp.key = make_philox_key(c.seed);
        fill_op_params(vp, c.params, d);
        vp.eval = 1;
        vp.update_z = 1;
        vp.fixed_gen = -1;
        vp.st = st.p;
        vp.bad_cap = kMaxBadRows;
        for (int q = 0; q < 2; ++q) {
            vp.B[q] = B[q].p;
            vp.bad_rows[q] = bad[q].p;
        }

        // initial populations (gmpea.cpp:430-437): Philox INIT stream
        for (int q = 0; q < 2; ++q) {
            vp.parX[q] = pop[q].X.p;
            vp.out[q] = pop[q].X.p;
            vp.outFcv[q] = pop[q].Fcv.p;
        }
        VaryParams ip = vp;
        ip.fixed_gen = 0;
        launch_vary(vary_kernel_for(p->fam, MODE_INIT, 0), ip, 2, s);
        CK(cudaGetLastError());
        finish_init();

        // generation parameter blocks
        for (int q = 0; q < 2; ++q) {
            vp.parX[q] = pop[q].X.p;
            vp.out[q] = off[q].X.p;
            vp.outFcv[q] = off[q].Fcv.p;
        }
        vary = vary_kernel_for(p->fam, MODE_VARY, c.op, p->dev.uniform ? d : 0, p->dev.id);
        vp.row0 = (int)(v0 - e0);
        vp.row_end = (int)(v1 - e0);
        op1p = Op1Params{(int)(v0 - e0), (int)(v1 - e0), m, (float)c.theta, U.p, {off[0].Fcv.p, off[1].Fcv.p},
                         {eff[0].p, eff[1].p}, srcbits.p, st.p};
        sp = SelParams{};
        sp.n = n;
        sp.row0 = (int)(own0 - e0);
        sp.row_end = (int)(own1 - e0);
        sp.rs4 = geo.rs4;
        sp.ldr = ld;
        sp.m = m;
        sp.theta = (float)c.theta;
        sp.U = U.p;
        for (int q = 0; q < 2; ++q) {
            sp.X[q] = pop[q].X.p;
            sp.Fcv[q] = pop[q].Fcv.p;
            sp.oX[q] = off[q].X.p;
            sp.oFcv[q] = off[q].Fcv.p;
            sp.eff[q] = eff[q].p;
            sp.R[q] = R[q].p;
            sp.Rp[q] = rpack ? Rp[q].p : nullptr;
            sp.Rdeg[q] = Rdeg[q].p;
            sp.winner[q] = nullptr;
            if (time_mode) {
                sp.uX[q] = undo[q].X.p;
                sp.uFcv[q] = undo[q].Fcv.p;
                sp.ustamp[q] = ustamp[q].p;
                rp.X[q] = pop[q].X.p;
                rp.Fcv[q] = pop[q].Fcv.p;
                rp.uX[q] = undo[q].X.p;
                rp.uFcv[q] = undo[q].Fcv.p;
                rp.ustamp[q] = ustamp[q].p;
            }
        }
        sp.srcbits = srcbits.p;
        sp.apply = 1;
        sp.st = st.p;
        sp.rec = rec.p;
        done_ctr.alloc(1);
        done_ctr.zero(s);
        sp.done = done_ctr.p;
        sp.host_flag = host_flag_dev;
        rp.row0 = (int)(own0 - e0);
        rp.row_end = (int)(own1 - e0);
        rp.rs4 = geo.rs4;
        rp.st = st.p;
        // transfer buffers and the generation graph are made here, so that
        // set_population / step / get_population allocate nothing and the
        // first step does not instantiate the graph (the graph's parameters
        // never change after construction)
        staging.alloc((size_t)n * (std::max({d, nc, m}) + 1));
        rowsbuf.alloc(std::max(n, 1));
        nbad_buf.alloc(1);
        if (!sharded) build_graph();
        CK(cudaStreamSynchronize(s));
        check_errors(0);
    }

    // evaluation of the initial populations done: z, record 0, gen = 1
    void finish_init() {
        init_state_kernel<<<1, 1, 0, s>>>(st.p, m);
        const int o0 = (int)(own0 - e0), on = (int)(own1 - own0);
        for (int q = 0; q < 2; ++q)
            z_of_kernel<<<blocks_for(on, 256), 256, 0, s>>>(pop[q].Fcv.p + o0, on, m, st.p);
        rec.zero(s);
        count_feasible_kernel<<<blocks_for(on, 256), 256, 0, s>>>(pop[0].Fcv.p, o0, o0 + on, &rec.p[0].feasible);
        DevState init{};
        CK(cudaMemcpyAsync(&init, st.p, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        DevState fresh{};
        for (int k = 0; k < 4; ++k) fresh.zbits[k] = init.zbits[k];
        fresh.gen = 1;
        fresh.err = init.err;
        fresh.err_gen = init.err_gen;
        fresh.n_bad[0] = init.n_bad[0];
        fresh.n_bad[1] = init.n_bad[1];
        fresh.budget_ns = time_mode ? (unsigned long long)std::llround(cfg.time_budget_s * 1e9) : 0ull;
        CK(cudaMemcpyAsync(st.p, &fresh, offsetof(DevState, bad_rows), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(&st.p->t_gen_start, &fresh.t_gen_start,
                           sizeof(DevState) - offsetof(DevState, t_gen_start), cudaMemcpyHostToDevice, s));
        gens_enqueued = 0;
        finished = false;
    }

    void set_population(int which, const double* X) {
        if (which != 1 && which != 2) throw std::invalid_argument("set_population: which must be 1 or 2");
        if (gens_enqueued) throw std::invalid_argument("set_population: the run has started");
        const int q = which - 1;
        if (staging.n < (size_t)n * (std::max({d, nc, m}) + 1)) staging.alloc((size_t)n * (std::max({d, nc, m}) + 1));
        DevBuf<double>& h = staging;
        // X holds all N rows; this engine keeps its window [e0, e1)
        CK(cudaMemcpyAsync(h.p, X + e0 * d, (size_t)n * d * sizeof(double), cudaMemcpyHostToDevice, s));
        DevBuf<int>& nbad = nbad_buf;
        nbad.zero(s);
        if (rowsbuf.n < (size_t)std::max(n, 1)) rowsbuf.alloc(std::max(n, 1));
        DevBuf<int>& rows = rowsbuf;
        to_rows_kernel<<<blocks_for((long long)n * d, 256), 256, 0, s>>>(
            h.p, n, d, (float*)pop[q].X.p, geo.rs4 * 4, prob->dlo64.p, prob->dhi64.p, rows.p, nbad.p);
        int hb = 0;
        CK(cudaMemcpyAsync(&hb, nbad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (hb) {
            std::vector<int> r(hb);
            CK(cudaMemcpy(r.data(), rows.p, hb * sizeof(int), cudaMemcpyDeviceToHost));
            for (int& v : r) v += (int)e0;
            throw std::invalid_argument(rows_message(r));
        }
        VaryParams ep = vp;
        ep.row0 = 0;
        ep.row_end = n;
        ep.parX[0] = pop[q].X.p;
        ep.out[0] = pop[q].X.p;
        ep.outFcv[0] = pop[q].Fcv.p;
        ep.update_z = 0;
        ep.fixed_gen = 0;
        launch_vary(vary_kernel_for(prob->fam, MODE_EVAL, 0), ep, 1, s);
        CK(cudaGetLastError());
        finish_init();
        CK(cudaStreamSynchronize(s));
    }

    void enqueue_generation() {
        enqueue_phase1();
        enqueue_phase2();  // select's last block also publishes the stop flag
    }

    void launch_select() {
        const dim3 grid(blocks_for(own1 - own0, 256), 2);
        if (rpack)
            select_kernel<true><<<grid, 256, 0, s>>>(sp);
        else
            select_kernel<false><<<grid, 256, 0, s>>>(sp);
    }

    // phase 1: variation + evaluation (+ local ideal-point partial)
    void enqueue_phase1() { launch_vary(vary, vp, 2, s); }
    // phase 2: OP1, selection, bookkeeping (a sharded run all-reduces z in between)
    void enqueue_phase2() {
        op1_kernel<<<blocks_for(v1 - v0, 256), 256, 0, s>>>(op1p);
        launch_select();  // + end_gen
        if (time_mode) restore_kernel<<<dim3(blocks_for(own1 - own0, 256), 2), 256, 0, s>>>(rp);
    }

    // two graphs of one generation: graph_first also restarts the loop clock
    // (the first generation of a step() call), so step(1) is one launch
    cudaGraphExec_t capture_generation(bool clock) {
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t g;
        cudaGraphExec_t x;
        CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        cudaStream_t saved = s;
        s = cs;
        if (clock) start_loop_clock();
        enqueue_generation();
        s = saved;
        CK(cudaStreamEndCapture(cs, &g));
        CK(cudaGraphInstantiate(&x, g, 0));
        CK(cudaGraphDestroy(g));
        CK(cudaStreamDestroy(cs));
        return x;
    }

    void build_graph() {
        if (graph) return;
        graph = capture_generation(false);
        graph_first = capture_generation(true);
    }

    // the loop clock restarts at every step() so host work between calls
    // (metric hooks) stays outside the loop time, as in gmpea.cpp:442-453
    void start_loop_clock() { mark_start_kernel<<<1, 1, 0, s>>>(st.p); }

    // enqueue up to k generations, respecting the generation limit
    long long step(long long k) {
        if (gen_limit >= 0) k = std::min(k, gen_limit - gens_enqueued);
        if (k <= 0) return 0;
        build_graph();
        CK(cudaGraphLaunch(graph_first, s));
        for (long long i = 1; i < k; ++i) CK(cudaGraphLaunch(graph, s));
        gens_enqueued += k;
        return k;
    }

    // one generation in two phases (sharded runs; no graph, plain launches)
    void phase(int ph) {
        if (ph == 1) {
            if (gen_limit >= 0 && gens_enqueued >= gen_limit)
                throw std::invalid_argument("phase: generation limit reached");
            start_loop_clock();
            enqueue_phase1();
        } else if (ph == 2) {
            enqueue_phase2();
            gens_enqueued += 1;
        } else {
            throw std::invalid_argument("phase: must be 1 or 2");
        }
        CK(cudaGetLastError());
    }

    void run() {
        if (!time_mode) {
            if (gen_limit < 0) throw std::invalid_argument("run: unbounded run without a budget");
            step(gen_limit - gens_enqueued);
            CK(cudaStreamSynchronize(s));
        } else {
            // time budget: keep at most two chunks in flight and stop launching
            // once the device reports the deadline (gmpea.cpp:458, :481-486)
            const long long chunk = n >= 100000 ? 2 : 16;
            cudaEvent_t ev[2];
            CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
            int k = 0;
            bool pending[2] = {false, false};
            for (;;) {
                if (pending[k]) {
                    CK(cudaEventSynchronize(ev[k]));
                    pending[k] = false;
                    if (*(volatile int*)host_flag) break;
                }
                long long launched = step(chunk);
                if (launched == 0) break;
                CK(cudaEventRecord(ev[k], s));
                pending[k] = true;
                k ^= 1;
            }
            CK(cudaStreamSynchronize(s));
            cudaEventDestroy(ev[0]);
            cudaEventDestroy(ev[1]);
        }
        finished = true;
        check_errors(-1);
    }

    DevState read_state() {
        DevState h{};
        CK(cudaMemcpyAsync(&h, st.p, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return h;
    }

    void check_errors(int phase) {
        DevState h = read_state();
        if (!h.err) return;
        std::string where = phase == 0 ? std::string("") :
            "run_gmpea: evaluation failed at generation " + std::to_string(h.err_gen) + ": ";
        if (h.err == ERR_EVAL_OOB) {
            int q = h.n_bad[0] > 0 ? 0 : 1;
            int cnt = std::min(h.n_bad[q], kMaxBadRows);
            std::vector<int> r(h.bad_rows[q], h.bad_rows[q] + cnt);
            if (phase == 0) throw std::invalid_argument(rows_message(r));
            throw std::runtime_error(where + rows_message(r));
        }
        if (h.err == ERR_NONFINITE) throw std::invalid_argument("non-finite mask source");
        if (h.err == ERR_NEG_CV) throw std::invalid_argument("fpr_better: negative constraint violation");
        throw std::runtime_error("engine error " + std::to_string(h.err));
    }

    std::vector<gmpea_gen_record> history() {
        DevState h = read_state();
        long long g = std::min<long long>(h.gens_done, rec_cap - 1);
        std::vector<DevRecord> r(g + 1);
        CK(cudaMemcpyAsync(r.data(), rec.p, (g + 1) * sizeof(DevRecord), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<gmpea_gen_record> out(g + 1);
        for (long long k = 0; k <= g; ++k) {
            gmpea_gen_record& o = out[k];
            o = gmpea_gen_record{};
            o.gen = k;
            o.evals = 2ll * N * (k + 1);
            o.wall_ms = cfg.record_walltime ? (k == 0 ? 0.0 : (double)r[k].loop_ns * 1e-6) : 0.0;
            o.feasible_ratio = (double)r[k].feasible / (double)(own1 - own0);
            o.igd = std::numeric_limits<double>::quiet_NaN();
            o.hv = std::numeric_limits<double>::quiet_NaN();
        }
        return out;
    }


    std::vector<int64_t> replacements() {
        DevState h = read_state();
        long long g = std::min<long long>(h.gens_done, rec_cap - 1);
        std::vector<DevRecord> r(g + 1);
        CK(cudaMemcpyAsync(r.data(), rec.p, (g + 1) * sizeof(DevRecord), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<int64_t> out(g + 1);
        for (long long k = 0; k <= g; ++k) out[k] = k == 0 ? 0 : (int64_t)r[k].replaced;
        return out;
    }

    void record_async(void* dst) {
        static_assert(sizeof(DevRecord) == sizeof(gmpea_raw_record), "raw record layout");
        const long long k = std::min<long long>(gens_enqueued, rec_cap - 1);
        CK(cudaMemcpyAsync(dst, rec.p + k, sizeof(DevRecord), cudaMemcpyDeviceToHost, s));
    }

    // the newest generation record only (one small D2H; the per-step result)
    gmpea_gen_record last_record() {
        struct {
            int gens_done;
        } g{};
        CK(cudaMemcpyAsync(&g.gens_done, &st.p->gens_done, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        DevRecord r{};
        long long k = std::min<long long>(g.gens_done, rec_cap - 1);
        CK(cudaMemcpyAsync(&r, rec.p + k, sizeof(DevRecord), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        gmpea_gen_record o{};
        o.gen = k;
        o.evals = 2ll * N * (k + 1);
        o.wall_ms = cfg.record_walltime && k ? (double)r.loop_ns * 1e-6 : 0.0;
        o.feasible_ratio = (double)r.feasible / (double)(own1 - own0);
        o.igd = o.hv = std::numeric_limits<double>::quiet_NaN();
        return o;
    }

    // the owned rows [own0, own1) (all N unsharded)
    void get_population(int which, double* X, double* F, double* C, double* cv) {
        if (which != 1 && which != 2) throw std::invalid_argument("get_population: which must be 1 or 2");
        const int q = which - 1;
        const long long o0 = own0 - e0, on = own1 - own0;
        if (staging.n < (size_t)n * (std::max({d, nc, m}) + 1)) staging.alloc((size_t)n * (std::max({d, nc, m}) + 1));
        DevBuf<double>& tmp = staging;
        const float* rows = (const float*)(pop[q].X.p + o0 * geo.rs4);
        auto pull = [&](int col0, int k, double* out) {
            if (!out || k == 0) return;
            from_rows_kernel<<<blocks_for(on * k, 256), 256, 0, s>>>(rows, geo.rs4 * 4, on, col0, k, tmp.p);
            CK(cudaMemcpyAsync(out, tmp.p, (size_t)on * k * sizeof(double), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        };
        pull(0, d, X);
        pull(d, nc, C);
        if (F || cv) {
            double* f = tmp.p;
            double* c = tmp.p + (size_t)on * m;
            fcv_to_rows_kernel<<<blocks_for(on, 256), 256, 0, s>>>(pop[q].Fcv.p + o0, on, m, f, c);
            if (F) CK(cudaMemcpyAsync(F, f, (size_t)on * m * sizeof(double), cudaMemcpyDeviceToHost, s));
            if (cv) CK(cudaMemcpyAsync(cv, c, (size_t)on * sizeof(double), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
    }

    void profile(long long gens, double* ms) {
        if (gen_limit >= 0) gens = std::min(gens, gen_limit - gens_enqueued);
        if (gens <= 0) throw std::invalid_argument("profile: no generations left");
        start_loop_clock();
        std::vector<cudaEvent_t> ev(5 * gens);
        for (auto& e : ev) CK(cudaEventCreate(&e));
        for (long long g = 0; g < gens; ++g) {
            cudaEvent_t* e = &ev[5 * g];
            CK(cudaEventRecord(e[0], s));
            launch_vary(vary, vp, 2, s);
            CK(cudaEventRecord(e[1], s));
            op1_kernel<<<blocks_for(v1 - v0, 256), 256, 0, s>>>(op1p);
            CK(cudaEventRecord(e[2], s));
            launch_select();  // + end_gen
            CK(cudaEventRecord(e[3], s));
            if (time_mode) restore_kernel<<<dim3(blocks_for(own1 - own0, 256), 2), 256, 0, s>>>(rp);
            CK(cudaEventRecord(e[4], s));
        }
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
        gens_enqueued += gens;
        double acc[5] = {0, 0, 0, 0, 0};
        for (long long g = 0; g < gens; ++g) {
            cudaEvent_t* e = &ev[5 * g];
            for (int k = 0; k < 4; ++k) {
                float t = 0.0f;
                CK(cudaEventElapsedTime(&t, e[k], e[k + 1]));
                acc[k] += t;
            }
            float t = 0.0f;
            CK(cudaEventElapsedTime(&t, e[0], e[4]));
            acc[4] += t;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        for (int k = 0; k < 5; ++k) ms[k] = acc[k] / (double)gens;
        check_errors(-1);
    }
};

// ====================================================================== C ABI
extern "C" {

const char* gmpea_last_error(void) { return g_err.c_str(); }
int gmpea_abi_version(void) { return 1; }

int gmpea_problem_create(const char* name, gmpea_problem** out) {
    return guarded([&] {
        if (!name || !out) throw std::invalid_argument("gmpea_problem_create: null argument");
        auto p = make_problem(name);
        p->upload();
        *out = p.release();
    });
}

int gmpea_problem_create_wta(const char* scenario, int32_t targets, int32_t vehicles,
                             const int32_t* strikes, const int32_t* capacity, const double* pv,
                             gmpea_problem** out) {
    return guarded([&] {
        WtaHost w;
        w.scenario = scenario ? scenario : "custom";
        w.targets = targets;
        w.vehicles = vehicles;
        w.strikes.assign(strikes, strikes + targets);
        w.cap.assign(capacity, capacity + vehicles);
        int slots = 0;
        for (int s : w.strikes) {
            if (s < 0) throw std::invalid_argument("WTA: negative strike count");
            slots += s;
        }
        w.p.assign(pv, pv + slots);
        for (double v : w.p)
            if (!(v >= 0.0 && v <= 1.0)) throw std::invalid_argument("WTA: probability out of range");
        auto p = std::make_unique<gmpea_problem>();
        make_wta(*p, w);
        p->upload();
        *out = p.release();
    });
}

int gmpea_wta_scenario(int32_t num, int32_t* targets, int32_t* vehicles, int32_t* strikes, int32_t* capacity,
                       double* p) {
    return guarded([&] {
        if (num < 1 || num > 10) throw std::invalid_argument("unknown WTA scenario: P" + std::to_string(num));
        WtaHost w = wta_scenario(num);
        *targets = w.targets;
        *vehicles = w.vehicles;
        if (strikes) std::copy(w.strikes.begin(), w.strikes.end(), strikes);
        if (capacity) std::copy(w.cap.begin(), w.cap.end(), capacity);
        if (p) std::copy(w.p.begin(), w.p.end(), p);
    });
}

int gmpea_problem_info(const gmpea_problem* p, int32_t* d, int32_t* m, int32_t* nin, int32_t* neq) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("null problem");
        if (d) *d = p->d;
        if (m) *m = p->m;
        if (nin) *nin = p->nin;
        if (neq) *neq = p->neq;
    });
}

int gmpea_problem_bounds(const gmpea_problem* p, double* lo, double* hi) {
    return guarded([&] {
        if (lo) std::copy(p->lo.begin(), p->lo.end(), lo);
        if (hi) std::copy(p->hi.begin(), p->hi.end(), hi);
    });
}

void gmpea_problem_destroy(gmpea_problem* p) { delete p; }

const char* gmpea_problem_names(void) {
    static std::string names = [] {
        std::string s;
        for (int i = 1; i <= 14; ++i) s += "LIRCMOP" + std::to_string(i) + "\n";
        for (const char* n : {"C1-DTLZ1", "C1-DTLZ3", "C2-DTLZ2", "C3-DTLZ4", "DC1-DTLZ1", "DC1-DTLZ3",
                              "DC2-DTLZ1", "DC2-DTLZ3", "DC3-DTLZ1", "DC3-DTLZ3"})
            s += std::string(n) + "\n";
        for (int i = 1; i <= 10; ++i) s += "WTA-P" + std::to_string(i) + "\n";
        for (int i = 1; i <= 14; ++i) s += "MW" + std::to_string(i) + "\n";
        for (int i = 1; i <= 9; ++i) s += "DASCMOP" + std::to_string(i) + "\n";
        return s;
    }();
    return names.c_str();
}

int gmpea_evaluate(const gmpea_problem* p, const double* X, int64_t n, double* F, double* G, double* cv) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("null problem");
        if (n < 0) throw std::invalid_argument("evaluate: negative row count");
        if (n == 0) return;
        if (n > (1ll << 30)) throw std::invalid_argument("evaluate: too many rows");
        CK(cudaSetDevice(p->device));
        const int d = p->d, m = p->m, nc = p->nin + p->neq;
        const long long ld = round_up(n, 32);
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct SG {
            cudaStream_t s;
            ~SG() { cudaStreamDestroy(s); }
        } sg{s};
        DevBuf<double> h((size_t)n * d);
        CK(cudaMemcpyAsync(h.p, X, (size_t)n * d * sizeof(double), cudaMemcpyHostToDevice, s));
        const RowGeom geo = row_geom(d, nc, p->fam == FAM_WTA ? p->dev.wta_n8 : 0);
        PopBuf pb;
        pb.alloc(n, geo.rs4, ld);
        DevBuf<int> rows(n), nbad(1);
        nbad.zero(s);
        to_rows_kernel<<<blocks_for(n * d, 256), 256, 0, s>>>(h.p, n, d, (float*)pb.X.p, geo.rs4 * 4, p->dlo64.p,
                                                             p->dhi64.p, rows.p, nbad.p);
        int hb = 0;
        CK(cudaMemcpyAsync(&hb, nbad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (hb) {
            std::vector<int> r(hb);
            CK(cudaMemcpy(r.data(), rows.p, hb * sizeof(int), cudaMemcpyDeviceToHost));
            throw std::invalid_argument(rows_message(r));
        }
        DevBuf<DevState> st(1);
        st.zero(s);
        DevBuf<int> bad(n);
        VaryParams ep{};
        ep.n = (int)n;
        ep.row0 = 0;
        ep.row_end = (int)n;
        ep.rs4 = geo.rs4;
        ep.srs4 = geo.srs4;
        ep.scratch8 = geo.stream8;
        ep.pop_id[0] = 1;
        ep.P = p->dev;
        ep.parX[0] = pb.X.p;
        ep.out[0] = pb.X.p;
        ep.outFcv[0] = pb.Fcv.p;
        ep.eval = 1;
        ep.fixed_gen = 0;
        ep.st = st.p;
        ep.bad_rows[0] = bad.p;
        ep.bad_cap = (int)n;
        launch_vary(vary_kernel_for(p->fam, MODE_EVAL, 0), ep, 1, s);
        CK(cudaGetLastError());
        DevBuf<double> out((size_t)n * std::max({m, nc, 1}));
        DevBuf<double> c(n);
        fcv_to_rows_kernel<<<blocks_for(n, 256), 256, 0, s>>>(pb.Fcv.p, n, m, out.p, c.p);
        CK(cudaMemcpyAsync(F, out.p, (size_t)n * m * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (cv) CK(cudaMemcpyAsync(cv, c.p, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (G && nc) {
            from_rows_kernel<<<blocks_for(n * nc, 256), 256, 0, s>>>((const float*)pb.X.p, geo.rs4 * 4, n, d, nc,
                                                                    out.p);
            CK(cudaMemcpyAsync(G, out.p, (size_t)n * nc * sizeof(double), cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        CK(cudaGetLastError());
    });
}

int gmpea_reference_vectors(int32_t m, int64_t n, double* W) {
    return guarded([&] {
        if (n <= 0) throw std::invalid_argument("reference_vectors: target_n must be positive");
        if (m < 2 || m > 3) throw std::invalid_argument("reference_vectors: m must be 2 or 3");
        require_device();
        DevBuf<double> w((size_t)n * m);
        DevBuf<float4> u(n);
        lattice_kernel<<<blocks_for(n, 256), 256>>>((int)n, m, lattice_H(m, n), w.p, u.p);
        CK(cudaGetLastError());
        CK(cudaMemcpy(W, w.p, (size_t)n * m * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

static void knn_api(const double* Wh, int64_t n, int32_t m, int32_t t1, int32_t t2, uint32_t* B1,
                    uint32_t* B2, bool lattice) {
    if (n <= 0) throw std::invalid_argument("build_neighborhoods: empty population");
    if (m < 2 || m > 3) throw std::invalid_argument("build_neighborhoods: m must be 2 or 3");
    if (t1 > n || t2 > n) throw std::invalid_argument("build_neighborhoods: neighborhood exceeds population");
    require_device();
    cudaStream_t s = 0;
    DevBuf<double> w((size_t)n * m);
    DevBuf<float4> u(n);
    long long H = lattice_H(m, n);
    if (lattice)
        lattice_kernel<<<blocks_for(n, 256), 256>>>((int)n, m, H, w.p, u.p);
    else
        CK(cudaMemcpy(w.p, Wh, (size_t)n * m * sizeof(double), cudaMemcpyHostToDevice));
    DevBuf<int> b1((size_t)n * std::max(t1, 1)), b2((size_t)n * std::max(t2, 1));
    device_knn(s, (int)n, m, t1, t2, w.p, lattice, H, b1.p, b2.p);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(B1, b1.p, (size_t)n * t1 * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(B2, b2.p, (size_t)n * t2 * sizeof(int), cudaMemcpyDeviceToHost));
}

int gmpea_build_neighborhoods(const double* W, int64_t n, int32_t m, int32_t t1, int32_t t2, uint32_t* B1,
                              uint32_t* B2) {
    return guarded([&] { knn_api(W, n, m, t1, t2, B1, B2, false); });
}

int gmpea_lattice_neighborhoods(int32_t m, int64_t n, int32_t t1, int32_t t2, uint32_t* B1, uint32_t* B2) {
    return guarded([&] { knn_api(nullptr, n, m, t1, t2, B1, B2, true); });
}

int gmpea_operator_params_default(gmpea_operator_params* o) {
    // OperatorParams defaults (gmpea.hpp:58-66)
    *o = gmpea_operator_params{1.0, 20.0, 20.0, 1.0, 0.5, -1.0};
    return GMPEA_OK;
}

int gmpea_reproduce(const gmpea_problem* p, const double* X, int64_t n, const uint32_t* nbrs, int32_t t,
                    int32_t op, const gmpea_operator_params* params, uint64_t seed, uint32_t gen,
                    uint32_t pop, double* off) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("null problem");
        if (n <= 0) return;
        if (t <= 0) throw std::invalid_argument("reproduce: topology/population mismatch");
        if (op != GMPEA_OP_SBX_PM && op != GMPEA_OP_DE) throw std::invalid_argument("reproduce: unknown operator");
        CK(cudaSetDevice(p->device));
        const int d = p->d, nc = p->nin + p->neq;
        const RowGeom geo = row_geom(d, nc, p->fam == FAM_WTA ? p->dev.wta_n8 : 0);
        cudaStream_t s = 0;
        DevBuf<double> h((size_t)n * d);
        CK(cudaMemcpy(h.p, X, (size_t)n * d * sizeof(double), cudaMemcpyHostToDevice));
        DevBuf<float4> Xp((size_t)n * geo.rs4), Op((size_t)n * geo.rs4);
        to_rows_kernel<<<blocks_for(n * d, 256), 256>>>(h.p, n, d, (float*)Xp.p, geo.rs4 * 4, nullptr, nullptr,
                                                        nullptr, nullptr);
        DevBuf<unsigned> bu((size_t)n * t);
        DevBuf<int> bi((size_t)n * t), err(1);
        err.zero(s);
        CK(cudaMemcpy(bu.p, nbrs, (size_t)n * t * sizeof(unsigned), cudaMemcpyHostToDevice));
        u32_to_i32_kernel<<<blocks_for(n * t, 256), 256>>>(bu.p, n * t, bi.p, (int)n, err.p);
        int herr = 0;
        CK(cudaMemcpy(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (herr) throw std::invalid_argument("reproduce: neighbour index out of range");
        DevBuf<DevState> st(1);
        st.zero(s);
        DevBuf<int> bad(1);
        VaryParams vp{};
        vp.n = (int)n;
        vp.row0 = 0;
        vp.row_end = (int)n;
        vp.rs4 = geo.rs4;
        vp.srs4 = geo.srs4;
        vp.scratch8 = geo.stream8;
        vp.pop_id[0] = (int)pop;
        vp.P = p->dev;
        vp.parX[0] = Xp.p;
        vp.B[0] = bi.p;
        vp.t[0] = t;
        vp.ui[0] = make_uidx((unsigned long long)t);
        vp.out[0] = Op.p;
        vp.key = make_philox_key(seed);
        gmpea_operator_params prm;
        gmpea_operator_params_default(&prm);
        if (params) prm = *params;
        fill_op_params(vp, prm, d);
        vp.eval = 0;
        vp.fixed_gen = (int)gen;
        vp.st = st.p;
        vp.bad_rows[0] = bad.p;
        vp.bad_cap = 0;  // reproduce itself never throws on bounds
        launch_vary(vary_kernel_for(p->fam, MODE_VARY, op, p->dev.uniform ? d : 0, p->dev.id), vp, 1, s);
        CK(cudaGetLastError());
        from_rows_kernel<<<blocks_for(n * d, 256), 256>>>((const float*)Op.p, geo.rs4 * 4, n, 0, d, h.p);
        CK(cudaMemcpy(off, h.p, (size_t)n * d * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int gmpea_environmental_selection(int64_t n, int32_t d, int32_t m, int32_t nc,
                                  const gmpea_population_view* pop1, const gmpea_population_view* pop2,
                                  const gmpea_population_view* off1, const gmpea_population_view* off2,
                                  const double* W, const double* z, double theta, const uint32_t* B1,
                                  int32_t t1, const uint32_t* B2, int32_t t2, gmpea_population_out* out1,
                                  gmpea_population_out* out2, int32_t* winner1, int32_t* winner2) {
    return guarded([&] {
        if (n <= 0) return;
        if (m < 2 || m > 3) throw std::invalid_argument("environmental_selection: m must be 2 or 3");
        if (t1 <= 0 || t2 <= 0) throw std::invalid_argument("environmental_selection: empty neighbourhood");
        require_device();
        const long long ld = round_up(n, 32);
        cudaStream_t s = 0;
        const gmpea_population_view* views[4] = {pop1, pop2, off1, off2};
        DevBuf<float4> fcv[4];
        DevBuf<double> hF((size_t)n * m), hc(n);
        for (int k = 0; k < 4; ++k) {
            fcv[k].alloc(ld);
            CK(cudaMemcpy(hF.p, views[k]->F, (size_t)n * m * sizeof(double), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(hc.p, views[k]->cv, (size_t)n * sizeof(double), cudaMemcpyHostToDevice));
            fcv_from_rows_kernel<<<blocks_for(n, 256), 256>>>(hF.p, hc.p, n, m, fcv[k].p);
        }
        DevBuf<double> w((size_t)n * m);
        CK(cudaMemcpy(w.p, W, (size_t)n * m * sizeof(double), cudaMemcpyHostToDevice));
        DevBuf<float4> U(ld);
        DevBuf<int> err(1);
        err.zero(s);
        unit_kernel<<<blocks_for(n, 256), 256>>>((int)n, m, w.p, U.p, err.p);
        int herr = 0;
        CK(cudaMemcpy(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (herr) throw std::invalid_argument("pbi: zero-norm reference vector");
        DevBuf<int> Bd[2], R[2], Rdeg[2];
        DevBuf<uint2> Rp[2];
        int md[2] = {0, 0};
        const uint32_t* Bh[2] = {B1, B2};
        const int ts[2] = {t1, t2};
        for (int q = 0; q < 2; ++q) {
            DevBuf<unsigned> bu((size_t)n * ts[q]);
            Bd[q].alloc((size_t)n * ts[q]);
            CK(cudaMemcpy(bu.p, Bh[q], (size_t)n * ts[q] * sizeof(unsigned), cudaMemcpyHostToDevice));
            err.zero(s);
            u32_to_i32_kernel<<<blocks_for(n * ts[q], 256), 256>>>(bu.p, n * ts[q], Bd[q].p, (int)n, err.p);
            CK(cudaMemcpy(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost));
            if (herr) throw std::invalid_argument("environmental_selection: neighbour index out of range");
            md[q] = device_reverse(s, (int)n, ts[q], Bd[q].p, ld, Rdeg[q], R[q]);
        }
        const bool pack = device_pack_reverse(s, (int)n, md[0], R[0], ld, Rdeg[0], Rp[0]) &&
                          device_pack_reverse(s, (int)n, md[1], R[1], ld, Rdeg[1], Rp[1]);
        DevBuf<DevState> st(1);
        st.zero(s);
        set_z_kernel<<<1, 1>>>(st.p, m, (float)z[0], (float)z[1], m > 2 ? (float)z[2] : 0.0f);
        DevBuf<float4> eff[2];
        eff[0].alloc(ld);
        eff[1].alloc(ld);
        DevBuf<unsigned char> sb(ld);
        Op1Params o1{0, (int)n, m, (float)theta, U.p, {fcv[2].p, fcv[3].p}, {eff[0].p, eff[1].p}, sb.p, st.p};
        op1_kernel<<<blocks_for(n, 256), 256>>>(o1);
        DevBuf<int> win[2];
        win[0].alloc(n);
        win[1].alloc(n);
        SelParams sp{};
        sp.n = (int)n;
        sp.row0 = 0;
        sp.row_end = (int)n;
        sp.ldr = ld;
        sp.m = m;
        sp.theta = (float)theta;
        sp.U = U.p;
        for (int q = 0; q < 2; ++q) {
            sp.Fcv[q] = fcv[q].p;
            sp.oFcv[q] = fcv[2 + q].p;
            sp.eff[q] = eff[q].p;
            sp.R[q] = R[q].p;
            sp.Rp[q] = pack ? Rp[q].p : nullptr;
            sp.Rdeg[q] = Rdeg[q].p;
            sp.winner[q] = win[q].p;
        }
        sp.srcbits = sb.p;
        sp.apply = 0;
        sp.st = st.p;
        if (pack)
            select_kernel<true><<<dim3(blocks_for(n, 256), 2), 256>>>(sp);
        else
            select_kernel<false><<<dim3(blocks_for(n, 256), 2), 256>>>(sp);
        CK(cudaGetLastError());
        std::vector<int> w1(n), w2(n);
        CK(cudaMemcpy(w1.data(), win[0].p, n * sizeof(int), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(w2.data(), win[1].p, n * sizeof(int), cudaMemcpyDeviceToHost));
        DevState h{};
        CK(cudaMemcpy(&h, st.p, sizeof(DevState), cudaMemcpyDeviceToHost));
        if (h.err == ERR_NONFINITE) throw std::invalid_argument("non-finite mask source");
        if (h.err == ERR_NEG_CV) throw std::invalid_argument("fpr_better: negative constraint violation");
        if (winner1) std::copy(w1.begin(), w1.end(), winner1);
        if (winner2) std::copy(w2.begin(), w2.end(), winner2);
        // copy_row (gmpea.cpp:329-331): assemble the survivors from the f64 inputs
        auto assemble = [&](const gmpea_population_view* par, const std::vector<int>& win,
                            gmpea_population_out* out) {
            if (!out) return;
            for (int64_t j = 0; j < n; ++j) {
                const gmpea_population_view* src = par;
                int64_t r = j;
                if (win[j] >= 0) {
                    src = win[j] < n ? off1 : off2;
                    r = win[j] < n ? win[j] : win[j] - n;
                }
                if (out->X) std::memcpy(out->X + j * d, src->X + r * d, d * sizeof(double));
                if (out->F) std::memcpy(out->F + j * m, src->F + r * m, m * sizeof(double));
                if (out->C && nc) std::memcpy(out->C + j * nc, src->C + r * nc, nc * sizeof(double));
                if (out->cv) out->cv[j] = src->cv[r];
            }
        };
        assemble(pop1, w1, out1);
        assemble(pop2, w2, out2);
    });
}

// ---- metrics (metrics.hpp:15-29)
namespace {

__global__ void gather_rows_kernel(const double* F, const long long* idx, long long k, int m, double* out) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= k) return;
    for (int c = 0; c < m; ++c) out[r * m + c] = F[idx[r] * m + c];
}

// nondominated + deduplicated subset of the candidate rows `cand` of F (n x m,
// device, row-major); returns the kept row ids sorted lexicographically by F
// dedup = 0 (m = 3 only): equal rows are all kept, as fronts.cpp:34-41 does
thrust::device_vector<long long> front_filter(const double* dF, int m, thrust::device_vector<long long>& cand,
                                              int dedup = 1) {
    const long long k = (long long)cand.size();
    thrust::device_vector<long long> kept;
    if (k == 0) return kept;
    thrust::sort(thrust::device, cand.begin(), cand.end(), LexLess{dF, m});
    thrust::device_vector<long long> gs(k);
    const long long* order = thrust::raw_pointer_cast(cand.data());
    group_start_kernel<<<blocks_for(k, 256), 256>>>(dF, order, k, m, thrust::raw_pointer_cast(gs.data()));
    thrust::device_vector<unsigned char> keep(k);
    if (m == 2) {
        thrust::device_vector<double> col(k);
        gather_col_kernel<<<blocks_for(k, 256), 256>>>(dF, order, k, m, 1, thrust::raw_pointer_cast(col.data()));
        thrust::inclusive_scan(thrust::device, col.begin(), col.end(), col.begin(), thrust::minimum<double>());
        nd2_kernel<<<blocks_for(k, 256), 256>>>(dF, order, thrust::raw_pointer_cast(gs.data()),
                                                thrust::raw_pointer_cast(col.data()), k,
                                                thrust::raw_pointer_cast(keep.data()));
    } else {
        nd3_kernel<<<blocks_for(k, 256), 256>>>(dF, order, thrust::raw_pointer_cast(gs.data()), k,
                                                thrust::raw_pointer_cast(keep.data()), dedup);
    }
    CK(cudaGetLastError());
    kept.resize(k);
    auto end = thrust::copy_if(thrust::device, cand.begin(), cand.end(), keep.begin(), kept.begin(),
                               NonZero{});
    kept.resize(end - kept.begin());
    return kept;
}

}  // namespace

int gmpea_pf_reference(const gmpea_problem* p, int64_t n_points, double* out, int64_t cap, int64_t* rows) {
    return guarded([&] {
        if (n_points < 0) throw std::invalid_argument("pf_reference: negative point count");
        PfParams pp{};
        if (p->fam == FAM_LIR) {
            pp.kind = PF_LIR;
        } else if (p->fam == FAM_DTLZ) {
            const int id = p->id;
            if (id == C1_DTLZ1 || id == DC1_DTLZ1 || id == DC2_DTLZ1 || id == DC3_DTLZ1) {
                pp.kind = PF_DTLZ1;  // problems.cpp:436, 520
            } else if (id == C3_DTLZ4) {
                pp.kind = PF_SPHERE;  // problems.cpp:484-486
                pp.alpha = 100.0;
                pp.rnum = 0.0;
                pp.rden = 1.0;
            } else {
                pp.kind = PF_SPHERE;  // problems.cpp:447-449, 469-471, 522-524
                pp.alpha = 1.0;
                pp.rnum = 1.0;
                pp.rden = 0.0;
            }
        } else if (p->fam == FAM_MW || p->fam == FAM_DAS) {
            pp.kind = PF_LEVEL;  // restated fronts (no reference counterpart)
        } else {
            throw std::runtime_error("pf_reference: no analytic front for " + p->name +
                                     "; use the hypervolume metric instead");
        }
        if (p->d > kPfMaxD) throw std::invalid_argument("pf_reference: dimension too large");
        require_device();
        const int m = p->m;
        pp.P = p->dev;
        // fronts.cpp:60-84
        long long over = std::max<long long>(8 * n_points, 2000);
        if (m >= 3) over = std::min<long long>(over, 12000);
        auto emit = [&](const std::vector<double>& h, long long nrows) {
            if (nrows > cap) throw std::invalid_argument("pf_reference: output capacity too small");
            if (out && nrows) std::copy(h.begin(), h.begin() + nrows * m, out);
            *rows = nrows;
        };
        for (int attempt = 0; attempt < 4; ++attempt) {
            pp.n_samples = over;
            if ((pp.kind == PF_LIR && p->id <= 12) || (pp.kind == PF_LEVEL && m == 2)) {
                pp.rows = over;
            } else if (pp.kind == PF_LEVEL) {
                long long side = 1;
                while (side * side < over) ++side;
                pp.h = side;
                pp.rows = side * side;
            } else {
                long long h = 1;
                while ((h + 1) * (h + 2) / 2 < over) ++h;  // simplex_weights (problems.cpp:205-218)
                pp.h = h;
                pp.rows = (h + 1) * (h + 2) / 2;
            }
            thrust::device_vector<double> dF(pp.rows * m);
            thrust::device_vector<unsigned char> feas(pp.rows);
            thrust::device_vector<int> noob(1, 0);
            pp.F = thrust::raw_pointer_cast(dF.data());
            pp.feas = thrust::raw_pointer_cast(feas.data());
            pp.n_oob = thrust::raw_pointer_cast(noob.data());
            pf_candidates_kernel<<<blocks_for(pp.rows, 128), 128>>>(pp);
            CK(cudaGetLastError());
            if ((int)noob[0]) throw std::invalid_argument("evaluate: front candidate rows out of bounds");
            thrust::device_vector<long long> cand(pp.rows);
            auto end = thrust::copy_if(thrust::device, thrust::counting_iterator<long long>(0),
                                       thrust::counting_iterator<long long>(pp.rows), feas.begin(), cand.begin(),
                                       NonZero{});
            cand.resize(end - cand.begin());
            if ((long long)cand.size() >= std::max<long long>(n_points, 1)) {
                // nondominated_rows (fronts.cpp:15-42): m = 2 drops duplicates, m = 3 keeps them
                auto kept = front_filter(pp.F, m, cand, m == 2 ? 1 : 0);  // lexicographic order
                const long long nk = (long long)kept.size();
                const bool enough = nk >= n_points;
                if (enough || attempt == 3) {
                    std::vector<double> h;
                    if (!enough || nk <= n_points || n_points == 0) {
                        // the filtered rows in their original order (subsample_front returns F)
                        thrust::sort(thrust::device, kept.begin(), kept.end());
                        thrust::device_vector<double> o(nk * m);
                        gather_rows_kernel<<<blocks_for(nk, 256), 256>>>(pp.F, thrust::raw_pointer_cast(kept.data()),
                                                                        nk, m, thrust::raw_pointer_cast(o.data()));
                        h.resize(nk * m);
                        thrust::copy(o.begin(), o.end(), h.begin());
                        emit(h, nk);
                    } else {
                        // subsample_front (fronts.cpp:86-103): stable lexicographic order, even picks
                        thrust::device_vector<double> o(n_points * m);
                        pf_pick_kernel<<<blocks_for(n_points, 256), 256>>>(
                            pp.F, thrust::raw_pointer_cast(kept.data()), nk, n_points, m,
                            thrust::raw_pointer_cast(o.data()));
                        h.resize(n_points * m);
                        thrust::copy(o.begin(), o.end(), h.begin());
                        emit(h, n_points);
                    }
                    CK(cudaGetLastError());
                    return;
                }
            }
            over *= 4;
            if (m >= 3) over = std::min<long long>(over, 50000);
        }
        throw std::runtime_error("pf_reference: could not build a feasible front for " + p->name);
    });
}

int gmpea_metric_front(const double* F, const double* cv, int64_t n, int32_t m, int64_t* idx, int64_t* count) {
    return guarded([&] {
        if (m < 2 || m > 3) throw std::invalid_argument("metric_front: m must be 2 or 3");
        *count = 0;
        if (n <= 0) return;
        require_device();
        thrust::device_vector<double> dF(F, F + n * m), dcv(cv, cv + n);
        thrust::device_vector<long long> cand(n);
        auto end = thrust::copy_if(thrust::device, thrust::counting_iterator<long long>(0),
                                   thrust::counting_iterator<long long>(n), cand.begin(),
                                   IsFeasible{thrust::raw_pointer_cast(dcv.data())});
        cand.resize(end - cand.begin());
        auto kept = front_filter(thrust::raw_pointer_cast(dF.data()), m, cand);
        thrust::sort(thrust::device, kept.begin(), kept.end());
        std::vector<long long> h(kept.size());
        thrust::copy(kept.begin(), kept.end(), h.begin());
        for (size_t i = 0; i < h.size(); ++i) idx[i] = h[i];
        *count = (int64_t)h.size();
    });
}

int gmpea_igd(const double* A, int64_t na, const double* R, int64_t nr, int32_t m, double* out) {
    return guarded([&] {
        if (nr <= 0) throw std::invalid_argument("igd: empty reference front");
        if (na <= 0) {
            *out = std::numeric_limits<double>::infinity();
            return;
        }
        if (m < 1 || m > 3) throw std::invalid_argument("igd: objective count mismatch");
        require_device();
        thrust::device_vector<double> dA(A, A + na * m), dR(R, R + nr * m), res(1);
        thrust::device_vector<unsigned long long> best(nr, 0x7ff0000000000000ull);  // +inf
        int gx = (int)std::min<long long>(blocks_for(na, 256), 64);
        igd_min_kernel<<<dim3(gx, (unsigned)nr), 256>>>(thrust::raw_pointer_cast(dA.data()), na,
                                                         thrust::raw_pointer_cast(dR.data()), nr, m,
                                                         thrust::raw_pointer_cast(best.data()));
        igd_sum_kernel<<<1, 1>>>(thrust::raw_pointer_cast(best.data()), nr, thrust::raw_pointer_cast(res.data()));
        CK(cudaGetLastError());
        *out = res[0];
    });
}

int gmpea_hypervolume(const double* P, int64_t n, int32_t m, const double* ref, double* out) {
    return guarded([&] {
        if (m < 2 || m > 3) throw std::invalid_argument("hypervolume: m must be 2 or 3 on device");
        *out = 0.0;
        if (n <= 0) return;
        require_device();
        thrust::device_vector<double> dP(P, P + n * m), dref(ref, ref + m);
        const double* pP = thrust::raw_pointer_cast(dP.data());
        thrust::device_vector<long long> cand(n);
        auto end = thrust::copy_if(thrust::device, thrust::counting_iterator<long long>(0),
                                   thrust::counting_iterator<long long>(n), cand.begin(),
                                   InsideBox{pP, thrust::raw_pointer_cast(dref.data()), m});
        cand.resize(end - cand.begin());
        auto xy = front_filter(pP, m, cand);  // hv_relevant, sorted by (x, y[, z])
        const long long cnt = (long long)xy.size();
        if (cnt == 0) return;
        thrust::device_vector<double> slab(m == 2 ? 1 : cnt), res(1);
        thrust::device_vector<long long> zorder, zrank;
        if (m == 3) {
            zorder = xy;
            thrust::sort(thrust::device, zorder.begin(), zorder.end(), ZLess{pP});
            zrank.resize(n);
            thrust::scatter(thrust::device, thrust::counting_iterator<long long>(0),
                            thrust::counting_iterator<long long>(cnt), zorder.begin(), zrank.begin());
        }
        hv_slab_kernel<<<blocks_for(m == 2 ? 1 : cnt, 128), 128>>>(
            pP, thrust::raw_pointer_cast(xy.data()), m == 3 ? thrust::raw_pointer_cast(zrank.data()) : nullptr,
            cnt, m, m == 2 ? 1 : cnt, thrust::raw_pointer_cast(dref.data()), thrust::raw_pointer_cast(slab.data()));
        CK(cudaGetLastError());
        if (m == 2) {
            *out = slab[0];
            return;
        }
        hv3_sum_kernel<<<1, 1>>>(pP, thrust::raw_pointer_cast(zorder.data()), cnt,
                                 thrust::raw_pointer_cast(dref.data()), thrust::raw_pointer_cast(slab.data()),
                                 thrust::raw_pointer_cast(res.data()));
        CK(cudaGetLastError());
        *out = res[0];
    });
}

int gmpea_run_config_default(gmpea_run_config* c) {
    // RunConfig defaults (gmpea.hpp:113-127)
    *c = gmpea_run_config{};
    c->n = 100;
    c->k_max = 0;
    c->time_budget_s = -1.0;
    c->eval_budget = -1;
    c->seed = 1;
    c->op = GMPEA_OP_SBX_PM;
    gmpea_operator_params_default(&c->params);
    c->theta = 5.0;
    c->t1 = 5;
    c->t2 = 20;
    c->record_walltime = 1;
    c->device = 0;
    c->stream = 0;
    return GMPEA_OK;
}

int gmpea_engine_create(const gmpea_problem* p, const gmpea_run_config* cfg, gmpea_engine** out) {
    return guarded([&] {
        if (!p || !cfg || !out) throw std::invalid_argument("gmpea_engine_create: null argument");
        require_device();
        auto e = std::make_unique<gmpea_engine>();
        e->setup(p, *cfg);
        *out = e.release();
    });
}

int gmpea_engine_set_population(gmpea_engine* e, int32_t which, const double* X) {
    return guarded([&] { e->set_population(which, X); });
}

int gmpea_engine_run(gmpea_engine* e) {
    return guarded([&] { e->run(); });
}

int gmpea_engine_step(gmpea_engine* e, int64_t gens) {
    return guarded([&] { e->step(gens); });
}

int gmpea_engine_sync(gmpea_engine* e) {
    return guarded([&] {
        CK(cudaStreamSynchronize(e->s));
        e->check_errors(-1);
    });
}

int64_t gmpea_engine_effective_n(const gmpea_engine* e) { return e ? e->N : 0; }

int gmpea_engine_history(gmpea_engine* e, gmpea_gen_record* out, int64_t cap, int64_t* nrec) {
    return guarded([&] {
        auto h = e->history();
        int64_t k = std::min<int64_t>(cap, (int64_t)h.size());
        if (out) std::copy(h.begin(), h.begin() + k, out);
        *nrec = (int64_t)h.size();
    });
}

int gmpea_engine_record_async(gmpea_engine* e, gmpea_raw_record* dst) {
    return guarded([&] { e->record_async(dst); });
}

int gmpea_engine_replacements(gmpea_engine* e, int64_t* out, int64_t cap, int64_t* nrec) {
    return guarded([&] {
        auto h = e->replacements();
        int64_t k = std::min<int64_t>(cap, (int64_t)h.size());
        if (out) std::copy(h.begin(), h.begin() + k, out);
        *nrec = (int64_t)h.size();
    });
}

int gmpea_engine_last_record(gmpea_engine* e, gmpea_gen_record* out) {
    return guarded([&] {
        *out = e->last_record();
        e->check_errors(-1);
    });
}

int gmpea_engine_get_population(gmpea_engine* e, int32_t which, double* X, double* F, double* C, double* cv) {
    return guarded([&] { e->get_population(which, X, F, C, cv); });
}

int gmpea_engine_ideal(gmpea_engine* e, double* z) {
    return guarded([&] {
        DevState h = e->read_state();
        for (int k = 0; k < e->m; ++k) z[k] = ordered_to_float(h.zbits[k]);
    });
}

int gmpea_engine_neighborhoods(gmpea_engine* e, uint32_t* B1, uint32_t* B2) {
    return guarded([&] {
        const long long o0 = e->own0 - e->e0, on = e->own1 - e->own0;
        uint32_t* outs[2] = {B1, B2};
        for (int q = 0; q < 2; ++q) {
            if (!outs[q]) continue;
            const int t = q ? e->t2 : e->t1;
            CK(cudaMemcpy(outs[q], e->B[q].p + o0 * t, (size_t)on * t * sizeof(int), cudaMemcpyDeviceToHost));
            for (long long k = 0; k < on * t; ++k) outs[q][k] += (uint32_t)e->e0;  // global slots
        }
    });
}

int gmpea_engine_profile(gmpea_engine* e, int64_t gens, double* ms) {
    return guarded([&] { e->profile(gens, ms); });
}

void gmpea_engine_destroy(gmpea_engine* e) { delete e; }

int gmpea_engine_shard_info(gmpea_engine* e, gmpea_shard_info* o) {
    return guarded([&] {
        *o = gmpea_shard_info{e->N, e->e0, e->e1, e->v0, e->v1, e->own0, e->own1, e->reach};
    });
}

int gmpea_engine_phase(gmpea_engine* e, int32_t phase) {
    return guarded([&] { e->phase(phase); });
}

int gmpea_engine_device_buffers(gmpea_engine* e, gmpea_device_buffers* o) {
    return guarded([&] {
        o->ideal_bits = e->st.p->zbits;
        for (int q = 0; q < 2; ++q) {
            o->rows[q] = e->pop[q].X.p;
            o->keys[q] = e->pop[q].Fcv.p;
        }
        o->row_bytes = (int64_t)e->geo.rs4 * 16;
    });
}

}  // extern "C"

// ---- comparison-algorithm operators (baselines.hpp; baselines.cu kernels in baselines.cuh)
namespace {

struct PosLess {  // rows of F at front positions, lexicographic, then position
    const double* F;
    const long long* front;
    int m;
    __host__ __device__ bool operator()(long long a, long long b) const {
        for (int c = 0; c < m; ++c) {
            const double x = F[front[a] * m + c], y = F[front[b] * m + c];
            if (x < y) return true;
            if (x > y) return false;
        }
        return a < b;
    }
};

__global__ void dup_zero_kernel(const double* F, const long long* front, const long long* order, long long k, int m,
                                double* dist) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q == 0 || q >= k) return;
    const long long a = front[order[q]], b = front[order[q - 1]];
    for (int c = 0; c < m; ++c)
        if (!(F[a * m + c] == F[b * m + c])) return;
    dist[order[q]] = 0.0;  // an earlier position holds the same row (baselines.cpp:84-90)
}

__global__ void gather_col_pos_kernel(const double* F, const long long* front, long long k, int m, int c,
                                      double* out) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < k) out[q] = F[front[q] * m + c];
}

struct FitBelowOne {
    const double* fit;
    __host__ __device__ bool operator()(long long i) const { return fit[i] < 1.0; }
};
struct FitAtLeastOne {
    const double* fit;
    __host__ __device__ bool operator()(long long i) const { return fit[i] >= 1.0; }
};
struct IsInfeasible {
    const double* cv;
    __host__ __device__ bool operator()(long long i) const { return cv[i] > 0.0; }
};

void check_cdp_cv(const double* cv, int64_t n, int32_t use_cdp) {
    if (!use_cdp || n < 2) return;
    for (int64_t i = 0; i < n; ++i)
        if (cv[i] < 0.0) throw std::invalid_argument("cdp_better: negative constraint violation");
}

// Pareto ranks of the rows `sub` by front peeling; returns the front count
long long peel_ranks(const DomRel& R, thrust::device_vector<long long>& sub, thrust::device_vector<long long>& rank) {
    const long long ns = (long long)sub.size();
    if (ns == 0) return 0;
    thrust::device_vector<int> cnt(ns), fsz(1, 0), nsz(1, 0);
    thrust::device_vector<long long> front(ns), next(ns);
    const long long* ps = thrust::raw_pointer_cast(sub.data());
    nds_count_kernel<<<blocks_for(ns, 128), 128>>>(R, ps, ns, thrust::raw_pointer_cast(cnt.data()));
    nds_front0_kernel<<<blocks_for(ns, 256), 256>>>(thrust::raw_pointer_cast(cnt.data()), ns,
                                                    thrust::raw_pointer_cast(front.data()),
                                                    thrust::raw_pointer_cast(fsz.data()));
    CK(cudaGetLastError());
    long long fsize = (int)fsz[0], r = 0;
    while (fsize > 0) {
        // fronts are sets: the order of `next` (atomic) does not affect ranks
        nds_set_rank_kernel<<<blocks_for(fsize, 256), 256>>>(ps, thrust::raw_pointer_cast(front.data()), fsize, r,
                                                             thrust::raw_pointer_cast(rank.data()));
        nsz[0] = 0;
        nds_peel_kernel<<<blocks_for(fsize * ns, 256), 256>>>(R, ps, ns, thrust::raw_pointer_cast(front.data()), fsize,
                                                              thrust::raw_pointer_cast(cnt.data()),
                                                              thrust::raw_pointer_cast(next.data()),
                                                              thrust::raw_pointer_cast(nsz.data()));
        CK(cudaGetLastError());
        fsize = (int)nsz[0];
        front.swap(next);
        ++r;
    }
    return r;
}

// spea2_fitness on device arrays (baselines.cpp:93-127)
void spea2_fitness_dev(const double* dF, const double* dcv, int64_t n, int32_t m, int32_t use_cdp, double* dfit) {
    if (n == 0) return;
    DomRel R{dF, dcv, m, use_cdp};
    thrust::device_vector<double> strength(n), raw(n);
    spea2_strength_kernel<<<blocks_for(n, 128), 128>>>(R, n, thrust::raw_pointer_cast(strength.data()));
    spea2_raw_kernel<<<blocks_for(n, 128), 128>>>(R, n, thrust::raw_pointer_cast(strength.data()),
                                                  thrust::raw_pointer_cast(raw.data()));
    size_t k = (size_t)std::sqrt((double)n);
    if (k >= (size_t)n) k = n > 1 ? n - 1 : 0;
    const long long nd = n - 1;  // distances per row
    const long long kk = nd > 0 ? (long long)(k < (size_t)nd ? k : nd - 1) : 0;
    spea2_sigma_kernel<<<(unsigned)n, 256>>>(dF, m, n, kk, thrust::raw_pointer_cast(raw.data()), dfit);
    CK(cudaGetLastError());
}

}  // namespace

namespace {

// nondominated_sort on device arrays (baselines.cpp:22-55)
void nds_dev(const double* dF, const double* dcv, int64_t n, int32_t m, int32_t use_cdp,
             thrust::device_vector<long long>& drank) {
    drank.assign(n, 0);
    if (n <= 0) return;
    thrust::device_vector<long long> sub(n);
    DomRel R{dF, dcv, m, 0};
    if (use_cdp) {
        auto end = thrust::copy_if(thrust::device, thrust::counting_iterator<long long>(0),
                                   thrust::counting_iterator<long long>(n), sub.begin(), IsFeasible{dcv});
        sub.resize(end - sub.begin());
    } else {
        thrust::sequence(thrust::device, sub.begin(), sub.end());
    }
    const long long rf = peel_ranks(R, sub, drank);
    if (!use_cdp) return;
    thrust::device_vector<long long> inf(n);
    auto e = thrust::copy_if(thrust::device, thrust::counting_iterator<long long>(0),
                             thrust::counting_iterator<long long>(n), inf.begin(), IsInfeasible{dcv});
    const long long ni = e - inf.begin();
    if (!ni) return;
    thrust::device_vector<double> u(ni);
    thrust::gather(thrust::device, inf.begin(), inf.begin() + ni, thrust::device_pointer_cast(dcv), u.begin());
    thrust::sort(thrust::device, u.begin(), u.end());
    const long long nu = thrust::unique(thrust::device, u.begin(), u.end()) - u.begin();
    nds_infeasible_rank_kernel<<<blocks_for(n, 256), 256>>>(dcv, n, thrust::raw_pointer_cast(u.data()), nu, rf,
                                                            thrust::raw_pointer_cast(drank.data()));
    CK(cudaGetLastError());
}

// crowding_distance on device arrays (baselines.cpp:56-91) for the rows dfront[0..k)
void crowd_dev(const double* pF, int32_t m, const long long* pf, int64_t k, thrust::device_vector<double>& dd) {
    dd.assign(k, 0.0);
    if (k <= 0) return;
    if (k <= 2) {
        thrust::fill(thrust::device, dd.begin(), dd.end(), std::numeric_limits<double>::infinity());
        return;
    }
    thrust::device_vector<double> key(k);
    thrust::device_vector<long long> order(k);
    for (int c = 0; c < m; ++c) {
        thrust::sequence(thrust::device, order.begin(), order.end());
        gather_col_pos_kernel<<<blocks_for(k, 256), 256>>>(pF, pf, k, m, c, thrust::raw_pointer_cast(key.data()));
        thrust::stable_sort_by_key(thrust::device, key.begin(), key.end(), order.begin());
        crowd_axis_kernel<<<blocks_for(k, 256), 256>>>(pF, m, c, pf, thrust::raw_pointer_cast(order.data()), k,
                                                       thrust::raw_pointer_cast(dd.data()));
    }
    thrust::sequence(thrust::device, order.begin(), order.end());
    thrust::sort(thrust::device, order.begin(), order.end(), PosLess{pF, pf, m});
    dup_zero_kernel<<<blocks_for(k, 256), 256>>>(pF, pf, thrust::raw_pointer_cast(order.data()), k, m,
                                                 thrust::raw_pointer_cast(dd.data()));
    CK(cudaGetLastError());
}

// spea2_select on device arrays (baselines.cpp:129-189); kept rows ascending
std::vector<long long> spea2_select_dev(const double* pF, const double* pcv, int64_t n, int32_t m, int32_t use_cdp,
                                        int64_t capacity) {
    std::vector<long long> out;
    if (n <= 0) return out;
    thrust::device_vector<double> dfit(n);
    double* pfit = thrust::raw_pointer_cast(dfit.data());
    spea2_fitness_dev(pF, pcv, n, m, use_cdp, pfit);
    thrust::device_vector<long long> kp(n);
    auto e = thrust::copy_if(thrust::device, thrust::counting_iterator<long long>(0),
                             thrust::counting_iterator<long long>(n), kp.begin(), FitBelowOne{pfit});
    long long nk = e - kp.begin();
    if (nk < capacity) {
        // fill with the dominated rows, lowest fitness first (stable)
        thrust::device_vector<long long> rest(n);
        auto e2 = thrust::copy_if(thrust::device, thrust::counting_iterator<long long>(0),
                                  thrust::counting_iterator<long long>(n), rest.begin(), FitAtLeastOne{pfit});
        const long long nr = e2 - rest.begin();
        thrust::device_vector<double> rf(nr);
        thrust::gather(thrust::device, rest.begin(), rest.begin() + nr, dfit.begin(), rf.begin());
        thrust::stable_sort_by_key(thrust::device, rf.begin(), rf.end(), rest.begin());
        const long long take = std::min<long long>(nr, capacity - nk);
        std::vector<long long> a(nk), b(take);
        thrust::copy(kp.begin(), kp.begin() + nk, a.begin());
        thrust::copy(rest.begin(), rest.begin() + take, b.begin());
        out = a;
        out.insert(out.end(), b.begin(), b.end());
        std::sort(out.begin(), out.end());
        return out;
    }
    // serial truncation (baselines.cpp:149-184) in one persistent block
    thrust::device_vector<unsigned char> alive(n, 0);
    thrust::device_vector<double> n1(nk), n2(nk), lv(nk);
    thrust::device_vector<long long> i1(nk), i2(nk), cand(nk);
    thrust::fill(thrust::device, thrust::make_permutation_iterator(alive.begin(), kp.begin()),
                 thrust::make_permutation_iterator(alive.begin(), kp.begin() + nk), (unsigned char)1);
    const long long* pk = thrust::raw_pointer_cast(kp.data());
    unsigned char* pa = thrust::raw_pointer_cast(alive.data());
    if (nk > capacity) {
        trunc_init_kernel<<<blocks_for(nk, 128), 128>>>(pF, m, pk, nk, pa, thrust::raw_pointer_cast(n1.data()),
                                                        thrust::raw_pointer_cast(i1.data()),
                                                        thrust::raw_pointer_cast(n2.data()),
                                                        thrust::raw_pointer_cast(i2.data()));
        trunc_loop_kernel<<<1, 1024>>>(pF, m, pk, nk, capacity, pa, thrust::raw_pointer_cast(n1.data()),
                                       thrust::raw_pointer_cast(i1.data()), thrust::raw_pointer_cast(n2.data()),
                                       thrust::raw_pointer_cast(i2.data()), thrust::raw_pointer_cast(lv.data()),
                                       thrust::raw_pointer_cast(cand.data()));
        CK(cudaGetLastError());
    }
    std::vector<unsigned char> h(n);
    thrust::copy(alive.begin(), alive.end(), h.begin());
    for (int64_t i = 0; i < n; ++i)
        if (h[i]) out.push_back(i);
    return out;
}

}  // namespace

int gmpea_nondominated_sort(const double* F, const double* cv, int64_t n, int32_t m, int32_t use_cdp,
                            int64_t* rank) {
    return guarded([&] {
        if (m < 1) throw std::invalid_argument("nondominated_sort: no objectives");
        check_cdp_cv(cv, n, use_cdp);
        if (n <= 0) return;
        require_device();
        thrust::device_vector<double> dF(F, F + n * m), dcv(cv, cv + n);
        thrust::device_vector<long long> drank;
        nds_dev(thrust::raw_pointer_cast(dF.data()), thrust::raw_pointer_cast(dcv.data()), n, m, use_cdp, drank);
        std::vector<long long> h(n);
        thrust::copy(drank.begin(), drank.end(), h.begin());
        for (int64_t i = 0; i < n; ++i) rank[i] = h[i];
    });
}

int gmpea_crowding_distance(const double* F, int64_t n, int32_t m, const int64_t* front, int64_t k, double* dist) {
    return guarded([&] {
        if (k <= 0) return;
        if (k <= 2) {
            for (int64_t q = 0; q < k; ++q) dist[q] = std::numeric_limits<double>::infinity();
            return;
        }
        for (int64_t q = 0; q < k; ++q)
            if (front[q] < 0 || front[q] >= n) throw std::invalid_argument("crowding_distance: front index out of range");
        require_device();
        thrust::device_vector<double> dF(F, F + n * m), dd;
        thrust::device_vector<long long> fr(front, front + k);
        crowd_dev(thrust::raw_pointer_cast(dF.data()), m, thrust::raw_pointer_cast(fr.data()), k, dd);
        thrust::copy(dd.begin(), dd.end(), dist);
    });
}

int gmpea_spea2_fitness(const double* F, const double* cv, int64_t n, int32_t m, int32_t use_cdp, double* fit) {
    return guarded([&] {
        check_cdp_cv(cv, n, use_cdp);
        if (n <= 0) return;
        require_device();
        thrust::device_vector<double> dF(F, F + n * m), dcv(cv, cv + n), dfit(n);
        spea2_fitness_dev(thrust::raw_pointer_cast(dF.data()), thrust::raw_pointer_cast(dcv.data()), n, m, use_cdp,
                          thrust::raw_pointer_cast(dfit.data()));
        thrust::copy(dfit.begin(), dfit.end(), fit);
    });
}

int gmpea_spea2_select(const double* F, const double* cv, int64_t n, int32_t m, int32_t use_cdp, int64_t capacity,
                       int64_t* keep, int64_t* count) {
    return guarded([&] {
        check_cdp_cv(cv, n, use_cdp);
        *count = 0;
        if (n <= 0) return;
        if (capacity < 0) throw std::invalid_argument("spea2_select: negative capacity");
        require_device();
        thrust::device_vector<double> dF(F, F + n * m), dcv(cv, cv + n);
        auto out = spea2_select_dev(thrust::raw_pointer_cast(dF.data()), thrust::raw_pointer_cast(dcv.data()), n, m,
                                    use_cdp, capacity);
        for (size_t i = 0; i < out.size(); ++i) keep[i] = out[i];
        *count = (int64_t)out.size();
    });
}

// ---- comparison algorithms as runs: run_cnsga2 / run_ccmo (baselines.cpp:320-459)
namespace {

__global__ void take_rows_kernel(const float4* X0, const float4* K0, const float4* X1, const float4* K1,
                                 const float4* X2, const float4* K2, long long n, const long long* idx, long long k,
                                 int rs4, float4* dX, float4* dK) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= k * rs4) return;
    const long long r = e / rs4;
    const int q = (int)(e - r * rs4);
    const long long src = idx[r], s = src / n, row = src - s * n;
    const float4* X = s == 0 ? X0 : (s == 1 ? X1 : X2);
    const float4* K = s == 0 ? K0 : (s == 1 ? K1 : K2);
    dX[r * rs4 + q] = X[row * rs4 + q];
    if (q == 0) dK[r] = K[row];
}

__global__ void col_kernel(const double* F, long long n, int m, int c, double* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = F[i * m + c];
}

__device__ __forceinline__ void seg_of(const long long* rs, long long n, long long q, long long& lo, long long& hi) {
    const long long r = rs[q];
    long long a = 0, b = q;  // first position with rank r
    while (a < b) {
        const long long mid = (a + b) / 2;
        if (rs[mid] < r)
            a = mid + 1;
        else
            b = mid;
    }
    lo = a;
    a = q;
    b = n - 1;  // last position with rank r
    while (a < b) {
        const long long mid = (a + b + 1) / 2;
        if (rs[mid] > r)
            b = mid - 1;
        else
            a = mid;
    }
    hi = a;
}

// crowding of every front at once: positions grouped by rank, F[:, c]-sorted
// within a front (stable: index order on ties), as crowding_distance sees them
__global__ void crowd_seg_kernel(const double* F, int m, int c, const long long* order, const long long* rs,
                                 long long n, double* crowd) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    long long lo, hi;
    seg_of(rs, n, q, lo, hi);
    const double inf = 1.0 / 0.0;
    if (hi - lo + 1 <= 2 || q == lo || q == hi) {
        crowd[order[q]] = inf;
        return;
    }
    const double flo = F[order[lo] * m + c], fhi = F[order[hi] * m + c];
    if (fhi == flo) return;
    crowd[order[q]] += (F[order[q + 1] * m + c] - F[order[q - 1] * m + c]) / (fhi - flo);
}

struct RankRowLess {
    const double* F;
    const long long* rank;
    int m;
    __host__ __device__ bool operator()(long long a, long long b) const {
        if (rank[a] != rank[b]) return rank[a] < rank[b];
        for (int c = 0; c < m; ++c) {
            const double x = F[a * m + c], y = F[b * m + c];
            if (x < y) return true;
            if (x > y) return false;
        }
        return a < b;
    }
};

__global__ void crowd_dup_kernel(const double* F, int m, const long long* order, const long long* rs, long long n,
                                 double* crowd) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q == 0 || q >= n || rs[q] != rs[q - 1]) return;
    long long lo, hi;
    seg_of(rs, n, q, lo, hi);
    if (hi - lo + 1 <= 2) return;  // crowding_distance returns before its duplicate pass
    const long long a = order[q], b = order[q - 1];
    for (int c = 0; c < m; ++c)
        if (!(F[a * m + c] == F[b * m + c])) return;
    crowd[a] = 0.0;
}

// crowding distance of every row within its own front (run_cnsga2's tournament keys)
void crowd_all_dev(const double* pF, int64_t n, int32_t m, const thrust::device_vector<long long>& rank,
                   thrust::device_vector<double>& crowd) {
    crowd.assign(n, 0.0);
    thrust::device_vector<double> key(n);
    thrust::device_vector<long long> order(n), rs(n);
    const long long* pr = thrust::raw_pointer_cast(rank.data());
    for (int c = 0; c < m; ++c) {
        thrust::sequence(thrust::device, order.begin(), order.end());
        col_kernel<<<blocks_for(n, 256), 256>>>(pF, n, m, c, thrust::raw_pointer_cast(key.data()));
        thrust::stable_sort_by_key(thrust::device, key.begin(), key.end(), order.begin());
        thrust::gather(thrust::device, order.begin(), order.end(), rank.begin(), rs.begin());
        thrust::stable_sort_by_key(thrust::device, rs.begin(), rs.end(), order.begin());
        crowd_seg_kernel<<<blocks_for(n, 256), 256>>>(pF, m, c, thrust::raw_pointer_cast(order.data()),
                                                      thrust::raw_pointer_cast(rs.data()), n,
                                                      thrust::raw_pointer_cast(crowd.data()));
    }
    thrust::sequence(thrust::device, order.begin(), order.end());
    thrust::sort(thrust::device, order.begin(), order.end(), RankRowLess{pF, pr, m});
    thrust::gather(thrust::device, order.begin(), order.end(), rank.begin(), rs.begin());
    crowd_dup_kernel<<<blocks_for(n, 256), 256>>>(pF, m, thrust::raw_pointer_cast(order.data()),
                                                  thrust::raw_pointer_cast(rs.data()), n,
                                                  thrust::raw_pointer_cast(crowd.data()));
    CK(cudaGetLastError());
}

struct CvIsZero {
    __host__ __device__ bool operator()(double v) const { return v == 0.0; }
};

// igd(metric_front(pop), ref) on device arrays (metrics.cpp:42-60, 155-175);
// +inf for an empty front, as the reference's IGD hook records it
double igd_dev(const double* dF, const double* dcv, long long n, int m, const double* dR, long long nr) {
    thrust::device_vector<long long> cand(n);
    auto end = thrust::copy_if(thrust::device, thrust::counting_iterator<long long>(0),
                               thrust::counting_iterator<long long>(n), cand.begin(), IsFeasible{dcv});
    cand.resize(end - cand.begin());
    auto kept = front_filter(dF, m, cand);
    const long long na = (long long)kept.size();
    if (na == 0) return std::numeric_limits<double>::infinity();
    thrust::sort(thrust::device, kept.begin(), kept.end());  // metric_front keeps row order
    thrust::device_vector<double> A(na * m), res(1);
    gather_rows_kernel<<<blocks_for(na, 256), 256>>>(dF, thrust::raw_pointer_cast(kept.data()), na, m,
                                                    thrust::raw_pointer_cast(A.data()));
    thrust::device_vector<unsigned long long> best(nr, 0x7ff0000000000000ull);
    const int gx = (int)std::min<long long>(blocks_for(na, 256), 64);
    igd_min_kernel<<<dim3(gx, (unsigned)nr), 256>>>(thrust::raw_pointer_cast(A.data()), na, dR, nr, m,
                                                     thrust::raw_pointer_cast(best.data()));
    igd_sum_kernel<<<1, 1>>>(thrust::raw_pointer_cast(best.data()), nr, thrust::raw_pointer_cast(res.data()));
    CK(cudaGetLastError());
    return res[0];
}

struct BaselineRun {
    const gmpea_problem* p;
    gmpea_run_config c;
    int algo, d, m, nc, npop;
    long long n;
    RowGeom geo;
    PopBuf pop[2], off[2], nxt[2], prev[2];
    DevBuf<DevState> st;
    DevBuf<int> bad[2];
    VaryParams vp{};
    VaryKernel init_k = nullptr, vary_k = nullptr;
    std::vector<gmpea_gen_record> hist;
    long long evals = 0;
    double loop_s = 0.0;
    thrust::device_vector<double> igd_ref;  // optional IGD hook front (experiment.cpp:200-205)
    long long n_ref = 0;
    gmpea_pop_hook hook = nullptr;          // optional host metric hook
    void* hook_user = nullptr;

    void setup(const gmpea_problem* prob, int a, const gmpea_run_config& cfg) {
        p = prob;
        c = cfg;
        algo = a;
        if (algo != 0 && algo != 1) throw std::invalid_argument("run_baseline: unknown algorithm");
        if (cfg.n <= 0) throw std::invalid_argument("run_baseline: population size must be positive");
        n = cfg.n;
        d = p->d;
        m = p->m;
        nc = p->nin + p->neq;
        npop = algo == 1 ? 2 : 1;
        CK(cudaSetDevice(cfg.device));
        geo = row_geom(d, nc, p->fam == FAM_WTA ? p->dev.wta_n8 : 0);
        for (int q = 0; q < npop; ++q) {
            pop[q].alloc(n, geo.rs4, n);
            off[q].alloc(n, geo.rs4, n);
            nxt[q].alloc(n, geo.rs4, n);
            bad[q].alloc(kMaxBadRows);
            if (c.time_budget_s > 0) prev[q].alloc(n, geo.rs4, n);
        }
        st.alloc(1);
        st.zero(0);
        init_state_kernel<<<1, 1>>>(st.p, m);
        vp.n = (int)n;
        vp.row0 = 0;
        vp.row_end = (int)n;
        vp.rs4 = geo.rs4;
        vp.srs4 = geo.srs4;
        vp.scratch8 = geo.stream8;
        vp.pop_id[0] = 1;
        vp.pop_id[1] = 2;
        vp.P = p->dev;
        vp.key = make_philox_key(c.seed);
        fill_op_params(vp, c.params, d);
        vp.eval = 1;
        vp.update_z = 0;
        vp.st = st.p;
        vp.bad_cap = kMaxBadRows;
        vp.tour = algo == 0 ? 1 : 2;
        vp.un = make_uidx((unsigned long long)n);
        for (int q = 0; q < npop; ++q) vp.bad_rows[q] = bad[q].p;
        init_k = vary_kernel_for(p->fam, MODE_INIT, 0);
        vary_k = vary_kernel_for(p->fam, MODE_VARY, OP_SBX, p->dev.uniform ? d : 0, p->dev.id, true);
    }

    void check() {
        DevState h{};
        CK(cudaMemcpy(&h, st.p, sizeof(DevState), cudaMemcpyDeviceToHost));
        if (!h.err) return;
        if (h.err == ERR_EVAL_OOB) {
            const int q = h.n_bad[0] > 0 ? 0 : 1;
            std::vector<int> r(std::min(h.n_bad[q], kMaxBadRows));
            CK(cudaMemcpy(r.data(), bad[q].p, r.size() * sizeof(int), cudaMemcpyDeviceToHost));
            throw std::invalid_argument(rows_message(r));
        }
        throw std::runtime_error("run_baseline: device error " + std::to_string(h.err));
    }

    // f64 objective rows / cv of the concatenation of key arrays
    void keys_f64(std::initializer_list<const float4*> src, thrust::device_vector<double>& F,
                  thrust::device_vector<double>& cv) {
        const long long tot = (long long)src.size() * n;
        F.resize(tot * m);
        cv.resize(tot);
        long long o = 0;
        for (const float4* k : src) {
            fcv_to_rows_kernel<<<blocks_for(n, 256), 256>>>(k, n, m, thrust::raw_pointer_cast(F.data()) + o * m,
                                                           thrust::raw_pointer_cast(cv.data()) + o);
            o += n;
        }
    }

    void take(int q, const std::vector<long long>& idx, const float4* X1, const float4* K1, const float4* X2,
              const float4* K2) {
        thrust::device_vector<long long> di(idx.begin(), idx.end());
        take_rows_kernel<<<blocks_for(n * geo.rs4, 256), 256>>>(pop[q].X.p, pop[q].Fcv.p, X1, K1, X2, K2, n,
                                                                thrust::raw_pointer_cast(di.data()), n, geo.rs4,
                                                                nxt[q].X.p, nxt[q].Fcv.p);
        CK(cudaGetLastError());
        std::swap(pop[q].X.p, nxt[q].X.p);
        std::swap(pop[q].Fcv.p, nxt[q].Fcv.p);
    }

    void record(long long gen) {
        thrust::device_vector<double> F, cv;
        keys_f64({pop[0].Fcv.p}, F, cv);
        const long long feas = thrust::count_if(thrust::device, cv.begin(), cv.end(), CvIsZero{});
        gmpea_gen_record r{};
        r.gen = gen;
        r.evals = evals;
        r.wall_ms = c.record_walltime ? loop_s * 1e3 : 0.0;
        r.feasible_ratio = (double)feas / (double)n;
        r.igd = r.hv = std::numeric_limits<double>::quiet_NaN();
        if (n_ref > 0) {  // metric hook: outside the loop clock
            r.igd = igd_dev(thrust::raw_pointer_cast(F.data()), thrust::raw_pointer_cast(cv.data()), n, m,
                            thrust::raw_pointer_cast(igd_ref.data()), n_ref);
            r.has_igd = 1;
        }
        if (hook) {
            std::vector<double> hX((size_t)n * d), hF((size_t)n * m), hC((size_t)n * nc), hcv(n);
            get_pop1(hX.data(), hF.data(), hC.data(), hcv.data());
            hook(hook_user, n, hX.data(), hF.data(), hC.data(), hcv.data(), &r.igd, &r.hv, &r.has_igd, &r.has_hv);
        }
        hist.push_back(r);
    }

    bool stop(long long gen, long long next) const {  // RunDriver::stop (baselines.cpp:300-307)
        const bool tb = c.time_budget_s > 0, eb = c.eval_budget > 0;
        const bool unbounded = c.k_max == 0 && (tb || eb);
        if (!unbounded && gen > c.k_max) return true;
        if (tb && loop_s >= c.time_budget_s) return true;
        if (eb && evals + next > c.eval_budget) return true;
        return false;
    }

    void generation(long long gen) {
        VaryParams g = vp;
        g.fixed_gen = (int)gen;
        thrust::device_vector<double> F, cv, fit[2];
        thrust::device_vector<long long> rank;
        thrust::device_vector<double> crowd;
        if (algo == 0) {
            // ranks and per-front crowding of the parents (baselines.cpp:332-344)
            keys_f64({pop[0].Fcv.p}, F, cv);
            nds_dev(thrust::raw_pointer_cast(F.data()), thrust::raw_pointer_cast(cv.data()), n, m, 1, rank);
            crowd_all_dev(thrust::raw_pointer_cast(F.data()), n, m, rank, crowd);
            g.trank[0] = thrust::raw_pointer_cast(rank.data());
            g.tkey[0] = thrust::raw_pointer_cast(crowd.data());
        } else {
            for (int q = 0; q < 2; ++q) {  // baselines.cpp:410-411
                keys_f64({pop[q].Fcv.p}, F, cv);
                fit[q].resize(n);
                spea2_fitness_dev(thrust::raw_pointer_cast(F.data()), thrust::raw_pointer_cast(cv.data()), n, m,
                                  q == 0 ? 1 : 0, thrust::raw_pointer_cast(fit[q].data()));
                g.tkey[q] = thrust::raw_pointer_cast(fit[q].data());
            }
        }
        for (int q = 0; q < npop; ++q) {
            g.parX[q] = pop[q].X.p;
            g.out[q] = off[q].X.p;
            g.outFcv[q] = off[q].Fcv.p;
        }
        launch_vary(vary_k, g, npop, 0);  // tournaments + SBX + PM + clip + evaluation
        CK(cudaGetLastError());
        check();
        if (algo == 0) {
            // merged pool: fronts in order, the last one cut by crowding (baselines.cpp:361-384)
            keys_f64({pop[0].Fcv.p, off[0].Fcv.p}, F, cv);
            const double* pF = thrust::raw_pointer_cast(F.data());
            thrust::device_vector<long long> mr;
            nds_dev(pF, thrust::raw_pointer_cast(cv.data()), 2 * n, m, 1, mr);
            std::vector<long long> hr(2 * n);
            thrust::copy(mr.begin(), mr.end(), hr.begin());
            const long long top = *std::max_element(hr.begin(), hr.end());
            std::vector<std::vector<long long>> fronts(top + 1);
            for (long long i = 0; i < 2 * n; ++i) fronts[hr[i]].push_back(i);
            std::vector<long long> chosen;
            for (long long r = 0; r <= top && (long long)chosen.size() < n; ++r) {
                const auto& fr = fronts[r];
                if ((long long)(chosen.size() + fr.size()) <= n) {
                    chosen.insert(chosen.end(), fr.begin(), fr.end());
                } else {
                    thrust::device_vector<long long> dfr(fr.begin(), fr.end());
                    thrust::device_vector<double> cd;
                    crowd_dev(pF, m, thrust::raw_pointer_cast(dfr.data()), (int64_t)fr.size(), cd);
                    std::vector<double> hcd(fr.size());
                    thrust::copy(cd.begin(), cd.end(), hcd.begin());
                    std::vector<size_t> order(fr.size());
                    std::iota(order.begin(), order.end(), 0);
                    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return hcd[a] > hcd[b]; });
                    for (size_t k : order) {
                        if ((long long)chosen.size() == n) break;
                        chosen.push_back(fr[k]);
                    }
                }
            }
            std::sort(chosen.begin(), chosen.end());
            take(0, chosen, off[0].X.p, off[0].Fcv.p, nullptr, nullptr);
        } else {
            // both offspring sets feed both selections (baselines.cpp:433-438)
            std::vector<long long> sel[2];
            for (int q = 0; q < 2; ++q) {
                keys_f64({pop[q].Fcv.p, off[0].Fcv.p, off[1].Fcv.p}, F, cv);
                sel[q] = spea2_select_dev(thrust::raw_pointer_cast(F.data()), thrust::raw_pointer_cast(cv.data()),
                                          3 * n, m, q == 0 ? 1 : 0, n);
            }
            for (int q = 0; q < 2; ++q) take(q, sel[q], off[0].X.p, off[0].Fcv.p, off[1].X.p, off[1].Fcv.p);
        }
        CK(cudaDeviceSynchronize());
    }

    void run() {
        VaryParams ip = vp;
        ip.fixed_gen = 0;
        for (int q = 0; q < npop; ++q) {
            ip.parX[q] = pop[q].X.p;
            ip.out[q] = pop[q].X.p;
            ip.outFcv[q] = pop[q].Fcv.p;
        }
        launch_vary(init_k, ip, npop, 0);  // random_population + evaluate (Philox INIT stream)
        CK(cudaGetLastError());
        check();
        const long long per = (long long)npop * n;
        evals = per;
        record(0);
        for (long long gen = 1; !stop(gen, per); ++gen) {
            const bool tb = c.time_budget_s > 0;
            if (tb)
                for (int q = 0; q < npop; ++q) {
                    CK(cudaMemcpy(prev[q].X.p, pop[q].X.p, (size_t)n * geo.rs4 * sizeof(float4), cudaMemcpyDeviceToDevice));
                    CK(cudaMemcpy(prev[q].Fcv.p, pop[q].Fcv.p, (size_t)n * sizeof(float4), cudaMemcpyDeviceToDevice));
                }
            const auto t0 = std::chrono::steady_clock::now();
            generation(gen);
            loop_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (tb && loop_s >= c.time_budget_s) {  // the crossing generation is discarded
                for (int q = 0; q < npop; ++q) {
                    std::swap(pop[q].X.p, prev[q].X.p);
                    std::swap(pop[q].Fcv.p, prev[q].Fcv.p);
                }
                break;
            }
            evals += per;
            record(gen);
        }
    }

    void get_pop1(double* X, double* F, double* C, double* cv) {
        DevBuf<double> tmp((size_t)n * (std::max({d, nc, m}) + 1));
        const float* rows = (const float*)pop[0].X.p;
        auto pull = [&](int col0, int k, double* out) {
            if (!out || k == 0) return;
            from_rows_kernel<<<blocks_for(n * k, 256), 256>>>(rows, geo.rs4 * 4, n, col0, k, tmp.p);
            CK(cudaMemcpy(out, tmp.p, (size_t)n * k * sizeof(double), cudaMemcpyDeviceToHost));
        };
        pull(0, d, X);
        pull(d, nc, C);
        if (F || cv) {
            fcv_to_rows_kernel<<<blocks_for(n, 256), 256>>>(pop[0].Fcv.p, n, m, tmp.p, tmp.p + (size_t)n * m);
            if (F) CK(cudaMemcpy(F, tmp.p, (size_t)n * m * sizeof(double), cudaMemcpyDeviceToHost));
            if (cv) CK(cudaMemcpy(cv, tmp.p + (size_t)n * m, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost));
        }
    }
};

}  // namespace

int gmpea_run_baseline(const gmpea_problem* p, int32_t algo, const gmpea_run_config* cfg, const double* igd_ref,
                       int64_t n_ref, gmpea_pop_hook hook, void* hook_user, gmpea_gen_record* hist, int64_t hist_cap,
                       int64_t* n_hist, double* X, double* F, double* C, double* cv) {
    return guarded([&] {
        if (!p || !cfg) throw std::invalid_argument("run_baseline: null argument");
        require_device();
        BaselineRun r;
        r.setup(p, algo, *cfg);
        r.hook = hook;
        r.hook_user = hook_user;
        if (igd_ref && n_ref > 0) {
            r.igd_ref.assign(igd_ref, igd_ref + n_ref * p->m);
            r.n_ref = n_ref;
        }
        r.run();
        *n_hist = (int64_t)r.hist.size();
        if (hist) std::copy(r.hist.begin(), r.hist.begin() + std::min<int64_t>(hist_cap, r.hist.size()), hist);
        r.get_pop1(X, F, C, cv);
    });
}
