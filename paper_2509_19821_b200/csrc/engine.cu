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
#include "common.cuh"
#include <dlfcn.h>
#include <nccl.h>

#include "exchange.cuh"
#include "host.cuh"
#include "select.cuh"
#include "problems.cuh"
#include "topology.cuh"

using namespace gmpea_b200;

namespace gmpea_b200 {
namespace host {
thread_local std::string g_err;
}  // namespace host
}  // namespace gmpea_b200

namespace {

// NCCL, resolved at run time from the process's libnccl.so.2 (torch's own when
// a torch process already loaded it, else the system one): only sharded
// multi-process runs need it, and the library links no NCCL at build time.
struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    static Nccl& get() {
        static Nccl n = [] {
            Nccl x;
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
            if (!h) return x;
            auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(h, name)); };
            sym(x.GetUniqueId, "ncclGetUniqueId");
            sym(x.CommInitRank, "ncclCommInitRank");
            sym(x.CommDestroy, "ncclCommDestroy");
            sym(x.AllReduce, "ncclAllReduce");
            sym(x.Broadcast, "ncclBroadcast");
            sym(x.Send, "ncclSend");
            sym(x.Recv, "ncclRecv");
            sym(x.GroupStart, "ncclGroupStart");
            sym(x.GroupEnd, "ncclGroupEnd");
            sym(x.GetErrorString, "ncclGetErrorString");
            return x;
        }();
        if (!n.GroupEnd || !n.AllReduce || !n.Send || !n.CommInitRank || !n.GetErrorString)
            throw std::runtime_error("NCCL (libnccl.so.2) is not available: a multi-process sharded run needs it");
        return n;
    }
};

#define NK(expr)                                                                                   \
    do {                                                                                           \
        ncclResult_t r_ = (expr);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            throw nccl_error(std::string(#expr) + ": " + Nccl::get().GetErrorString(r_));         \
    } while (0)

// wta_scenario (wta.cpp:23-49): sizes grow with the index, tables from the
// reference's seeded mt19937_64 draws (rng.hpp:18-30).  num > 10 continues
// the same formula (synthetic instances; the reference stops at P10)
constexpr int kWtaMaxScenario = 123;  // 3 + 122 / 2 = 64 vehicles: the engine's limit
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



void make_wta(gmpea_problem& p, const WtaHost& w) {
    if (w.targets <= 0 || w.vehicles <= 0) throw std::invalid_argument("WTA: empty scenario");
    if (w.vehicles > kWtaMaxVehicles)
        throw std::invalid_argument("WTA: at most " + std::to_string(kWtaMaxVehicles) + " vehicles");
    int slots = 0;
    for (int s : w.strikes) slots += s;
    if (slots > kWtaMaxSlots)
        throw std::invalid_argument("WTA: at most " + std::to_string(kWtaMaxSlots) + " strike slots");
    for (int c : w.cap)
        if (c < 0) throw std::invalid_argument("WTA: negative vehicle capacity");
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

__global__ void fcv_from_rows_kernel(const double* F, const double* cv, long long n, int m, float4* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 o = make_float4((float)F[i * m], (float)F[i * m + 1], m > 2 ? (float)F[i * m + 2] : 0.0f,
                           (float)cv[i]);
    out[i] = o;
}


__global__ void u32_to_i32_kernel(const unsigned* in, long long n, int* out, int lim, int* err) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    unsigned v = in[e];
    if (v >= (unsigned)lim) atomicExch(err, 1);
    out[e] = (int)v;
}


// the run state after the initial populations are evaluated (gmpea.cpp:430-437):
// generation 1 next, clocks and budget armed; an earlier error stops the run
__global__ void reset_state_kernel(DevState* st, unsigned long long budget_ns, int rec_cap) {
    st->gen = 1;
    st->discard = 0;
    st->t_gen_start = 0;
    st->loop_ns = 0;
    st->budget_ns = budget_ns;
    st->gens_done = 0;
    st->rec_base = 0;
    st->rec_cap = rec_cap;
    st->stop = 0;
    if (st->err) halt(st);
}

// host rows (f64, row-major) -> fp32 rows, with the reference's f64 bounds
// check (problems.cpp:554-568); offending rows (global index) go to the run
// state's second bad-row list and surface at the next synchronisation
__global__ void load_rows_kernel(const double* in, long long n, int k, float* out, int rs, const double* lo,
                                 const double* hi, long long row_base, DevState* st) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * k) return;
    const long long r = e / k;
    const int c = (int)(e % k);
    const double v = in[e];
    out[r * rs + c] = (float)v;
    if (!(v >= lo[c] && v <= hi[c])) {
        for (int cc = 0; cc < c; ++cc) {  // one entry per row: its first failing column
            const double w = in[r * k + cc];
            if (!(w >= lo[cc] && w <= hi[cc])) return;
        }
        const int q = atomicAdd(&st->n_bad[1], 1);
        if (q < kMaxBadRows) st->bad_rows[1][q] = (int)(r + row_base);
        atomicCAS(&st->err, 0, ERR_EVAL_OOB);
    }
}

__global__ void set_z_kernel(DevState* st, int m, float z0, float z1, float z2) {
    st->zbits[0] = float_to_ordered(z0);
    st->zbits[1] = float_to_ordered(z1);
    st->zbits[2] = m > 2 ? float_to_ordered(z2) : float_to_ordered(0.0f);
    st->zbits[3] = float_to_ordered(0.0f);  // the go flag (common.cuh halt)
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

}  // namespace

namespace gmpea_b200 {
namespace host {

// the generation kernel is compiled per family (vary_<family>.cu) for the
// registered suites' dimension
VaryKernel vary_kernel_for(const ProbDev& P, int mode, int op, bool tour) {
    tour = tour && mode == MODE_VARY;
    // the dimension-specialised kernels assume uniform bounds
    const int d = P.uniform ? P.d : 0, id = P.id;
    switch (P.fam) {
        case FAM_LIR: return vary_kernel_lir(mode, op, d, id, tour);
        case FAM_DTLZ: return vary_kernel_dtlz(mode, op, d, id, tour);
        case FAM_WTA: return vary_kernel_wta(mode, op, d, P.wta_slots > kWtaNarrowSlots ? 1 : 0, tour);
        case FAM_DAS: return vary_kernel_das(mode, op, d, id, tour);
        default: return vary_kernel_mw(mode, op, d, id, tour);
    }
}

}  // namespace host
}  // namespace gmpea_b200

namespace {

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
        if (lattice && m <= 3 && n > 4096) {  // the window search knows the m <= 3 lattices
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

// the aggregation (PBI / Tchebycheff) and reverse-table layout are
// compile-time parameters of the selection kernels
static void launch_op1_kernel(int blocks, int agg, const Op1Params& p, cudaStream_t s) {
    if (agg == AGG_TCH)
        op1_kernel<AGG_TCH><<<blocks, 256, 0, s>>>(p);
    else
        op1_kernel<AGG_PBI><<<blocks, 256, 0, s>>>(p);
}

// select over parent slots [row0, row0 + rows) of both populations (grid y)
static void launch_select_kernel(int rows, bool pack, int agg, const SelParams& p, cudaStream_t s) {
    const dim3 grid(blocks_for(rows, kSelectBS), 2);
    if (agg == AGG_TCH) {
        if (pack)
            select_kernel<true, AGG_TCH><<<grid, kSelectBS, 0, s>>>(p);
        else
            select_kernel<false, AGG_TCH><<<grid, kSelectBS, 0, s>>>(p);
    } else {
        if (pack)
            select_kernel<true, AGG_PBI><<<grid, kSelectBS, 0, s>>>(p);
        else
            select_kernel<false, AGG_PBI><<<grid, kSelectBS, 0, s>>>(p);
    }
}

static void check_aggregation(int agg) {
    if (agg != GMPEA_AGG_PBI && agg != GMPEA_AGG_TCH) throw std::invalid_argument("unknown aggregation");
}

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
    long long rec_base = 0;           // generation held by device record slot 0
    std::vector<DevRecord> archive;   // drained records of generations < rec_base
    DevBuf<float4> U;
    DevBuf<int> B[2], R[2], Rdeg[2];
    DevBuf<uint2> Rp[2];
    bool rpack = false;  // select reads the int16-packed reverse neighbourhood
    int maxdeg[2] = {0, 0};
    PopBuf pop[2], off[2], undo[2];
    DevBuf<float4> eff[2];
    DevBuf<unsigned char> srcbits;
    DevBuf<int> ustamp[2];
    int* host_flag = nullptr;
    DevBuf<unsigned> done_ctr;
    DevBuf<double> staging;  // f64 row-major staging for population transfers
    int* host_flag_dev = nullptr;

    VaryParams vp{};
    PmGaps gaps;  // the PM gap table vp.pm_gap points into
    Op1Params op1p{};
    SelParams sp{};
    RestoreParams rp{};
    VaryKernel vary = nullptr;
    cudaGraphExec_t graph = nullptr;
    cudaGraphExec_t graph_first = nullptr;

    long long gens_enqueued = 0;  // generations launched (host view)
    long long gen_limit = 0;      // max generations allowed by k_max / eval budget (-1 = inf)
    bool finished = false;

    // ---- weight-region shards with the exchange inside the engine
    int world = 1, rank = 0;   // shards of the run, this one's index
    bool exchange = false;     // the engine exchanges z / boundary rows itself
    bool member = false;       // a shard of a multi-device handle (the handle captures)
    bool follower = false;     // time budget: rank 0 keeps the loop clock
    ncclComm_t comm = nullptr; // one process per GPU
    struct Halo {
        int peer;
        long long send0, send1, recv0, recv1;  // global slot ranges
    };
    std::vector<Halo> halos;
    DevBuf<LeadState> lead;    // rank 0's loop state (time budget)
    int* lead_flag = nullptr;  // host-mapped: the run's agreed stop flag
    int* lead_flag_dev = nullptr;
    // multi-device handle (gmpea_engine_create_multi): one shard per device
    std::vector<std::unique_ptr<gmpea_problem>> member_prob;
    std::vector<std::unique_ptr<gmpea_engine>> members;
    std::vector<int> member_dev;

    ~gmpea_engine() {
        if (!members.empty()) {  // (no throwing calls in a destructor)
            for (size_t k = 0; k < members.size(); ++k) {
                cudaSetDevice(member_dev[k]);
                cudaStreamSynchronize(members[k]->s);
            }
            destroy_group_events();
        }
        members.clear();
        if (graph) cudaGraphExecDestroy(graph);
        if (graph_first) cudaGraphExecDestroy(graph_first);
        if (host_flag) cudaFreeHost(host_flag);
        if (lead_flag) cudaFreeHost(lead_flag);
        if (comm) Nccl::get().CommDestroy(comm);
        if (own_stream && s) cudaStreamDestroy(s);
    }

    bool is_group() const { return !members.empty(); }

    // member_world > 0: shard member_rank of a multi-device handle
    void setup(const gmpea_problem* p, const gmpea_run_config& c, int member_world = 0, int member_rank = 0) {
        prob = p;
        cfg = c;
        if (c.n <= 0) throw std::invalid_argument("reference_vectors: target_n must be positive");
        if (c.n > (1ll << 30)) throw std::invalid_argument("engine: n too large");
        if (p->m > kMaxM || p->m < 2) throw std::invalid_argument("engine: objectives must be 2 or 3");
        check_aggregation(c.aggregation);
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
        if (member_world > 0 || c.world > 1 || (c.world == 1 && c.nccl_id)) {
            // balanced weight-region shards, exchange inside the engine
            world = member_world > 0 ? member_world : c.world;
            rank = member_world > 0 ? member_rank : c.rank;
            if (world > kMaxShards) throw std::invalid_argument("engine: at most 16 shards");
            if (rank < 0 || rank >= world) throw std::invalid_argument("engine: rank outside [0, world)");
            if (c.shard_end > c.shard_begin) throw std::invalid_argument("engine: world and shard range are exclusive");
            if (member_world == 0 && !c.nccl_id) throw std::invalid_argument("engine: world > 1 needs an nccl_id");
            own0 = (long long)rank * N / world;
            own1 = (long long)(rank + 1) * N / world;
            sharded = world > 1;
            exchange = true;
            member = member_world > 0;
            follower = time_mode && rank > 0;
        } else if (c.shard_end > c.shard_begin) {
            if (c.shard_begin < 0 || c.shard_end > N)
                throw std::invalid_argument("engine: shard range outside [0, n)");
            own0 = c.shard_begin;
            own1 = c.shard_end;
            sharded = own0 > 0 || own1 < N;
        }
        // the caller-driven shards (gmpea_engine_phase) cannot agree on a deadline
        if (sharded && time_mode && !exchange)
            throw std::invalid_argument("engine: a sharded run takes k_max / eval budgets (the deadline would differ per rank)");

        st.alloc(1);
        st.zero(s);
        init_state_kernel<<<1, 1, 0, s>>>(st.p, m);
        if (follower) {
            static const int one = 1;
            CK(cudaMemcpyAsync(&st.p->follower, &one, sizeof(int), cudaMemcpyHostToDevice, s));
        }
        // generation limit (gmpea.cpp:456-459)
        bool unbounded = c.k_max == 0 && (time_mode || c.eval_budget > 0);
        long long lim = c.k_max > 0 ? c.k_max : (unbounded ? -1 : 0);
        if (c.eval_budget > 0) {
            long long e = c.eval_budget / (2ll * N) - 1;  // gens with evals + 2n <= budget
            if (e < 0) e = 0;
            lim = lim < 0 ? e : std::min(lim, e);
        }
        gen_limit = lim;
        // unbounded (time-budget) runs keep a window of records on the device
        // and drain it to the host archive (drain_records)
        long long window = 1ll << 16;
        if (const char* w = getenv("GMPEA_REC_WINDOW")) window = std::max(8ll, atoll(w));  // tests
        rec_cap = lim >= 0 ? lim + 2 : window;
        if (rec_cap > (1ll << 30)) throw std::invalid_argument("engine: generation limit too large");
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
                const long long narrowest = exchange ? N / world : own1 - own0;
                if (narrowest < 2 * reach)
                    throw std::invalid_argument("engine: shard narrower than twice the neighbourhood reach (" +
                                                std::to_string(2 * reach) + " slots)");
                // boundary rows: my first / last 2r owned rows to the neighbours,
                // theirs into my window (the exchange after every generation)
                if (exchange && reach > 0) {
                    if (rank > 0) halos.push_back({rank - 1, own0, own0 + 2 * reach, own0 - 2 * reach, own0});
                    if (rank < world - 1) halos.push_back({rank + 1, own1 - 2 * reach, own1, own1, own1 + 2 * reach});
                }
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
        pack_static();

        for (int q = 0; q < 2; ++q) {
            pop[q].alloc(n, geo.rs4, ld);
            off[q].alloc(n, geo.rs4, ld);
            eff[q].alloc(ld);
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
        if (exchange && time_mode) {
            lead.alloc(1);
            lead.zero(s);
            CK(cudaHostAlloc(&lead_flag, sizeof(int), cudaHostAllocMapped));
            *lead_flag = 0;
            CK(cudaHostGetDevicePointer((void**)&lead_flag_dev, lead_flag, 0));
        }

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
        fill_op_params(vp, c.params, d, gaps);
        vp.eval = 1;
        vp.update_z = 1;
        vp.fixed_gen = -1;
        vp.st = st.p;
        vp.bad_cap = kMaxBadRows;
        for (int q = 0; q < 2; ++q) {
            vp.B[q] = B[q].p;
            vp.bad_rows[q] = st.p->bad_rows[q];  // reported by check_errors
        }

        // initial populations (gmpea.cpp:430-437): Philox INIT stream
        for (int q = 0; q < 2; ++q) {
            vp.parX[q] = pop[q].X.p;
            vp.out[q] = pop[q].X.p;
            vp.outFcv[q] = pop[q].Fcv.p;
        }
        VaryParams ip = vp;
        ip.fixed_gen = 0;
        launch_vary(vary_kernel_for(p->dev, MODE_INIT, 0), ip, 2, s);
        CK(cudaGetLastError());
        finish_init();

        // generation parameter blocks
        for (int q = 0; q < 2; ++q) {
            vp.parX[q] = pop[q].X.p;
            vp.out[q] = off[q].X.p;
            vp.outFcv[q] = off[q].Fcv.p;
        }
        vary = vary_kernel_for(p->dev, MODE_VARY, c.op);
        vp.row0 = (int)(v0 - e0);
        vp.row_end = (int)(v1 - e0);
        op1p = Op1Params{(int)(v0 - e0), (int)(v1 - e0), m, (float)c.theta, sU ? sU : U.p, {off[0].Fcv.p, off[1].Fcv.p},
                         {eff[0].p, eff[1].p}, srcbits.p, st.p};
        sp = SelParams{};
        sp.n = n;
        sp.row0 = (int)(own0 - e0);
        sp.row_end = (int)(own1 - e0);
        sp.rs4 = geo.rs4;
        sp.ldr = ld;
        sp.m = m;
        sp.theta = (float)c.theta;
        sp.U = sU ? sU : U.p;
        for (int q = 0; q < 2; ++q) {
            sp.X[q] = pop[q].X.p;
            sp.Fcv[q] = pop[q].Fcv.p;
            sp.oX[q] = off[q].X.p;
            sp.oFcv[q] = off[q].Fcv.p;
            sp.eff[q] = eff[q].p;
            // the static tables from the L2-resident arena (pack_static), if any
            sp.R[q] = sRev[q] && !rpack ? (const int*)sRev[q] : R[q].p;
            sp.Rp[q] = rpack ? (sRev[q] ? (const uint2*)sRev[q] : Rp[q].p) : nullptr;
            sp.Rdeg[q] = sRdeg[q] ? sRdeg[q] : Rdeg[q].p;
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
        staging.alloc((size_t)n * (d + nc + m + 1));  // every plane of a population readback
        if (exchange && !member) {
            // one process per GPU: the communicator, then one eager exchange
            // (the initial ideal point is global, gmpea.cpp:435-437; it also
            // connects NCCL's channels before the generation graph captures them)
            ncclUniqueId id;
            std::memcpy(&id, c.nccl_id, sizeof(id));
            NK(Nccl::get().CommInitRank(&comm, world, id, rank));
            exchange_z();
            exchange_halo();
        }
        if (!sharded || comm) build_graph();
        if (c.igd_reference && c.igd_reference_rows > 0) {
            if (exchange || sharded) throw std::invalid_argument("igd_reference: unsharded runs only");
            igd_rows = c.igd_reference_rows;
            igd_ref.alloc((size_t)igd_rows * m);
            CK(cudaMemcpyAsync(igd_ref.p, c.igd_reference, (size_t)igd_rows * m * sizeof(double),
                               cudaMemcpyHostToDevice, s));
            igd_hist.assign(1, igd_now());  // record(0)
        }
        CK(cudaStreamSynchronize(s));
        check_errors(0);
    }

    // ---- the exchange steps of one generation (NCCL; a multi-device handle
    // runs the peer-memory forms of the same steps, group_generation)
    void exchange_z() {
        // ideal point MIN and the go flag (zbits[3]) over the shards
        if (comm) NK(Nccl::get().AllReduce(st.p->zbits, st.p->zbits, 4, ncclUint32, ncclMin, comm, s));
    }
    void exchange_lead(const LeadState* leader_lead) {
        // time budget: every shard adopts rank 0's clock / deadline decision
        if (!lead.p) return;
        if (rank == 0) lead_pack_kernel<<<1, 1, 0, s>>>(st.p, lead.p);
        if (comm) NK(Nccl::get().Broadcast(lead.p, lead.p, sizeof(LeadState), ncclUint8, 0, comm, s));
        follow_kernel<<<1, 1, 0, s>>>(st.p, comm ? lead.p : leader_lead, lead_flag_dev);
    }
    void exchange_halo() {
        if (!comm || halos.empty()) return;
        const Nccl& nc_ = Nccl::get();
        const size_t rb = (size_t)geo.rs4 * 16;
        NK(nc_.GroupStart());
        for (int q = 0; q < 2; ++q)
            for (const Halo& h : halos) {
                NK(nc_.Send(pop[q].X.p + (h.send0 - e0) * geo.rs4, (size_t)(h.send1 - h.send0) * rb, ncclUint8, h.peer,
                            comm, s));
                NK(nc_.Recv(pop[q].X.p + (h.recv0 - e0) * geo.rs4, (size_t)(h.recv1 - h.recv0) * rb, ncclUint8, h.peer,
                            comm, s));
            }
        NK(nc_.GroupEnd());
    }

    // evaluation of the initial populations done: z, record 0, gen = 1
    void finish_init() {
        init_state_kernel<<<1, 1, 0, s>>>(st.p, m);
        const int o0 = (int)(own0 - e0), on = (int)(own1 - own0);
        for (int q = 0; q < 2; ++q)
            z_of_kernel<<<blocks_for(on, 256), 256, 0, s>>>(pop[q].Fcv.p + o0, on, m, st.p);
        rec.zero(s);
        count_feasible_kernel<<<blocks_for(on, 256), 256, 0, s>>>(pop[0].Fcv.p, o0, o0 + on, &rec.p[0].feasible);
        // no host round trip: the state is reset on the device (errors of the
        // initial evaluation are kept and stop the run)
        reset_state_kernel<<<1, 1, 0, s>>>(
            st.p, time_mode ? (unsigned long long)std::llround(cfg.time_budget_s * 1e9) : 0ull, (int)rec_cap);
        CK(cudaGetLastError());
        archive.clear();
        rec_base = 0;
        gens_enqueued = 0;
        finished = false;
    }

    void set_population(int which, const double* X) {
        if (which != 1 && which != 2) throw std::invalid_argument("set_population: which must be 1 or 2");
        if (gens_enqueued) throw std::invalid_argument("set_population: the run has started");
        if (is_group()) return group_set_population(which, X);
        const int q = which - 1;
        // asynchronous (no host round trip): out-of-bounds rows are recorded on
        // the device and reported, as evaluate's invalid_argument, at the next
        // synchronisation (step, sync, population, history)
        DevBuf<double>& h = staging;
        // X holds all N rows; this engine keeps its window [e0, e1)
        CK(cudaMemcpyAsync(h.p, X + e0 * d, (size_t)n * d * sizeof(double), cudaMemcpyHostToDevice, s));
        load_rows_kernel<<<blocks_for((long long)n * d, 256), 256, 0, s>>>(
            h.p, n, d, (float*)pop[q].X.p, geo.rs4 * 4, prob->dlo64.p, prob->dhi64.p, e0, st.p);
        VaryParams ep = vp;
        ep.row0 = 0;
        ep.row_end = n;
        ep.parX[0] = pop[q].X.p;
        ep.out[0] = pop[q].X.p;
        ep.outFcv[0] = pop[q].Fcv.p;
        ep.update_z = 0;
        ep.fixed_gen = 0;
        launch_vary(vary_kernel_for(prob->dev, MODE_EVAL, 0), ep, 1, s);
        CK(cudaGetLastError());
        finish_init();
        exchange_z();  // NCCL shards: the ideal point of the new populations is global (all ranks call this)
        if (igd_rows > 0) igd_hist.assign(1, igd_now());
    }

    void enqueue_generation() {
        enqueue_phase1();
        exchange_z();      // sharded (NCCL): ideal point over the shards, in the graph
        enqueue_phase2();  // select's last block also publishes the stop flag
    }

    void launch_select() {
        launch_select_kernel((int)(own1 - own0), rpack, cfg.aggregation, sp, s);
    }
    void launch_op1() { launch_op1_kernel(blocks_for(v1 - v0, 256), cfg.aggregation, op1p, s); }

    // phase 1: variation + evaluation (+ local ideal-point partial)
    void enqueue_phase1() { launch_vary(vary, vp, 2, s); }
    // phase 2: OP1, selection, bookkeeping (a sharded run all-reduces z in between)
    void enqueue_phase2() {
        launch_op1();
        launch_select();  // + end_gen
        exchange_lead(nullptr);
        launch_restore();
        exchange_halo();
    }
    void launch_restore() {
        if (time_mode) restore_kernel<<<dim3(blocks_for(own1 - own0, 256), 2), 256, 0, s>>>(rp);
    }

    // ---- the selection's static tables (unit weights, reverse neighbourhood
    // in-degrees and rows) in one arena, so one L2 access-policy window can
    // keep them resident: select re-reads them every generation while
    // vary_eval streams ~600 MB through L2 in between.  Opt-in
    // (GMPEA_L2_PERSIST=1): measured, the persisting carve-out costs vary_eval
    // and op1 more L2 than it saves select (LIRCMOP13 N = 10^6: select
    // 0.0951 -> 0.0931 ms, vary_eval 0.208 -> 0.281, op1 0.017 -> 0.032;
    // profiles/r02/ab_l2_persist.txt)
    DevBuf<char> sarena;
    const float4* sU = nullptr;
    const int* sRdeg[2] = {nullptr, nullptr};
    const void* sRev[2] = {nullptr, nullptr};
    size_t persist_bytes = 0;

    void pack_static() {
        const char* env = getenv("GMPEA_L2_PERSIST");
        if (!env || *env != '1') return;
        int dev = 0, maxwin = 0, maxpersist = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev));
        CK(cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, dev));
        if (maxwin <= 0 || maxpersist <= 0) return;
        auto al = [](size_t b) { return (b + 255) / 256 * 256; };
        const size_t bU = (size_t)n * sizeof(float4), bd = (size_t)n * sizeof(int);
        size_t br[2];
        for (int q = 0; q < 2; ++q) br[q] = rpack ? Rp[q].n * sizeof(uint2) : R[q].n * sizeof(int);
        const size_t total = al(bU) + 2 * al(bd) + al(br[0]) + al(br[1]);
        sarena.alloc(total);
        size_t o = 0;
        auto put = [&](const void* src, size_t b) {
            char* dst = sarena.p + o;
            CK(cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToDevice, s));
            o += al(b);
            return (const void*)dst;
        };
        // the hottest first: the window may not cover everything
        for (int q = 1; q >= 0; --q) sRev[q] = put(rpack ? (const void*)Rp[q].p : (const void*)R[q].p, br[q]);
        for (int q = 1; q >= 0; --q) sRdeg[q] = (const int*)put(Rdeg[q].p, bd);
        sU = (const float4*)put(U.p, bU);
        persist_bytes = std::min<size_t>({total, (size_t)maxwin, (size_t)maxpersist});
        size_t cur = 0;
        CK(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
        if (cur < persist_bytes) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist_bytes));
    }

    // the access-policy window on the captured op1 / select nodes (not on
    // vary_eval, whose traffic streams)
    void set_l2_window(cudaGraph_t g) {
        if (!persist_bytes) return;
        size_t nn = 0;
        CK(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(g, nodes.data(), &nn));
        size_t lim = 0;
        CK(cudaDeviceGetLimit(&lim, cudaLimitPersistingL2CacheSize));
        cudaKernelNodeAttrValue v{};
        v.accessPolicyWindow.base_ptr = sarena.p;
        v.accessPolicyWindow.num_bytes = persist_bytes;
        v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)lim / (double)persist_bytes);
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType t;
            CK(cudaGraphNodeGetType(nd, &t));
            if (t != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams kp{};
            CK(cudaGraphKernelNodeGetParams(nd, &kp));
            if (kp.func == (void*)vary) continue;
            CK(cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v));
        }
    }

    // two graphs of one generation: graph_first also restarts the loop clock
    // (the first generation of a step() call), so step(1) is one launch
    cudaGraphExec_t capture_generation(bool clock) {
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t g;
        cudaGraphExec_t x;
        // NCCL may touch its own streams while its calls are captured
        CK(cudaStreamBeginCapture(cs, comm ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal));
        cudaStream_t saved = s;
        s = cs;
        if (clock) start_loop_clock();
        enqueue_generation();
        s = saved;
        CK(cudaStreamEndCapture(cs, &g));
        set_l2_window(g);
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

    // ---- the per-generation IGD hook (RunConfig::igd_metric, gmpea.cpp:442-453,
    // which the harness sets to igd(metric_front(pop1), ref) for problems with
    // a front, experiment.cpp:200-205): on the device, outside the loop clock
    DevBuf<double> igd_ref;
    long long igd_rows = 0;
    std::vector<double> igd_hist;  // index: generation

    double igd_now() {
        const long long o0 = own0 - e0, on = own1 - own0;
        double* tF = staging.p;
        double* tcv = tF + (size_t)on * m;
        fcv_to_rows_kernel<<<blocks_for(on, 256), 256, 0, s>>>(pop[0].Fcv.p + o0, on, m, tF, tcv);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));  // igd_dev works on the default stream
        return igd_dev(tF, tcv, on, m, igd_ref.p, igd_rows);
    }

    // enqueue up to k generations, respecting the generation limit
    long long step(long long k) {
        if (gen_limit >= 0) k = std::min(k, gen_limit - gens_enqueued);
        if (k <= 0) return 0;
        if (is_group()) return group_step(k);
        if (igd_rows == 0) return launch_gens(k);
        // with the IGD hook: one generation at a time, each its own loop-clock
        // interval, the metric after it (a discarded generation records none)
        long long done = 0;
        while (done < k) {
            if (launch_gens(1) == 0) break;
            ++done;
            const DevState h = read_state();
            if ((long long)igd_hist.size() <= h.gens_done) igd_hist.push_back(igd_now());
            if (h.stop) break;
        }
        return done;
    }

    long long launch_gens(long long k) {
        build_graph();
        long long done = 0;
        while (done < k) {
            // an unbounded run's record window: drain it before it fills
            long long room = rec_cap - 2 - (gens_enqueued - rec_base);
            if (room <= 0) {
                drain_records();
                room = rec_cap - 2 - (gens_enqueued - rec_base);
                if (room <= 0) break;  // the run stopped: nothing further would execute
            }
            const long long part = std::min(k - done, room);
            CK(cudaGraphLaunch(done == 0 ? graph_first : graph, s));
            for (long long i = 1; i < part; ++i) CK(cudaGraphLaunch(graph, s));
            gens_enqueued += part;
            done += part;
        }
        return done;
    }

    // moves the records of finished generations to the host archive and
    // restarts the device window at the next generation (syncs the stream)
    void drain_records() {
        CK(cudaStreamSynchronize(s));
        DevState h = read_state();
        if (h.stop) return;  // the run is over; nothing more will be written
        const long long upto = h.gen;  // generations < gen are complete
        const long long cnt = upto - rec_base;
        if (cnt <= 0) return;
        std::vector<DevRecord> r(cnt);
        CK(cudaMemcpyAsync(r.data(), rec.p, cnt * sizeof(DevRecord), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        archive.insert(archive.end(), r.begin(), r.end());
        rec_base = upto;
        rec.zero(s);
        int base = (int)rec_base;
        CK(cudaMemcpyAsync(&st.p->rec_base, &base, sizeof(int), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }

    // records of generations [0, gens_done] (archive + device window); the
    // feasible / replaced counts of every shard summed (a sharded run: all
    // ranks call this together)
    std::vector<DevRecord> all_records(long long gens_done) {
        std::vector<DevRecord> out(archive.begin(), archive.end());
        const long long cnt = std::min<long long>(gens_done + 1 - rec_base, rec_cap);
        if (cnt > 0) {
            std::vector<DevRecord> r(cnt);
            CK(cudaMemcpyAsync(r.data(), rec.p, cnt * sizeof(DevRecord), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            out.insert(out.end(), r.begin(), r.end());
        }
        out.resize(gens_done + 1);
        if (comm && !out.empty()) {
            std::vector<unsigned> c(2 * out.size());
            for (size_t k = 0; k < out.size(); ++k) {
                c[2 * k] = out[k].feasible;
                c[2 * k + 1] = out[k].replaced;
            }
            DevBuf<unsigned> dc(c.size());
            CK(cudaMemcpyAsync(dc.p, c.data(), c.size() * sizeof(unsigned), cudaMemcpyHostToDevice, s));
            NK(Nccl::get().AllReduce(dc.p, dc.p, c.size(), ncclUint32, ncclSum, comm, s));
            CK(cudaMemcpyAsync(c.data(), dc.p, c.size() * sizeof(unsigned), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            for (size_t k = 0; k < out.size(); ++k) {
                out[k].feasible = c[2 * k];
                out[k].replaced = c[2 * k + 1];
            }
        }
        return out;
    }

    // the run's records [0, gens_done]: a multi-device handle sums its shards
    std::vector<DevRecord> run_records() {
        if (!is_group()) return all_records(read_state().gens_done);
        on(0);
        const long long g = members[0]->read_state().gens_done;
        std::vector<DevRecord> out = members[0]->all_records(g);
        for (size_t k = 1; k < members.size(); ++k) {
            on(k);
            std::vector<DevRecord> r = members[k]->all_records(g);
            for (size_t i = 0; i < out.size(); ++i) {
                out[i].feasible += r[i].feasible;
                out[i].replaced += r[i].replaced;
            }
        }
        on(0);
        return out;
    }

    // slots whose records the history counts (all N when the shards are summed)
    long long counted_slots() const { return (comm || is_group()) ? N : own1 - own0; }

    // one generation in two phases (sharded runs; no graph, plain launches)
    void phase(int ph) {
        if (is_group() || comm) throw std::invalid_argument("phase: this run exchanges inside the engine");
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
            sync_all();
        } else {
            // time budget: keep at most two chunks in flight and stop launching
            // once the device reports the deadline (gmpea.cpp:458, :481-486).
            // Shards watch the agreed flag (rank 0's decision, follow_kernel)
            // and launch identical chunk sequences, so their collectives match.
            gmpea_engine& lead_e = is_group() ? *members[0] : *this;
            volatile int* flag = lead_e.exchange ? lead_e.lead_flag : lead_e.host_flag;
            const long long chunk = N / world >= 100000 ? 2 : 16;
            if (is_group()) on(0);
            cudaEvent_t ev[2];
            CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
            int k = 0;
            bool pending[2] = {false, false};
            for (;;) {
                if (pending[k]) {
                    CK(cudaEventSynchronize(ev[k]));
                    pending[k] = false;
                    if (*flag) break;
                }
                long long launched = step(chunk);
                if (launched == 0) break;
                CK(cudaEventRecord(ev[k], s));
                pending[k] = true;
                k ^= 1;
            }
            sync_all();
            cudaEventDestroy(ev[0]);
            cudaEventDestroy(ev[1]);
        }
        finished = true;
        check_errors(-1);
    }

    void sync_all() {
        if (!is_group()) {
            CK(cudaStreamSynchronize(s));
            return;
        }
        for (size_t k = 0; k < members.size(); ++k) {
            on(k);
            CK(cudaStreamSynchronize(members[k]->s));
        }
        on(0);
    }

    DevState read_state() {
        DevState h{};
        CK(cudaMemcpyAsync(&h, st.p, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return h;
    }

    void check_errors(int phase) {
        if (is_group()) {
            for (size_t k = 0; k < members.size(); ++k) {
                on(k);
                members[k]->check_errors(phase);
            }
            on(0);
            return;
        }
        DevState h = read_state();
        if (!h.err) return;
        std::string where = phase == 0 ? std::string("") :
            "run_gmpea: evaluation failed at generation " + std::to_string(h.err_gen) + ": ";
        if (h.err == ERR_EVAL_OOB) {
            // list 0: the evaluator's fp32 check, list 1: set_population's f64 check
            std::vector<int> r;
            for (int q = 0; q < 2; ++q) r.insert(r.end(), h.bad_rows[q], h.bad_rows[q] + std::min(h.n_bad[q], kMaxBadRows));
            std::sort(r.begin(), r.end());
            r.erase(std::unique(r.begin(), r.end()), r.end());
            // generation 0: the initial / injected populations (evaluate's invalid_argument)
            if (phase == 0 || h.err_gen == 0) throw std::invalid_argument(rows_message(r));
            throw std::runtime_error(where + rows_message(r));
        }
        if (h.err == ERR_NONFINITE) throw std::invalid_argument("non-finite mask source");
        if (h.err == ERR_NEG_CV) throw std::invalid_argument("fpr_better: negative constraint violation");
        if (h.err == ERR_RECORDS) throw std::runtime_error("engine: generation records were not drained");
        throw std::runtime_error("engine error " + std::to_string(h.err));
    }

    std::vector<gmpea_gen_record> history() {
        std::vector<DevRecord> r = run_records();
        const long long g = (long long)r.size() - 1;
        std::vector<gmpea_gen_record> out(g + 1);
        for (long long k = 0; k <= g; ++k) {
            gmpea_gen_record& o = out[k];
            o = gmpea_gen_record{};
            o.gen = k;
            o.evals = 2ll * N * (k + 1);
            o.wall_ms = cfg.record_walltime ? (k == 0 ? 0.0 : (double)r[k].loop_ns * 1e-6) : 0.0;
            o.feasible_ratio = (double)r[k].feasible / (double)counted_slots();
            o.igd = std::numeric_limits<double>::quiet_NaN();
            o.hv = std::numeric_limits<double>::quiet_NaN();
            if (k < (long long)igd_hist.size()) {
                o.igd = igd_hist[k];
                o.has_igd = 1;
            }
        }
        return out;
    }


    std::vector<int64_t> replacements() {
        std::vector<DevRecord> r = run_records();
        const long long g = (long long)r.size() - 1;
        std::vector<int64_t> out(g + 1);
        for (long long k = 0; k <= g; ++k) out[k] = k == 0 ? 0 : (int64_t)r[k].replaced;
        return out;
    }

    void record_async(void* dst) {
        static_assert(sizeof(DevRecord) == sizeof(gmpea_raw_record), "raw record layout");
        if (is_group()) {  // shard 0's record (its own slots' counts), in its stream order
            on(0);
            members[0]->gens_enqueued = gens_enqueued;
            members[0]->record_async(dst);
            return;
        }
        const long long k = gens_enqueued - rec_base;
        if (k < 0 || k >= rec_cap) throw std::invalid_argument("record_async: record outside the device window");
        CK(cudaMemcpyAsync(dst, rec.p + k, sizeof(DevRecord), cudaMemcpyDeviceToHost, s));
    }

    // the newest generation record only (one small D2H; the per-step result)
    gmpea_gen_record last_record() {
        if (is_group()) return history().back();
        struct {
            int gens_done;
        } g{};
        CK(cudaMemcpyAsync(&g.gens_done, &st.p->gens_done, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        DevRecord r{};
        const long long k = g.gens_done;
        if (k - rec_base >= 0 && k - rec_base < rec_cap) {
            CK(cudaMemcpyAsync(&r, rec.p + (k - rec_base), sizeof(DevRecord), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        } else if (k < (long long)archive.size()) {
            r = archive[k];
        }
        gmpea_gen_record o{};
        o.gen = k;
        o.evals = 2ll * N * (k + 1);
        o.wall_ms = cfg.record_walltime && k ? (double)r.loop_ns * 1e-6 : 0.0;
        o.feasible_ratio = (double)r.feasible / (double)(own1 - own0);  // this rank's slots
        o.igd = o.hv = std::numeric_limits<double>::quiet_NaN();
        return o;
    }

    // the owned rows [own0, own1) (all N unsharded)
    // the owned rows [own0, own1) (all N unsharded) of population `which`
    // (1, 2) or, with offspring = true, of the offspring stream `which` as the
    // last generation's variation + evaluation left it (diagnostic)
    void get_population(int which, double* X, double* F, double* C, double* cv, bool offspring = false) {
        if (which != 1 && which != 2) throw std::invalid_argument("get_population: which must be 1 or 2");
        check_errors(-1);  // never hand out a population a failed generation left behind
        if (is_group()) {  // the shards' owned rows in slot order
            for (size_t k = 0; k < members.size(); ++k) {
                on(k);
                gmpea_engine& e = *members[k];
                const long long o = e.own0;
                e.get_population(which, X ? X + o * d : nullptr, F ? F + o * m : nullptr, C ? C + o * nc : nullptr,
                                 cv ? cv + o : nullptr, offspring);
            }
            on(0);
            return;
        }
        const int q = which - 1;
        const long long o0 = own0 - e0, on = own1 - own0;
        const PopBuf& src = offspring ? off[q] : pop[q];
        // every plane is converted into its own part of the staging buffer and
        // copied out in stream order: one synchronisation for the whole readback
        double* tX = staging.p;
        double* tC = tX + (size_t)on * d;
        double* tF = tC + (size_t)on * nc;
        double* tcv = tF + (size_t)on * m;
        const float* rows = (const float*)(src.X.p + o0 * geo.rs4);
        if (X) {
            from_rows_kernel<<<blocks_for(on * d, 256), 256, 0, s>>>(rows, geo.rs4 * 4, on, 0, d, tX);
            CK(cudaMemcpyAsync(X, tX, (size_t)on * d * sizeof(double), cudaMemcpyDeviceToHost, s));
        }
        if (C && nc) {
            from_rows_kernel<<<blocks_for(on * nc, 256), 256, 0, s>>>(rows, geo.rs4 * 4, on, d, nc, tC);
            CK(cudaMemcpyAsync(C, tC, (size_t)on * nc * sizeof(double), cudaMemcpyDeviceToHost, s));
        }
        if (F || cv) {
            fcv_to_rows_kernel<<<blocks_for(on, 256), 256, 0, s>>>(src.Fcv.p + o0, on, m, tF, tcv);
            if (F) CK(cudaMemcpyAsync(F, tF, (size_t)on * m * sizeof(double), cudaMemcpyDeviceToHost, s));
            if (cv) CK(cudaMemcpyAsync(cv, tcv, (size_t)on * sizeof(double), cudaMemcpyDeviceToHost, s));
        }
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
    }

    // per-phase device times of `gens` generations (events on the launching
    // stream; a multi-device handle: shard 0's stream): ms = [vary_eval, op1,
    // select (+ end_gen), exchange + restore, total]
    void profile(long long gens, double* ms) {
        if (gen_limit >= 0) gens = std::min(gens, gen_limit - gens_enqueued);
        if (gens <= 0) throw std::invalid_argument("profile: no generations left");
        if (is_group()) {
            sync_all();
            on(0);
        } else {
            start_loop_clock();
        }
        std::vector<cudaEvent_t> ev(6 * gens);
        for (auto& e : ev) CK(cudaEventCreate(&e));
        for (long long g = 0; g < gens; ++g) {
            cudaEvent_t* e = &ev[6 * g];
            if (is_group()) {
                group_generation(g == 0, e);
                continue;
            }
            CK(cudaEventRecord(e[0], s));
            enqueue_phase1();
            CK(cudaEventRecord(e[1], s));
            exchange_z();
            CK(cudaEventRecord(e[2], s));
            launch_op1();
            CK(cudaEventRecord(e[3], s));
            launch_select();  // + end_gen
            CK(cudaEventRecord(e[4], s));
            exchange_lead(nullptr);
            launch_restore();
            exchange_halo();
            CK(cudaEventRecord(e[5], s));
        }
        CK(cudaGetLastError());
        sync_all();
        gens_enqueued += gens;
        double acc[5] = {0, 0, 0, 0, 0};
        auto dt = [&](cudaEvent_t a, cudaEvent_t b) {
            float t = 0.0f;
            CK(cudaEventElapsedTime(&t, a, b));
            return (double)t;
        };
        for (long long g = 0; g < gens; ++g) {
            cudaEvent_t* e = &ev[6 * g];
            acc[0] += dt(e[0], e[1]);
            acc[1] += dt(e[2], e[3]);
            acc[2] += dt(e[3], e[4]);
            acc[3] += dt(e[1], e[2]) + dt(e[4], e[5]);
            acc[4] += dt(e[0], e[5]);
        }
        for (auto& e : ev) cudaEventDestroy(e);
        for (int k = 0; k < 5; ++k) ms[k] = acc[k] / (double)gens;
        check_errors(-1);
    }

    // ================================================= multi-device handle
    // (gmpea_engine_create_multi): shard k runs on member_dev[k]; one
    // generation is one multi-device CUDA graph launched on shard 0's stream.
    std::vector<PeerStates> peers;       // per shard: every other shard's state
    std::vector<cudaEvent_t> gev[4];     // per shard: vary / select / finished / halo done
    cudaEvent_t gev_fork = nullptr, gev_lead = nullptr;

    void on(size_t k) const { CK(cudaSetDevice(member_dev[k])); }

    static std::unique_ptr<gmpea_problem> clone_problem(const gmpea_problem& p) {
        auto q = std::make_unique<gmpea_problem>();
        q->name = p.name;
        q->fam = p.fam;
        q->id = p.id;
        q->d = p.d;
        q->m = p.m;
        q->nin = p.nin;
        q->neq = p.neq;
        q->lo = p.lo;
        q->hi = p.hi;
        q->wta = p.wta;
        q->upload();  // on the current device
        return q;
    }

    void setup_group(const gmpea_problem* p, const gmpea_run_config& c, const int32_t* devices, int ndev) {
        if (!devices || ndev < 1 || ndev > kMaxShards)
            throw std::invalid_argument("gmpea_engine_create_multi: 1 to 16 devices");
        if (c.world > 1) throw std::invalid_argument("gmpea_engine_create_multi: world is for one process per GPU");
        if (c.shard_end > c.shard_begin) throw std::invalid_argument("gmpea_engine_create_multi: no shard range");
        prob = p;
        cfg = c;
        member_dev.assign(devices, devices + ndev);
        int ndevs = 0;
        CK(cudaGetDeviceCount(&ndevs));
        for (int dv : member_dev)
            if (dv < 0 || dv >= ndevs) throw std::invalid_argument("gmpea_engine_create_multi: no such device");
        // peer access between the distinct devices (z and the boundary rows)
        for (int a : member_dev)
            for (int b : member_dev) {
                if (a == b) continue;
                int ok = 0;
                CK(cudaDeviceCanAccessPeer(&ok, a, b));
                if (!ok) throw cuda_error("gmpea_engine_create_multi: no peer access between devices");
                CK(cudaSetDevice(a));
                cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else CK(e);
            }
        for (int k = 0; k < ndev; ++k) {
            on(k);
            member_prob.push_back(clone_problem(*p));
            gmpea_run_config ck = c;
            ck.device = member_dev[k];
            ck.stream = k == 0 ? c.stream : 0;
            ck.world = 0;
            ck.rank = 0;
            ck.nccl_id = nullptr;
            members.push_back(std::make_unique<gmpea_engine>());
            members.back()->setup(member_prob.back().get(), ck, ndev, k);
        }
        gmpea_engine& L = *members[0];
        N = L.N;
        d = L.d;
        m = L.m;
        nc = L.nc;
        t1 = L.t1;
        t2 = L.t2;
        H = L.H;
        geo = L.geo;
        reach = L.reach;
        own0 = e0 = v0 = 0;
        own1 = e1 = v1 = N;
        n = (int)N;
        world = ndev;
        exchange = true;
        sharded = ndev > 1;
        time_mode = L.time_mode;
        gen_limit = L.gen_limit;
        s = L.s;
        own_stream = false;
        peers.assign(ndev, PeerStates{});
        for (int k = 0; k < ndev; ++k)
            for (int j = 0; j < ndev; ++j)
                if (j != k) peers[k].st[peers[k].n++] = members[j]->st.p;
        for (int q = 0; q < 4; ++q) {
            gev[q].resize(ndev);
            for (int k = 0; k < ndev; ++k) {
                on(k);
                CK(cudaEventCreateWithFlags(&gev[q][k], cudaEventDisableTiming));
            }
        }
        on(0);
        CK(cudaEventCreateWithFlags(&gev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&gev_lead, cudaEventDisableTiming));
        exchange_z_eager();  // the initial ideal point is global (gmpea.cpp:435-437)
        graph = capture_group(false);
        graph_first = capture_group(true);
        on(0);
    }

    void destroy_group_events() {
        for (auto& v : gev)
            for (auto e : v) cudaEventDestroy(e);
        if (gev_fork) cudaEventDestroy(gev_fork);
        if (gev_lead) cudaEventDestroy(gev_lead);
    }

    // outside a generation (setup, set_population): z MIN over the shards
    void exchange_z_eager() {
        sync_all();
        for (size_t k = 0; k < members.size(); ++k) {
            on(k);
            z_peers_kernel<<<1, 32, 0, members[k]->s>>>(members[k]->st.p, peers[k]);
            CK(cudaGetLastError());
        }
        sync_all();
    }

    // one generation over every shard; prof (6 events on shard 0's stream)
    // brackets shard 0's phases for profile()
    void group_generation(bool clock, cudaEvent_t* prof) {
        const size_t K = members.size();
        gmpea_engine& L = *members[0];
        on(0);
        if (prof) CK(cudaEventRecord(prof[0], L.s));
        CK(cudaEventRecord(gev_fork, L.s));
        for (size_t k = 1; k < K; ++k) {
            on(k);
            CK(cudaStreamWaitEvent(members[k]->s, gev_fork, 0));
        }
        if (clock) {
            on(0);
            L.start_loop_clock();
        }
        for (size_t k = 0; k < K; ++k) {  // vary_eval (+ local ideal point)
            on(k);
            members[k]->enqueue_phase1();
            CK(cudaEventRecord(gev[0][k], members[k]->s));
        }
        if (prof) {
            on(0);
            CK(cudaEventRecord(prof[1], L.s));
        }
        for (size_t k = 0; k < K; ++k) {  // ideal point over the shards (peer loads)
            on(k);
            for (size_t j = 0; j < K; ++j)
                if (j != k) CK(cudaStreamWaitEvent(members[k]->s, gev[0][j], 0));
            z_peers_kernel<<<1, 32, 0, members[k]->s>>>(members[k]->st.p, peers[k]);
            if (prof && k == 0) CK(cudaEventRecord(prof[2], L.s));
            members[k]->launch_op1();
            if (prof && k == 0) CK(cudaEventRecord(prof[3], L.s));
            members[k]->launch_select();  // + end_gen (shard 0 keeps the clock)
            if (prof && k == 0) CK(cudaEventRecord(prof[4], L.s));
            CK(cudaEventRecord(gev[1][k], members[k]->s));
        }
        int fin = 1;
        if (time_mode) {  // every shard adopts shard 0's clock and deadline decision
            on(0);
            lead_pack_kernel<<<1, 1, 0, L.s>>>(L.st.p, L.lead.p);
            CK(cudaEventRecord(gev_lead, L.s));
            for (size_t k = 0; k < K; ++k) {
                on(k);
                if (k) CK(cudaStreamWaitEvent(members[k]->s, gev_lead, 0));
                follow_kernel<<<1, 1, 0, members[k]->s>>>(members[k]->st.p, L.lead.p, members[k]->lead_flag_dev);
                members[k]->launch_restore();
                CK(cudaEventRecord(gev[2][k], members[k]->s));
            }
            fin = 2;
        }
        for (size_t k = 0; k < K; ++k) {  // boundary parent rows from the neighbours
            gmpea_engine& E = *members[k];
            on(k);
            for (const Halo& h : E.halos) {
                gmpea_engine& P = *members[h.peer];
                CK(cudaStreamWaitEvent(E.s, gev[fin][h.peer], 0));
                HaloCopy hc;
                hc.n4 = (h.recv1 - h.recv0) * geo.rs4;
                for (int q = 0; q < 2; ++q) {
                    hc.dst[q] = E.pop[q].X.p + (h.recv0 - E.e0) * geo.rs4;
                    hc.src[q] = P.pop[q].X.p + (h.recv0 - P.e0) * geo.rs4;
                }
                halo_pull_kernel<<<(int)std::min<long long>(blocks_for(hc.n4, 256), 4 * 148), 256, 0, E.s>>>(hc);
            }
            CK(cudaEventRecord(gev[3][k], E.s));
        }
        on(0);
        for (size_t k = 1; k < K; ++k) CK(cudaStreamWaitEvent(L.s, gev[3][k], 0));
        if (prof) CK(cudaEventRecord(prof[5], L.s));
        CK(cudaGetLastError());
    }

    cudaGraphExec_t capture_group(bool clock) {
        gmpea_engine& L = *members[0];
        on(0);
        cudaGraph_t g;
        cudaGraphExec_t x;
        CK(cudaStreamBeginCapture(L.s, cudaStreamCaptureModeThreadLocal));
        group_generation(clock, nullptr);
        CK(cudaStreamEndCapture(L.s, &g));
        CK(cudaGraphInstantiate(&x, g, 0));
        CK(cudaGraphDestroy(g));
        return x;
    }

    long long group_step(long long k) {
        gmpea_engine& L = *members[0];
        on(0);
        long long done = 0;
        while (done < k) {
            long long room = L.rec_cap - 2 - (gens_enqueued - L.rec_base);
            if (room <= 0) {  // drain every shard's record window together
                sync_all();
                for (size_t j = 0; j < members.size(); ++j) {
                    on(j);
                    members[j]->drain_records();
                }
                on(0);
                room = L.rec_cap - 2 - (gens_enqueued - L.rec_base);
                if (room <= 0) break;
            }
            const long long part = std::min(k - done, room);
            CK(cudaGraphLaunch(done == 0 ? graph_first : graph, L.s));
            for (long long i = 1; i < part; ++i) CK(cudaGraphLaunch(graph, L.s));
            gens_enqueued += part;
            done += part;
        }
        return done;
    }

    void group_set_population(int which, const double* X) {
        if (gens_enqueued) throw std::invalid_argument("set_population: the run has started");
        sync_all();
        for (size_t k = 0; k < members.size(); ++k) {
            on(k);
            members[k]->set_population(which, X);
        }
        exchange_z_eager();
        on(0);
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
        // P1..P10 are the reference's scenarios (wta.cpp:23-49); larger num
        // extend its size formula and seeded tables (synthetic instances)
        if (num < 1 || num > kWtaMaxScenario)
            throw std::invalid_argument("unknown WTA scenario: P" + std::to_string(num));
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
        launch_vary(vary_kernel_for(p->dev, MODE_EVAL, 0), ep, 1, s);
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
        if (m < 2 || m > kMaxLatM) throw std::invalid_argument("reference_vectors: m must be 2 to 16");
        require_device();
        DevBuf<double> w((size_t)n * m);
        DevBuf<float4> u(n);
        if (m <= 3)
            lattice_kernel<<<blocks_for(n, 256), 256>>>((int)n, m, lattice_H(m, n), w.p, u.p);
        else
            lattice_m_kernel<<<blocks_for(n, 256), 256>>>((int)n, m, lattice_H(m, n), w.p);
        CK(cudaGetLastError());
        CK(cudaMemcpy(W, w.p, (size_t)n * m * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

static void knn_api(const double* Wh, int64_t n, int32_t m, int32_t t1, int32_t t2, uint32_t* B1,
                    uint32_t* B2, bool lattice) {
    if (n <= 0) throw std::invalid_argument("build_neighborhoods: empty population");
    if (m < 2 || m > kMaxLatM) throw std::invalid_argument("build_neighborhoods: m must be 2 to 16");
    if (t1 > n || t2 > n) throw std::invalid_argument("build_neighborhoods: neighborhood exceeds population");
    require_device();
    cudaStream_t s = 0;
    DevBuf<double> w((size_t)n * m);
    DevBuf<float4> u(n);
    long long H = lattice_H(m, n);
    if (lattice && m <= 3)
        lattice_kernel<<<blocks_for(n, 256), 256>>>((int)n, m, H, w.p, u.p);
    else if (lattice)
        lattice_m_kernel<<<blocks_for(n, 256), 256>>>((int)n, m, H, w.p);
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
        PmGaps gaps;
        fill_op_params(vp, prm, d, gaps);
        vp.eval = 0;
        vp.fixed_gen = (int)gen;
        vp.st = st.p;
        vp.bad_rows[0] = bad.p;
        vp.bad_cap = 0;  // reproduce itself never throws on bounds
        launch_vary(vary_kernel_for(p->dev, MODE_VARY, op), vp, 1, s);
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
    return gmpea_environmental_selection_ex(n, d, m, nc, pop1, pop2, off1, off2, W, z, theta, GMPEA_AGG_PBI, B1, t1,
                                            B2, t2, out1, out2, winner1, winner2);
}

int gmpea_environmental_selection_ex(int64_t n, int32_t d, int32_t m, int32_t nc,
                                     const gmpea_population_view* pop1, const gmpea_population_view* pop2,
                                     const gmpea_population_view* off1, const gmpea_population_view* off2,
                                     const double* W, const double* z, double theta, int32_t aggregation,
                                     const uint32_t* B1, int32_t t1, const uint32_t* B2, int32_t t2,
                                     gmpea_population_out* out1, gmpea_population_out* out2, int32_t* winner1,
                                     int32_t* winner2) {
    return guarded([&] {
        check_aggregation(aggregation);
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
        launch_op1_kernel(blocks_for(n, 256), aggregation, o1, 0);
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
        launch_select_kernel((int)n, pack, aggregation, sp, 0);
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

int gmpea_engine_create_multi(const gmpea_problem* p, const gmpea_run_config* cfg, const int32_t* devices,
                              int32_t ndev, gmpea_engine** out) {
    return guarded([&] {
        if (!p || !cfg || !out) throw std::invalid_argument("gmpea_engine_create_multi: null argument");
        require_device();
        int saved = 0;
        CK(cudaGetDevice(&saved));
        auto e = std::make_unique<gmpea_engine>();
        e->setup_group(p, *cfg, devices, ndev);
        *out = e.release();
        CK(cudaSetDevice(saved));
    });
}

int gmpea_nccl_unique_id(void* id128) {
    return guarded([&] {
        if (!id128) throw std::invalid_argument("gmpea_nccl_unique_id: null argument");
        ncclUniqueId id;
        NK(Nccl::get().GetUniqueId(&id));
        std::memcpy(id128, &id, sizeof(id));
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

int gmpea_engine_get_offspring(gmpea_engine* e, int32_t which, double* X, double* F, double* C, double* cv) {
    return guarded([&] { e->get_population(which, X, F, C, cv, true); });
}

int gmpea_engine_ideal(gmpea_engine* e, double* z) {
    return guarded([&] {
        if (e->is_group()) {
            e->sync_all();
            e->on(0);
        }
        DevState h = (e->is_group() ? *e->members[0] : *e).read_state();
        for (int k = 0; k < e->m; ++k) z[k] = ordered_to_float(h.zbits[k]);
    });
}

int gmpea_engine_neighborhoods(gmpea_engine* e, uint32_t* B1, uint32_t* B2) {
    return guarded([&] {
        auto one = [&](gmpea_engine* x, uint32_t* b1, uint32_t* b2) {
            const long long o0 = x->own0 - x->e0, on = x->own1 - x->own0;
            uint32_t* outs[2] = {b1, b2};
            for (int q = 0; q < 2; ++q) {
                if (!outs[q]) continue;
                const int t = q ? x->t2 : x->t1;
                CK(cudaMemcpy(outs[q], x->B[q].p + o0 * t, (size_t)on * t * sizeof(int), cudaMemcpyDeviceToHost));
                for (long long k = 0; k < on * t; ++k) outs[q][k] += (uint32_t)x->e0;  // global slots
            }
        };
        if (!e->is_group()) return one(e, B1, B2);
        for (size_t k = 0; k < e->members.size(); ++k) {  // the shards' owned rows in slot order
            e->on(k);
            gmpea_engine* x = e->members[k].get();
            one(x, B1 ? B1 + x->own0 * e->t1 : nullptr, B2 ? B2 + x->own0 * e->t2 : nullptr);
        }
        e->on(0);
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
        if (e->is_group()) throw std::invalid_argument("device_buffers: a multi-device handle has one set per shard");
        o->ideal_bits = e->st.p->zbits;
        for (int q = 0; q < 2; ++q) {
            o->rows[q] = e->pop[q].X.p;
            o->keys[q] = e->pop[q].Fcv.p;
        }
        o->row_bytes = (int64_t)e->geo.rs4 * 16;
    });
}

}  // extern "C"
