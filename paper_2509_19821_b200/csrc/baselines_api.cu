// Comparison-algorithm operators and runs on the device (baselines.hpp,
// baselines.cpp:22-190, 320-459): nondominated sort, crowding, SPEA2
// fitness / selection, run_cnsga2 / run_ccmo.
#include <thrust/copy.h>
#include <thrust/count.h>
#include <thrust/device_vector.h>
#include <thrust/execution_policy.h>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>

#include "host.cuh"
#include "baselines.cuh"

// (the gmpea_* entry points take C linkage from include/gmpea_b200.h)
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
struct FeasibleRow {
    const double* cv;
    __host__ __device__ bool operator()(long long i) const { return cv[i] == 0.0; }
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
                                   thrust::counting_iterator<long long>(n), sub.begin(), FeasibleRow{dcv});
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
    PmGaps gaps;
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
        fill_op_params(vp, c.params, d, gaps);
        vp.eval = 1;
        vp.update_z = 0;
        vp.st = st.p;
        vp.bad_cap = kMaxBadRows;
        vp.tour = algo == 0 ? 1 : 2;
        vp.un = make_uidx((unsigned long long)n);
        for (int q = 0; q < npop; ++q) vp.bad_rows[q] = bad[q].p;
        init_k = vary_kernel_for(p->dev, MODE_INIT, 0);
        vary_k = vary_kernel_for(p->dev, MODE_VARY, OP_SBX, true);
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
