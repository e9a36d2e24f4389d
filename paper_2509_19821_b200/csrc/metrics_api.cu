// Metrics and reference fronts on the device (metrics.hpp:15-57,
// fronts.cpp:54-103): metric_front, IGD, HV2/HV3, pf_reference, and the
// per-generation IGD hook of the runs (igd_dev).
#include "host.cuh"
#include "fronts.cuh"
#include "metrics.cuh"

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
    if (m > 3) {  // any m: the reference's pairwise form; kept rows in row order
        thrust::device_vector<unsigned char> keep(k);
        nd_any_kernel<<<blocks_for(k, 128), 128>>>(dF, thrust::raw_pointer_cast(cand.data()), k, m, dedup,
                                                   thrust::raw_pointer_cast(keep.data()));
        CK(cudaGetLastError());
        kept.resize(k);
        auto end = thrust::copy_if(thrust::device, cand.begin(), cand.end(), keep.begin(), kept.begin(), NonZero{});
        kept.resize(end - kept.begin());
        return kept;
    }
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

// igd(metric_front(pop), ref) on device arrays (metrics.cpp:42-60, 155-175);
// +inf for an empty front, as the reference's IGD hook records it
}  // namespace

namespace gmpea_b200 {
namespace host {
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

}  // namespace host
}  // namespace gmpea_b200

extern "C" {

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
        if (m < 2 || m > kMaxObj) throw std::invalid_argument("metric_front: m must be 2 to 16");
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
        if (m < 1 || m > kMaxObj) throw std::invalid_argument("igd: objective count mismatch");
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
        if (m < 2 || m > kMaxObj) throw std::invalid_argument("hypervolume: m must be 2 to 16");
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
        if (m > 3) {  // hv_mc (metrics.cpp:95-121)
            std::vector<long long> keep(cnt);
            thrust::copy(xy.begin(), xy.end(), keep.begin());
            std::vector<double> lo(m, std::numeric_limits<double>::infinity());
            for (long long i : keep)
                for (int c = 0; c < m; ++c) lo[c] = std::min(lo[c], P[i * m + c]);
            double box = 1.0;
            for (int c = 0; c < m; ++c) box *= ref[c] - lo[c];
            if (box <= 0.0) return;
            // the reference's sample stream: Rng(0x48563D) = mt19937_64, uniform(lo, hi)
            std::mt19937_64 e(0x48563D);
            const long long samples = 1000000;
            std::vector<double> X((size_t)samples * m);
            for (long long s2 = 0; s2 < samples; ++s2)
                for (int c = 0; c < m; ++c)
                    X[(size_t)s2 * m + c] = lo[c] + (ref[c] - lo[c]) * ((double)(e() >> 11) * 0x1.0p-53);
            thrust::device_vector<double> dX(X.begin(), X.end());
            thrust::device_vector<unsigned long long> hits(1, 0ull);
            hv_mc_kernel<<<blocks_for(samples, 256), 256>>>(pP, thrust::raw_pointer_cast(xy.data()), cnt, m,
                                                            thrust::raw_pointer_cast(dX.data()), samples,
                                                            thrust::raw_pointer_cast(hits.data()));
            CK(cudaGetLastError());
            *out = box * (double)(unsigned long long)hits[0] / (double)samples;
            return;
        }
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

}  // extern "C"
