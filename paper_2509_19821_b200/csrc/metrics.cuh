// On-device quality indicators (proj/src/metrics.cpp):
//   metric_front  feasible (cv == 0) & deduplicated (first index kept) &
//                 mutually nondominated rows (:155-175).  After a lexicographic
//                 sort (f, index) every dominator of a row lies before its
//                 group of equal rows, so the filter is a prefix query: a
//                 running minimum of f2 (m = 2) or a tiled prefix scan for a
//                 (f2, f3) dominator (m = 3).
//   igd           mean over reference points of the min Euclidean distance
//                 (:15-37).  Squared distances are formed in coordinate order
//                 without contraction and min-reduced (order-free), and the
//                 final sum runs in reference order, so the result is
//                 bit-identical to the reference's.
//   hypervolume   relevant set (:42-61) + 2D sweep (:63-74) / 3D slicing
//                 (:76-93), with the per-slab 2D areas computed in parallel and
//                 the outer sums in the reference's order.
#pragma once
#include <thrust/copy.h>
#include <thrust/scan.h>
#include <thrust/scatter.h>
#include <thrust/functional.h>
#include <thrust/device_vector.h>
#include <thrust/execution_policy.h>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>

#include "common.cuh"

namespace gmpea_b200 {

struct LexLess {
    const double* F;
    int m;
    __host__ __device__ bool operator()(long long a, long long b) const {
        for (int c = 0; c < m; ++c) {
            double x = F[a * m + c], y = F[b * m + c];
            if (x < y) return true;
            if (x > y) return false;
        }
        return a < b;
    }
};

struct ZLess {
    const double* P;
    __host__ __device__ bool operator()(long long a, long long b) const {
        double x = P[a * 3 + 2], y = P[b * 3 + 2];
        return x < y || (x == y && a < b);
    }
};

struct NonZero {
    __host__ __device__ bool operator()(unsigned char v) const { return v != 0; }
};

struct IsFeasible {
    const double* cv;
    __host__ __device__ bool operator()(long long i) const { return cv[i] == 0.0; }
};

struct InsideBox {
    const double* P;
    const double* ref;
    int m;
    __host__ __device__ bool operator()(long long i) const {
        for (int c = 0; c < m; ++c)
            if (!(P[i * m + c] < ref[c])) return false;
        return true;
    }
};

__device__ __forceinline__ bool same_row(const double* F, long long a, long long b, int m) {
    for (int c = 0; c < m; ++c)
        if (F[a * m + c] != F[b * m + c]) return false;
    return true;
}

// group start position for each sorted position (equal rows form a group)
__global__ void group_start_kernel(const double* F, const long long* order, long long k, int m, long long* gs) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= k) return;
    long long q = p;
    while (q > 0 && same_row(F, order[q - 1], order[p], m)) --q;
    gs[p] = q;
}

// m = 2: keep iff first of group and min f2 over earlier groups > own f2
__global__ void nd2_kernel(const double* F, const long long* order, const long long* gs,
                           const double* prefmin, long long k, unsigned char* keep) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= k) return;
    const long long a = order[p];
    const bool first = gs[p] == p;
    const double before = p == 0 ? 1.0 / 0.0 : prefmin[p - 1];
    keep[p] = first && (before > F[a * 2 + 1]);
}

__global__ void gather_col_kernel(const double* F, const long long* order, long long k, int m, int c, double* out) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= k) return;
    out[p] = F[order[p] * m + c];
}

// m = 3: does any row before the group weakly dominate in (f2, f3)?
__global__ void nd3_kernel(const double* F, const long long* order, const long long* gs, long long k,
                           unsigned char* keep, int dedup = 1) {
    __shared__ double s2[256], s3[256];
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = p < k;
    long long lim = 0;
    double a2 = 0.0, a3 = 0.0;
    bool alive = false;
    if (act) {
        const long long a = order[p];
        a2 = F[a * 3 + 1];
        a3 = F[a * 3 + 2];
        lim = gs[p];
        alive = !dedup || lim == p;  // dedup: duplicates of an earlier row are dropped
    }
    // block-wide prefix length: the largest group start in the block
    __shared__ long long blim;
    if (threadIdx.x == 0) blim = 0;
    __syncthreads();
    if (act) atomicMax((unsigned long long*)&blim, (unsigned long long)lim);
    __syncthreads();
    const long long total = blim;
    for (long long base = 0; base < total; base += blockDim.x) {
        __syncthreads();
        long long q = base + threadIdx.x;
        if (q < total) {
            long long b = order[q];
            s2[threadIdx.x] = F[b * 3 + 1];
            s3[threadIdx.x] = F[b * 3 + 2];
        }
        __syncthreads();
        if (alive) {
            const long long n_here = min((long long)blockDim.x, lim - base);
            for (long long t = 0; t < n_here; ++t)
                if (s2[t] <= a2 && s3[t] <= a3) {
                    alive = false;
                    break;
                }
        }
        if (!__syncthreads_or(alive)) break;
    }
    if (act) keep[p] = alive;
}

// IGD partial: best squared distance of reference point r over a chunk of A
// objectives the metrics take on the device (any m up to this)
constexpr int kMaxObj = 16;

// nondominated (+ deduplicated, the earlier of equal rows kept) subset of the
// candidate rows, any m, O(k^2): metrics.cpp:155-175 (metric_front) and
// :42-61 (hv_relevant) as the reference writes them; cand in row order
__global__ void nd_any_kernel(const double* F, const long long* cand, long long k, int m, int dedup,
                              unsigned char* keep) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= k) return;
    const long long i = cand[p];
    bool ok = true;
    for (long long q = 0; q < k && ok; ++q) {
        if (q == p) continue;
        const long long j = cand[q];
        bool le = true, lt = false, eq = true;
        for (int c = 0; c < m; ++c) {
            const double a = F[j * m + c], b = F[i * m + c];
            if (a > b) le = false;
            if (a < b) lt = true;
            if (a != b) eq = false;
        }
        if (le && lt) ok = false;  // pareto_dominates(row j, row i)
        if (dedup && eq && q < p) ok = false;
    }
    keep[p] = ok ? 1 : 0;
}

// hv_mc (metrics.cpp:95-121): the number of samples (host-drawn from the
// reference's fixed-seed stream, s-major, m coordinates each) dominated by
// some relevant point; the count is an integer, so the estimate is exact
__global__ void hv_mc_kernel(const double* P, const long long* keep, long long nk, int m, const double* X,
                             long long samples, unsigned long long* hits) {
    __shared__ unsigned cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < samples) {
        const double* x = X + s * m;
        for (long long t = 0; t < nk; ++t) {
            const double* pi = P + keep[t] * m;
            bool dom = true;
            for (int c = 0; c < m && dom; ++c)
                if (pi[c] > x[c]) dom = false;
            if (dom) {
                atomicAdd(&cnt, 1u);
                break;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && cnt) atomicAdd(hits, (unsigned long long)cnt);
}

__global__ void igd_min_kernel(const double* A, long long na, const double* Rf, long long nr, int m,
                               unsigned long long* best) {
    const long long r = blockIdx.y;
    double rr[kMaxObj];
    for (int c = 0; c < m; ++c) rr[c] = Rf[r * m + c];
    double b = 1.0 / 0.0;
    for (long long a = (long long)blockIdx.x * blockDim.x + threadIdx.x; a < na;
         a += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < m; ++c) {
            double d = __dsub_rn(A[a * m + c], rr[c]);
            s = __dadd_rn(s, __dmul_rn(d, d));
        }
        b = fmin(b, s);
    }
    for (int o = 16; o > 0; o >>= 1) b = fmin(b, __shfl_xor_sync(0xffffffffu, b, o));
    if ((threadIdx.x & 31) == 0) atomicMin(&best[r], (unsigned long long)__double_as_longlong(b));
}

__global__ void igd_sum_kernel(const unsigned long long* best, long long nr, double* out) {
    double total = 0.0;
    for (long long r = 0; r < nr; ++r) total += sqrt(__longlong_as_double((long long)best[r]));
    *out = total / (double)nr;
}

// 2D hypervolume of the points whose z-rank <= k, swept in (x, y) order:
// xyorder lists all relevant points sorted by (x, y); zrank[i] = position of
// point i in z order.  slab[k] = hv2 of the slab (metrics.cpp:63-74).
__global__ void hv_slab_kernel(const double* P, const long long* xyorder, const long long* zrank, long long cnt,
                               int m, long long kmax_all, const double* ref, double* slab) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kmax_all) return;
    const long long zk = m == 2 ? cnt : k;
    double vol = 0.0, prev = ref[1];
    for (long long t = 0; t < cnt; ++t) {
        const long long i = xyorder[t];
        if (m == 3 && zrank[i] > zk) continue;
        const double x = P[i * m], y = P[i * m + 1];
        if (y < prev) {
            vol = __dadd_rn(vol, __dmul_rn(ref[0] - x, prev - y));
            prev = y;
        }
    }
    slab[k] = vol;
}

// hv3 outer sum (metrics.cpp:82-92), sequential in z order
__global__ void hv3_sum_kernel(const double* P, const long long* zorder, long long cnt, const double* ref,
                               const double* slab, double* out) {
    double vol = 0.0;
    for (long long k = 0; k < cnt; ++k) {
        double z0 = P[zorder[k] * 3 + 2];
        double z1 = k + 1 < cnt ? P[zorder[k + 1] * 3 + 2] : ref[2];
        if (z1 <= z0) continue;
        vol = __dadd_rn(vol, __dmul_rn(z1 - z0, slab[k]));
    }
    *out = vol;
}

}  // namespace gmpea_b200
