// Comparison-algorithm operators on device (proj/include/gmpea/baselines.hpp,
// proj/src/baselines.cpp:22-190): constrained nondominated sorting, crowding
// distance, SPEA2 fitness and SPEA2 environmental selection.  Inputs are the
// reference's fp64 objective rows and cv; every result (ranks, distances,
// fitness, kept indices) is the reference's bit for bit, with the reference's
// serial algorithms replaced by parallel ones:
//   * nondominated_sort: front peeling with dominator counts (each dominating
//     pair is visited once over all fronts).  Under CDP the infeasible rows
//     need no pair work: every feasible row beats them and among themselves
//     they are ordered by cv alone, so their rank is R_feasible + the dense
//     rank of their cv.
//   * spea2_fitness: strength / raw sums over tiled pair sweeps (integer-valued
//     doubles, exact in any order) and the k-th nearest distance by a per-row
//     radix select over the fp64 bit patterns (non-negative doubles order like
//     their bits).
//   * spea2_select truncation: one persistent block keeps, per alive row, its
//     two smallest distances to the other alive rows; the victim is the row
//     with the lexicographically smallest sorted distance profile, decided on
//     those two levels and, in the rare remaining ties, level by level with a
//     block radix select — the reference's first-minimum-in-index-order rule.
#pragma once
#include <thrust/gather.h>
#include <thrust/iterator/permutation_iterator.h>
#include <thrust/fill.h>
#include <thrust/unique.h>

#include "common.cuh"

namespace gmpea_b200 {

struct DomRel {
    const double* F;
    const double* cv;
    int m;
    int cdp;
    // pareto_dominates (scalarize.cpp:51-60)
    __device__ __forceinline__ bool pareto(long long a, long long b) const {
        bool strict = false;
        for (int c = 0; c < m; ++c) {
            const double x = F[a * m + c], y = F[b * m + c];
            if (x > y) return false;
            if (x < y) strict = true;
        }
        return strict;
    }
    // cdp_better (scalarize.cpp:62-70) or pareto_dominates
    __device__ __forceinline__ bool better(long long a, long long b) const {
        if (!cdp) return pareto(a, b);
        const double ca = cv[a], cb = cv[b];
        if (ca == 0.0 && cb > 0.0) return true;
        if (ca == 0.0 && cb == 0.0) return pareto(a, b);
        if (ca > 0.0 && cb > 0.0) return ca < cb;
        return false;
    }
};

// ---- nondominated sort (Pareto) on a subset of rows: dominator counts
__global__ void nds_count_kernel(DomRel R, const long long* sub, long long ns, int* cnt) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ns) return;
    const long long i = sub[t];
    int c = 0;
    for (long long u = 0; u < ns; ++u)
        if (R.pareto(sub[u], i)) ++c;
    cnt[t] = c;
}

// rows (subset positions) with no dominator start front 0
__global__ void nds_front0_kernel(const int* cnt, long long ns, long long* front, int* fsize) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ns || cnt[t] != 0) return;
    front[atomicAdd(fsize, 1)] = t;
}

// peel one front: every (front row a, subset row j) pair with a dominating j
// removes one dominator of j; j joins the next front when it has none left
__global__ void nds_peel_kernel(DomRel R, const long long* sub, long long ns, const long long* front,
                                long long fsize, int* cnt, long long* next, int* nsize) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= fsize * ns) return;
    const long long a = front[p / ns], j = p % ns;
    if (R.pareto(sub[a], sub[j]) && atomicSub(&cnt[j], 1) == 1) next[atomicAdd(nsize, 1)] = j;
}

__global__ void nds_set_rank_kernel(const long long* sub, const long long* front, long long fsize, long long r,
                                    long long* rank) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < fsize) rank[sub[front[t]]] = r;
}

// CDP: infeasible rows (cv > 0) take R_f + the dense rank of their cv
__global__ void nds_infeasible_rank_kernel(const double* cv, long long n, const double* ucv, long long nu,
                                           long long rf, long long* rank) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !(cv[i] > 0.0)) return;
    long long lo = 0, hi = nu;  // first unique value >= cv[i]
    while (lo < hi) {
        const long long mid = (lo + hi) / 2;
        if (ucv[mid] < cv[i])
            lo = mid + 1;
        else
            hi = mid;
    }
    rank[i] = rf + lo;
}

// ---- crowding distance (baselines.cpp:56-91), one objective per launch
__global__ void crowd_axis_kernel(const double* F, int m, int c, const long long* front, const long long* order,
                                  long long k, double* dist) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= k) return;
    const double lo = F[front[order[0]] * m + c], hi = F[front[order[k - 1]] * m + c];
    const double inf = 1.0 / 0.0;
    if (q == 0 || q == k - 1) {
        dist[order[q]] = inf;
        return;
    }
    if (hi == lo) return;
    dist[order[q]] += (F[front[order[q + 1]] * m + c] - F[front[order[q - 1]] * m + c]) / (hi - lo);
}

// ---- SPEA2 fitness (baselines.cpp:93-127)
__global__ void spea2_strength_kernel(DomRel R, long long n, double* strength) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long s = 0;
    for (long long j = 0; j < n; ++j)
        if (j != i && R.better(i, j)) ++s;
    strength[i] = (double)s;
}

__global__ void spea2_raw_kernel(DomRel R, long long n, const double* strength, double* raw) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;  // integer-valued terms: exact in any order
    for (long long j = 0; j < n; ++j)
        if (j != i && R.better(j, i)) s += strength[j];
    raw[i] = s;
}

// squared distance with the reference's rounding: separate multiply and add
// (the reference builds with -ffp-contract=off, CMakeLists.txt:15-16)
__device__ __forceinline__ double sq_dist(const double* F, int m, long long a, long long b) {
    double s = 0.0;
    for (int c = 0; c < m; ++c) {
        const double d = F[a * m + c] - F[b * m + c];
        s = __dadd_rn(s, __dmul_rn(d, d));
    }
    return s;
}

// kk-th smallest (0-based) of { sq_dist(i, j) : j in cand, j != i, alive } by an
// 8-pass byte radix select over the bit patterns, one block; returns the value
// in every thread.  cand == nullptr: all rows 0..n-1; alive == nullptr: all.
__device__ double block_select_dist(const double* F, int m, long long i, const long long* cand, long long nc,
                                    const unsigned char* alive, long long kk) {
    __shared__ unsigned hist[256];
    __shared__ unsigned long long s_prefix;
    __shared__ long long s_kk;
    if (threadIdx.x == 0) {
        s_prefix = 0ull;
        s_kk = kk;
    }
    __syncthreads();
    for (int pass = 7; pass >= 0; --pass) {
        for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0u;
        __syncthreads();
        const unsigned long long prefix = s_prefix;
        const int shift = pass * 8;
        const unsigned long long hmask = pass == 7 ? 0ull : (~0ull << (shift + 8));
        for (long long t = threadIdx.x; t < nc; t += blockDim.x) {
            const long long j = cand ? cand[t] : t;
            if (j == i || (alive && !alive[j])) continue;
            const unsigned long long key = (unsigned long long)__double_as_longlong(sq_dist(F, m, i, j));
            if ((key & hmask) != prefix) continue;
            atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long want = s_kk;
            int b = 0;
            for (; b < 256; ++b) {
                if (want < (long long)hist[b]) break;
                want -= hist[b];
            }
            s_prefix = prefix | ((unsigned long long)b << shift);
            s_kk = want;
        }
        __syncthreads();
    }
    const double v = __longlong_as_double((long long)s_prefix);
    __syncthreads();
    return v;
}

__global__ void spea2_sigma_kernel(const double* F, int m, long long n, long long kk, const double* raw,
                                   double* fit) {
    const long long i = blockIdx.x;
    double sigma = 0.0;
    if (n > 1) sigma = sqrt(block_select_dist(F, m, i, nullptr, n, nullptr, kk));
    if (threadIdx.x == 0) fit[i] = raw[i] + 1.0 / (sigma + 2.0);
}

// ---- SPEA2 truncation (baselines.cpp:149-184)
// two smallest distances (with multiplicity) from row i to the other alive rows
__device__ __forceinline__ void nn2_of(const double* F, int m, long long i, const long long* keep, long long nk,
                                       const unsigned char* alive, long long start, long long step, double& d1,
                                       long long& j1, double& d2, long long& j2) {
    d1 = d2 = 1.0 / 0.0;
    j1 = j2 = -1;
    for (long long t = start; t < nk; t += step) {
        const long long j = keep[t];
        if (j == i || !alive[j]) continue;
        const double d = sq_dist(F, m, i, j);
        if (d < d1 || (d == d1 && j < j1)) {
            d2 = d1;
            j2 = j1;
            d1 = d;
            j1 = j;
        } else if (d < d2 || (d == d2 && j < j2)) {
            d2 = d;
            j2 = j;
        }
    }
}

__device__ __forceinline__ void nn2_merge(double& d1, long long& j1, double& d2, long long& j2, double e1,
                                          long long k1, double e2, long long k2) {
    const double a[4] = {d1, d2, e1, e2};
    const long long b[4] = {j1, j2, k1, k2};
    double x1 = 1.0 / 0.0, x2 = 1.0 / 0.0;
    long long y1 = -1, y2 = -1;
    for (int q = 0; q < 4; ++q) {
        if (b[q] < 0) continue;
        if (b[q] == y1) continue;  // the same neighbour seen twice (never across disjoint scans)
        if (a[q] < x1 || (a[q] == x1 && (y1 < 0 || b[q] < y1))) {
            x2 = x1;
            y2 = y1;
            x1 = a[q];
            y1 = b[q];
        } else if (a[q] < x2 || (a[q] == x2 && (y2 < 0 || b[q] < y2))) {
            x2 = a[q];
            y2 = b[q];
        }
    }
    d1 = x1;
    j1 = y1;
    d2 = x2;
    j2 = y2;
}

// one thread per kept row: its two nearest alive neighbours
__global__ void trunc_init_kernel(const double* F, int m, const long long* keep, long long nk,
                                  const unsigned char* alive, double* n1, long long* i1, double* n2, long long* i2) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nk) return;
    double d1, d2;
    long long j1, j2;
    nn2_of(F, m, keep[t], keep, nk, alive, 0, 1, d1, j1, d2, j2);
    n1[t] = d1;
    i1[t] = j1;
    n2[t] = d2;
    i2[t] = j2;
}

// block-wide two-nearest scan of row i over the alive kept rows; the result
// is valid in thread 0
__device__ void block_nn2(const double* F, int m, long long i, const long long* keep, long long nk,
                          const unsigned char* alive, double& d1, long long& j1, double& d2, long long& j2) {
    __shared__ double r1[32], r2[32];
    __shared__ long long q1[32], q2[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    nn2_of(F, m, i, keep, nk, alive, threadIdx.x, blockDim.x, d1, j1, d2, j2);
    for (int o = 16; o; o >>= 1) {
        const double e1 = __shfl_xor_sync(0xffffffffu, d1, o), e2 = __shfl_xor_sync(0xffffffffu, d2, o);
        const long long k1 = __shfl_xor_sync(0xffffffffu, j1, o), k2 = __shfl_xor_sync(0xffffffffu, j2, o);
        nn2_merge(d1, j1, d2, j2, e1, k1, e2, k2);
    }
    if (lane == 0) {
        r1[wid] = d1;
        q1[wid] = j1;
        r2[wid] = d2;
        q2[wid] = j2;
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int w = 1; w < nw; ++w) nn2_merge(d1, j1, d2, j2, r1[w], q1[w], r2[w], q2[w]);
    __syncthreads();
}

// The serial truncation loop in one block.  Positions t index `keep` (kept
// rows in ascending row order); n1/n2 are the two smallest distances of the
// row at t to the other alive rows (i1/i2 the neighbours), lv is scratch.
__global__ void __launch_bounds__(1024) trunc_loop_kernel(const double* F, int m, const long long* keep, long long nk,
                                                         long long capacity, unsigned char* alive, double* n1,
                                                         long long* i1, double* n2, long long* i2, double* lv,
                                                         long long* cand) {
    __shared__ double s_b1, s_b2, red[32];
    __shared__ unsigned long long s_count;
    __shared__ long long s_l;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    long long alive_n = 0;
    for (long long t = 0; t < nk; ++t) alive_n += alive[keep[t]] ? 1 : 0;
    auto block_min = [&](double v) {
        for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) red[wid] = v;
        __syncthreads();
        double b = red[0];
        for (int w = 1; w < nw; ++w) b = fmin(b, red[w]);
        __syncthreads();
        return b;
    };
    while (alive_n > capacity) {
        // levels 0 and 1 of the sorted distance profile
        double b = 1.0 / 0.0;
        for (long long t = tid; t < nk; t += blockDim.x)
            if (alive[keep[t]]) b = fmin(b, n1[t]);
        b = block_min(b);
        if (tid == 0) s_b1 = b;
        __syncthreads();
        b = 1.0 / 0.0;
        for (long long t = tid; t < nk; t += blockDim.x)
            if (alive[keep[t]] && n1[t] == s_b1) b = fmin(b, n2[t]);
        b = block_min(b);
        if (tid == 0) {
            s_b2 = b;
            s_count = 0ull;
        }
        __syncthreads();
        for (long long t = tid; t < nk; t += blockDim.x)
            if (alive[keep[t]] && n1[t] == s_b1 && n2[t] == s_b2) cand[atomicAdd(&s_count, 1ull)] = t;
        __syncthreads();
        if (tid == 0) {  // candidates in row order (few)
            const long long c = (long long)s_count;
            for (long long a = 1; a < c; ++a) {
                const long long v = cand[a];
                long long q = a - 1;
                while (q >= 0 && cand[q] > v) {
                    cand[q + 1] = cand[q];
                    --q;
                }
                cand[q + 1] = v;
            }
            s_l = 2;
        }
        __syncthreads();
        // deeper levels only while candidates still tie (rare)
        while (s_count > 1ull && s_l < alive_n - 1) {
            const long long l = s_l, c = (long long)s_count;
            for (long long a = 0; a < c; ++a) {
                const double v = block_select_dist(F, m, keep[cand[a]], keep, nk, alive, l);
                if (tid == 0) lv[a] = v;
            }
            __syncthreads();
            if (tid == 0) {
                double mn = 1.0 / 0.0;
                for (long long a = 0; a < c; ++a) mn = fmin(mn, lv[a]);
                long long w = 0;
                for (long long a = 0; a < c; ++a)
                    if (lv[a] == mn) cand[w++] = cand[a];
                s_count = (unsigned long long)w;
                s_l = l + 1;
            }
            __syncthreads();
        }
        // the first lexicographic minimum in row order is removed
        const long long vrow = keep[cand[0]];
        __syncthreads();
        if (tid == 0) {
            alive[vrow] = 0;
            s_count = 0ull;
        }
        __syncthreads();
        --alive_n;
        // rows that had the victim among their two nearest are rescanned
        for (long long t = tid; t < nk; t += blockDim.x)
            if (alive[keep[t]] && (i1[t] == vrow || i2[t] == vrow)) cand[atomicAdd(&s_count, 1ull)] = t;
        __syncthreads();
        const long long naff = (long long)s_count;
        for (long long a = 0; a < naff; ++a) {
            const long long t = cand[a];
            double d1, d2;
            long long j1, j2;
            block_nn2(F, m, keep[t], keep, nk, alive, d1, j1, d2, j2);
            if (tid == 0) {
                n1[t] = d1;
                i1[t] = j1;
                n2[t] = d2;
                i2[t] = j2;
            }
        }
        __syncthreads();
    }
}

}  // namespace gmpea_b200
