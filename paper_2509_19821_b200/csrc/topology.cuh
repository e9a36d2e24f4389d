// Setup kernels: Das-Dennis reference vectors and neighbourhoods.
//
//   lattice_kernel   reference_vectors (gmpea.cpp:27-71): the smallest lattice
//                    with >= N rows, lexicographic, truncated at the tail.  Each
//                    thread unranks its own composition (closed form for m <= 3)
//                    and writes the exact fp64 weights plus the fp32 unit vector
//                    used by PBI.
//   knn kernels      build_neighborhoods (gmpea.cpp:73-100): t-NN under fp64
//                    squared distance accumulated in coordinate order with no
//                    contraction, ordered by (d2, j) — the std::sort order.
//                    The lattice variant searches a window of lattice offsets
//                    and proves it sufficient (every point outside the window
//                    is strictly farther than the t-th candidate) or flags the
//                    row for a wider retry.  The brute-force variant serves any W.
//   reverse lists    for the pull-based selection: R[k*ld + j] lists, in
//                    ascending order, every offspring c with j in B[c].
#pragma once
#include "common.cuh"

namespace gmpea_b200 {

constexpr int kMaxT = 64;  // insertion-list length for t <= kMaxT
constexpr int kMaxLatM = 16;  // objectives of the operator API's lattices / KNN / metrics (the engine: m <= 3)

__device__ __forceinline__ double d2_exact(const double* a, const double* b, int m) {
    double s = 0.0;
    for (int c = 0; c < m; ++c) {
        double d = __dsub_rn(a[c], b[c]);
        s = __dadd_rn(s, __dmul_rn(d, d));
    }
    return s;
}

// index of composition (a, b) in the m = 3 lexicographic lattice of size H
__host__ __device__ inline long long lat3_start(long long a, long long H) {
    return a * (H + 1) - a * (a - 1) / 2;
}

__device__ __forceinline__ void lat_unrank(long long i, int m, long long H, long long& a,
                                           long long& b) {
    if (m == 2) {
        a = i;
        b = H - i;
        return;
    }
    long long lo = 0, hi = H;  // largest a with start(a) <= i
    while (lo < hi) {
        long long mid = (lo + hi + 1) / 2;
        if (lat3_start(mid, H) <= i)
            lo = mid;
        else
            hi = mid - 1;
    }
    a = lo;
    b = i - lat3_start(lo, H);
}

__device__ __forceinline__ void lat_weights(int m, long long H, long long a, long long b, double* w) {
    const double h = (double)H;
    if (m == 2) {
        w[0] = (double)a / h;
        w[1] = (double)(H - a) / h;
    } else {
        w[0] = (double)a / h;
        w[1] = (double)b / h;
        w[2] = (double)(H - a - b) / h;
    }
}

// compositions of `total` into `parts` non-negative parts: C(total + parts - 1, parts - 1)
__host__ __device__ inline long long lat_count(long long total, int parts) {
    long long c = 1;
    for (int i = 1; i < parts; ++i) c = c * (total + i) / i;
    return c;
}

// reference_vectors for any m (gmpea.cpp:27-71): row i is the i-th composition
// (a_0, .., a_{m-2}, H - sum) in the reference's recursion order (lexicographic,
// a_0 outermost), unranked by counting the compositions of each prefix;
// w_c = a_c / H exactly as the reference divides
__global__ void lattice_m_kernel(int n, int m, long long H, double* W) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long r = i, rem = H;
    const double h = (double)H;
    for (int p = 0; p < m - 1; ++p) {
        long long v = 0;
        for (;; ++v) {
            const long long c = lat_count(rem - v, m - 1 - p);
            if (r < c) break;
            r -= c;
        }
        W[(long long)i * m + p] = (double)v / h;
        rem -= v;
    }
    W[(long long)i * m + m - 1] = (double)rem / h;
}

__global__ void lattice_kernel(int n, int m, long long H, double* W, float4* U) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long a, b;
    lat_unrank(i, m, H, a, b);
    double w[3] = {0.0, 0.0, 0.0};
    lat_weights(m, H, a, b, w);
    double n2 = 0.0;
    for (int c = 0; c < m; ++c) {
        W[(long long)i * m + c] = w[c];
        n2 += w[c] * w[c];
    }
    const double wn = sqrt(n2);
    // lane w: the Tchebycheff weight floor 1e-6 on the unit scale (select.cuh agg_key)
    U[i] = make_float4((float)(w[0] / wn), (float)(w[1] / wn), m > 2 ? (float)(w[2] / wn) : 0.0f,
                       (float)(1e-6 / wn));
}

// unit vectors of an arbitrary W (operator API)
__global__ void unit_kernel(int n, int m, const double* W, float4* U, int* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double w[3] = {0.0, 0.0, 0.0}, n2 = 0.0;
    for (int c = 0; c < m; ++c) {
        w[c] = W[(long long)i * m + c];
        n2 += w[c] * w[c];
    }
    if (n2 == 0.0) atomicExch(err, 1);  // pbi: zero-norm reference vector
    const double wn = sqrt(n2);
    // lane w: the Tchebycheff weight floor 1e-6 on the unit scale (select.cuh agg_key)
    U[i] = make_float4((float)(w[0] / wn), (float)(w[1] / wn), m > 2 ? (float)(w[2] / wn) : 0.0f,
                       (float)(1e-6 / wn));
}

struct TopK {
    double d[kMaxT];
    int j[kMaxT];
    int cnt, t;
    __device__ __forceinline__ void init(int t_) {
        cnt = 0;
        t = t_;
    }
    __device__ __forceinline__ void push(double dd, int jj) {
        // keep ascending (d2, j)
        if (cnt == t && !(dd < d[t - 1] || (dd == d[t - 1] && jj < j[t - 1]))) return;
        int pos = cnt < t ? cnt : t - 1;
        while (pos > 0 && (dd < d[pos - 1] || (dd == d[pos - 1] && jj < j[pos - 1]))) {
            d[pos] = d[pos - 1];
            j[pos] = j[pos - 1];
            --pos;
        }
        d[pos] = dd;
        j[pos] = jj;
        if (cnt < t) ++cnt;
    }
};

// lattice KNN over a window of +-R lattice steps (both lattice axes for m = 3)
__global__ void knn_lattice_kernel(int n, int m, long long H, int t1, int t2, int R, const double* W,
                                   int* B1, int* B2, int* needs_retry) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double wi[kMaxLatM];
    for (int c = 0; c < m; ++c) wi[c] = W[(long long)i * m + c];
    TopK tk;
    tk.init(t2);
    bool covers_all;
    long long a, b;
    lat_unrank(i, m, H, a, b);
    if (m == 2) {
        long long lo = i - R < 0 ? 0 : i - R, hi = i + R >= n ? n - 1 : i + R;
        covers_all = lo == 0 && hi == n - 1;
        for (long long j = lo; j <= hi; ++j) tk.push(d2_exact(wi, W + j * m, m), (int)j);
    } else {
        for (long long aa = a - R; aa <= a + R; ++aa) {
            if (aa < 0 || aa > H) continue;
            for (long long bb = b - R; bb <= b + R; ++bb) {
                if (bb < 0 || aa + bb > H) continue;
                long long j = lat3_start(aa, H) + bb;
                if (j >= n) continue;
                tk.push(d2_exact(wi, W + j * m, m), (int)j);
            }
        }
        // the window holds every lattice point when it spans both axes
        covers_all = (a - R <= 0) && (a + R >= H) && (b - R <= 0) && (b + R >= H);
    }
    if (!covers_all) {
        // every point outside the window has some |delta| >= R + 1 lattice
        // steps: d2 >= (R+1)^2 / H^2 (m = 3), 2 (R+1)^2 / H^2 (m = 2)
        const double step = (double)(R + 1) / (double)H;
        double bound = (m == 2 ? 2.0 : 1.0) * step * step * (1.0 - 1e-9);
        if (tk.cnt < t2 || !(tk.d[t2 - 1] < bound)) {
            atomicExch(needs_retry, 1);
            return;
        }
    }
    for (int k = 0; k < t1; ++k) B1[(long long)i * t1 + k] = tk.j[k];
    for (int k = 0; k < t2; ++k) B2[(long long)i * t2 + k] = tk.j[k];
}

// brute force, any W; t <= kMaxT
__global__ void knn_brute_kernel(int n, int m, int t1, int t2, const double* W, int* B1, int* B2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double wi[kMaxLatM];
    for (int c = 0; c < m; ++c) wi[c] = W[(long long)i * m + c];
    TopK tk;
    tk.init(t2);
    for (int j = 0; j < n; ++j) tk.push(d2_exact(wi, W + (long long)j * m, m), j);
    for (int k = 0; k < t1; ++k) B1[(long long)i * t1 + k] = tk.j[k];
    for (int k = 0; k < t2; ++k) B2[(long long)i * t2 + k] = tk.j[k];
}

// brute force by repeated selection, any t (operator API with t > kMaxT)
__global__ void knn_select_kernel(int n, int m, int t, const double* W, int* B) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double wi[kMaxLatM];
    for (int c = 0; c < m; ++c) wi[c] = W[(long long)i * m + c];
    double pd = -1.0;
    int pj = -1;
    for (int k = 0; k < t; ++k) {
        double bd = 0.0;
        int bj = -1;
        for (int j = 0; j < n; ++j) {
            double dd = d2_exact(wi, W + (long long)j * m, m);
            bool after = dd > pd || (dd == pd && j > pj);
            if (!after) continue;
            if (bj < 0 || dd < bd || (dd == bd && j < bj)) {
                bd = dd;
                bj = j;
            }
        }
        B[(long long)i * t + k] = bj;
        pd = bd;
        pj = bj;
    }
}

// ---- reverse neighbourhood
__global__ void indegree_kernel(int n, int t, const int* B, int* deg) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)n * t) return;
    atomicAdd(&deg[B[e]], 1);
}

__global__ void reverse_fill_kernel(int n, int t, const int* B, int c0, int* fill, int* R, long long ld) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)n * t) return;
    const int c = c0 + (int)(e / t);
    const int j = B[e];
    const int k = atomicAdd(&fill[j], 1);
    R[(long long)k * ld + j] = c;
}

__global__ void reverse_sort_kernel(int n, const int* deg, int* R, long long ld) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int d = deg[j];
    for (int a = 1; a < d; ++a) {
        int v = R[(long long)a * ld + j];
        int b = a - 1;
        while (b >= 0 && R[(long long)b * ld + j] > v) {
            R[(long long)(b + 1) * ld + j] = R[(long long)b * ld + j];
            --b;
        }
        R[(long long)(b + 1) * ld + j] = v;
    }
}

// the reverse neighbourhood packed for select: claimants 4q..4q+3 of slot j
// as int16 offsets c - j in Rp[q*ld + j] (zero past the in-degree); sets
// *overflow when an offset does not fit (the engine then keeps R)
__global__ void pack_reverse_kernel(int n, const int* deg, const int* R, long long ld, int nq, uint2* Rp,
                                    int* overflow) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int d = deg[j];
    for (int q = 0; q < nq; ++q) {
        unsigned w[2] = {0u, 0u};
        for (int u = 0; u < 4; ++u) {
            const int k = 4 * q + u;
            if (k >= d) break;
            const int off = R[(long long)k * ld + j] - j;
            if (off < -32768 || off > 32767) *overflow = 1;
            w[u >> 1] |= ((unsigned)off & 0xffffu) << (16 * (u & 1));
        }
        Rp[(long long)q * ld + j] = make_uint2(w[0], w[1]);
    }
}

}  // namespace gmpea_b200
