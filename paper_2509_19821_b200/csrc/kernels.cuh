// Hot-path kernels of one GMPEA generation (proj/src/gmpea.cpp:457-489):
//
//   vary_eval  : reproduce x2 (gmpea.cpp:463-464, :113-206) fused with
//                evaluate_population x2 (:467-468, problems.cpp:552-573) and the
//                ideal-point partial min (update_ideal, :474-475).  One thread
//                per (slot, population); the child row is built in shared
//                memory, evaluated there, and the block's rows leave as one
//                contiguous, fully coalesced store.
//   op1        : offspring cooperation (gmpea.cpp:248-279) as two bits per
//                slot plus the packed keys of the row each stream keeps.
//   select     : OP2 update indexing + OP3 elite update (gmpea.cpp:283-390) as
//                a pull over the reverse neighbourhood: the thread owning parent
//                slot j visits every offspring c with j in B[c], recomputes the
//                mark of (c, j) and keeps the lexicographic argmin of the
//                claimants; the winner row is copied into slot j in place
//                (one writer per slot, race-free; no other parent row is read).
//   end_gen    : loop time / budget bookkeeping (gmpea.cpp:458-488).
//
// Individuals are stored as padded rows  [x_0 .. x_{d-1} | g_0 .. g_{nc-1} | pad]
// of rs4 float4 (LIRCMOP13: 30 + 2 floats = one 128 B line), so a parent or
// winner row is one cache line instead of d separate sectors; the selection
// keys live apart as packed float4 {f0, f1, f2, cv} per slot.
#pragma once
#include <type_traits>

#include "common.cuh"
#include "problems.cuh"

namespace gmpea_b200 {

enum : int { OP_SBX = 0, OP_DE = 1 };
enum : int { MODE_VARY = 0, MODE_EVAL = 1, MODE_INIT = 2 };

// a divisor of uniform_index (rng.hpp:23-30) on 32-bit words: values >= lim
// are rejected, the rest taken modulo n through a reciprocal
struct UIdx {
    unsigned n;
    unsigned mag;            // floor(2^32 / n) (n >= 2; 0 for n = 1)
    unsigned long long lim;  // 2^32 - (2^32 mod n)
};
__host__ inline UIdx make_uidx(unsigned long long n) {
    UIdx u;
    u.n = (unsigned)n;
    u.mag = n >= 2 ? (unsigned)((1ull << 32) / n) : 0u;
    u.lim = (1ull << 32) - (1ull << 32) % n;
    return u;
}


struct VaryParams {
    int n;                   // local rows per population (buffer extent)
    int row0, row_end;       // rows [row0, row_end) are produced by this launch
    int rs4;                 // row stride (float4)
    int srs4;                // shared-memory row stride (float4, odd: bank-conflict free)
    int slot_base;           // global slot index of local row 0 (sharding)
    int pop_id[2];           // Philox population id (1 or 2) per blockIdx.y
    ProbDev P;
    const float4* parX[2];   // parent rows (MODE_VARY) / input rows (MODE_EVAL)
    const int* B[2];         // neighbourhood rows (local indices), row-major
    int t[2];
    float4* out[2];          // output rows (x | g)
    float4* outFcv[2];
    PhiloxKey key;           // Philox key (seed) with its round keys
    unsigned long long sbx_T; // SBX per-child coin: cross iff the PICK word < sbx_T (= ceil(pc 2^32))
    float sbx_e;             // 1 / (eta_c + 1)
    float pm_e1;             // eta_m + 1
    float pm_einv;           // 1 / (eta_m + 1)
    long long pm_T;          // PM on (>= 0) / off (-1)
    const long long* pm_gap; // PM gap table: gap = max k in [0, d] with w <= pm_gap[k] (host.cuh PmGaps)
    float pm_glog;           // 1 / log2(1 - pm): the gap's first estimate (MutCursor)
    long long pm_coinT;      // DE kernels' PM coin: mutate iff w <= pm_coinT (-1 never)
    long long de_T;          // DE: take iff w <= de_T (>= 2^32 - 1: always)
    UIdx ui[2], uid;         // uniform_index divisors: t per population, d (jrand)
    // tournament parents (comparison algorithms, baselines.cpp:347-352, 416-420):
    // tour 1: binary tournament on (rank asc, crowding desc, else the first);
    // tour 2: on fitness (fit[a] <= fit[b] ? a : b); 0: neighbourhood picks
    int tour;
    UIdx un;                 // uniform_index(n) over the population
    const long long* trank[2];
    const double* tkey[2];
    float de_f;
    int scratch8;            // streaming evaluators: per-thread shared words (srs4 = 0)
    int eval;                // evaluate the child (0: reproduce only)
    int update_z;
    int fixed_gen;           // >= 0: use this generation number instead of st->gen
    DevState* st;
    int* bad_rows[2];        // out-of-bounds rows (local index) per population
    int bad_cap;
};

// ---- constraint violation with the reference accumulation order
// (scalarize.cpp:39-49, kernels.cpp:56-67: four lanes over the blocked
// prefix of the inequalities, lanes combined left to right, tail in order,
// then the relaxed equalities).  Values arrive in ascending index.
struct CvAcc {
    double acc[4];
    int nin, blocked;
    __device__ __forceinline__ void init(int nin_) {
        acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
        nin = nin_;
        blocked = nin_ / 4 * 4;
    }
    __device__ __forceinline__ void add(int k, double g) {
        const double r = g > 0.0 ? g : 0.0;
        switch (k & 3) {
            case 0: acc[0] += r; break;
            case 1: acc[1] += r; break;
            case 2: acc[2] += r; break;
            default: acc[3] += r; break;
        }
    }
    __device__ __forceinline__ double total() const {
        return ((acc[0] + acc[1]) + acc[2]) + acc[3];
    }
};

// Emits raw constraints into the row's g part and folds them into cv in the
// reference's order.  For the tail we need s = lanes; s += t_k (in order), so
// the running lane total is materialised when the first tail term arrives.
struct Emitter {
    float* G;
    CvAcc cv;
    double s;
    bool s_ready;
    __device__ __forceinline__ void operator()(int k, double g) {
        if (G) G[k] = (float)g;
        if (k < cv.blocked) {
            cv.add(k, g);
        } else {
            if (!s_ready) {
                s = cv.total();
                s_ready = true;
            }
            if (k < cv.nin) {
                s += g > 0.0 ? g : 0.0;
            } else {
                double v = fabs(g) - 1e-6;
                s += v > 0.0 ? v : 0.0;
            }
        }
    }
    __device__ __forceinline__ double result() {
        if (!s_ready) {
            s = cv.total();
            s_ready = true;
        }
        return s;
    }
};

// ---- Philox-keyed draws (draw schema v2, common.cuh / oracle/philox.h)
// DE's crossover coin when CR < 1 (gmpea.cpp:196, u < CR): eight exact 32-bit
// coins "w <= T" (T in [-1, 2^32 - 1]) from the 16-bit heads of one counter:
// bit k is set when gene j0 + k wins.  A head equal to T's head is refined
// with the tail drawn from its own counter (probability 2^-16 per gene), so
// the result equals the full 32-bit comparison.
__device__ __forceinline__ unsigned coins8(const u32x4& w, long long T, int ngenes, unsigned slot, unsigned gen,
                                           unsigned tag_ref, unsigned j0, const PhiloxKey& K) {
    if (T < 0) return 0u;
    if (T >= 0xffffffffll) return (1u << ngenes) - 1u;
    const unsigned thi = (unsigned)(T >> 16), tlo = (unsigned)(T & 0xffff);
    const unsigned words[4] = {w.x, w.y, w.z, w.w};
    const unsigned valid = (1u << ngenes) - 1u;
    unsigned win = 0u, tie = 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const unsigned h = (k & 1) ? (words[k >> 1] >> 16) : (words[k >> 1] & 0xffffu);
        win |= (unsigned)(h < thi) << k;
        tie |= (unsigned)(h == thi) << k;
    }
    win &= valid;
    tie &= valid;
    while (tie) {  // rare
        const int k = __ffs(tie) - 1;
        tie &= tie - 1u;
        win |= (unsigned)((philox4x32_10(slot, gen, tag_ref, j0 + (unsigned)k, K).x & 0xffffu) <= tlo) << k;
    }
    return win;
}

__device__ __forceinline__ unsigned pick_word(const u32x4& w, int k) {
    return k == 0 ? w.x : (k == 1 ? w.y : (k == 2 ? w.z : w.w));
}

// the PICK stream: 32-bit words, four per counter, consumed in order (a 64-bit
// draw sequence as rng.hpp's measured no faster for DE, A/B DESIGN.md)
struct PickStream {
    unsigned slot, gen, tag;
    const PhiloxKey& K;
    unsigned q;
    u32x4 cache;
    __device__ __forceinline__ unsigned next() {
        if ((q & 3) == 0) cache = philox4x32_10(slot, gen, tag, q >> 2, K);
        return pick_word(cache, (int)(q++ & 3));
    }
    // rng.hpp:23-30: uniform integer in [0, n) by rejection; v mod n by the
    // reciprocal: q = hi32(v floor(2^32 / n)) is floor(v / n) or one less
    __device__ __forceinline__ unsigned index(const UIdx& u) {
        unsigned v;
        do {
            v = next();
        } while ((unsigned long long)v >= u.lim);
        unsigned r = v - __umulhi(v, u.mag) * u.n;
        if (r >= u.n) r -= u.n;
        return r;
    }
};

// the MUFU log2 / exp2 without the denormal fix-ups of __log2f / exp2f (for
// operands known to be normal or zero)
__device__ __forceinline__ float lg2_ftz(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_ftz(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Polynomial mutation's per-gene coin (gmpea.cpp:139, skip iff U > pm) as
// gaps between mutated genes: word t of MSKIP gives the t-th gap, the largest
// k in [0, d] with w <= T[k], T[k] = ceil((1 - pm)^k 2^32) - 1 -- Geometric(pm)
// gaps, i.e. every gene mutates independently with probability pm, at ~2
// words per child instead of one coin per gene.  `next` walks the mutated
// genes in ascending order (d or more: none left).  A float estimate from
// log2(u) / log2(1 - pm) is corrected against the table (one or two loads).
// The SBX kernels draw PM this way; the DE kernels keep one coin per gene
// (MCOIN: its per-group Philox hides the parent loads' latency, A/B DESIGN.md).
struct MutCursor {
    unsigned slot, gen, tag;
    unsigned t;
    u32x4 cache;
    int next;
    __device__ __forceinline__ void advance(const PhiloxKey& K, const long long* __restrict__ T, int d,
                                            float glog) {
        if ((t & 3) == 0) cache = philox4x32_10(slot, gen, tag, t >> 2, K);
        const unsigned w = pick_word(cache, (int)(t++ & 3));
        const float u = ((float)w + 0.5f) * 0x1.0p-32f;
        int k = (int)fminf(fmaxf(lg2_ftz(u) * glog, 0.0f), (float)d);  // u >= 2^-33: normal
        while (k > 0 && (long long)w > T[k]) --k;
        while (k < d && (long long)w <= T[k + 1]) ++k;
        next += k + 1;
    }
};

// 256-bit global load (sm_100: LDG.E.256); p must be 32 B aligned
__device__ __forceinline__ void ldg256(const float4* p, float4& a, float4& b) {
    asm("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
}

__device__ __forceinline__ float clamp_ref(float v, float lo, float hi) {
    return v < lo ? lo : (hi < v ? hi : v);  // NaN passes through (std::clamp)
}

// y^e1 for the mutation; eta_m + 1 is an integer in practice (default 21):
// square-and-multiply then, powf otherwise
__device__ __forceinline__ float pow_e1(float y, float e1) {
    const int k = (int)e1;
    if ((float)k != e1 || k < 1 || k > 64) return powf(y, e1);
    float r = 1.0f, b = y;
    for (int e = k; e; e >>= 1) {
        if (e & 1) r *= b;
        b *= b;
    }
    return r;
}

// gmpea.cpp:135-160 for one gene; w = the MU draw.  Both branches share one
// pair of powf: for u < 0.5  dq = (2u + (1-2u)(1-d1)^e1)^einv - 1, otherwise
// dq = 1 - (2(1-u) + 2(u-0.5)(1-d2)^e1)^einv; the operands are selected first
// so a warp whose lanes disagree on the branch pays for one evaluation.
__device__ __forceinline__ float pm_apply(float x, float lo, float hi, unsigned w, float e1,
                                          float einv) {
    const float span = hi - lo;
    if (!(span > 0.0f)) return x;
    const bool low = w < 0x80000000u;  // u < 0.5
    const float A = low ? (float)w * 0x1.0p-31f           // 2u
                        : (float)(0u - w) * 0x1.0p-31f;   // 2(1-u): 2^32 - w, exact in 32 bits
    const float B = low ? (float)(0x80000000u - w) * 0x1.0p-31f                          // 1 - 2u
                        : (float)(w - 0x80000000u) * 0x1.0p-31f;                         // 2(u-0.5)
    const float dd = (low ? (x - lo) : (hi - x)) * (span == 1.0f ? 1.0f : 1.0f / span);  // d1 / d2
    // (base)^(1/(eta+1)) with base in [0, 2] (NaN for the reference's negative-base
    // hazard, which then fails the bounds check as in gmpea.cpp:146-150)
    const float base = A + B * pow_e1(1.0f - dd, e1);
    const float r = base == 0.0f ? 0.0f : exp2f(einv * __log2f(base));
    const float dq = low ? r - 1.0f : 1.0f - r;
    return x + dq * span;
}

// SBX spread factor (gmpea.cpp:121-124): u <= 0.5: (2u)^e, else
// (1 / (2(1-u)))^e = (2(1-u))^-e with 2(1-u) = (2^32 - w) 2^-31 > 0.  The base
// lies in (0, 2] and e = 1/(eta+1) is small, so exp2(e log2 b) through the
// MUFU pair is accurate to ~2 ulp here (the child differs from the f64 oracle
// by < 1e-6 of the parents' spread) at a fraction of powf's cost.
#ifndef GMPEA_SBX_BRANCHY
#define GMPEA_SBX_BRANCHY 0  // the per-gene branch around the SBX spread (A/B switch)
#endif
// The MUFU pair is issued directly (.ftz: b >= 2^-31 or 0 and the exponent
// lies in [-1.5, 1.5], so the denormal fix-ups exp2f / __log2f wrap around
// it never apply); b = 0 gives lg2 = -inf, ex2(-inf) = +0 = beta.  No branch,
// so a warp computes the spread of a group's genes in one pass.
__device__ __forceinline__ float sbx_beta(unsigned w, float e) {
#if GMPEA_SBX_BRANCHY
    const bool low = w <= 0x80000000u;
    const float b = low ? (float)w * 0x1.0p-31f : (float)(0u - w) * 0x1.0p-31f;  // 2^32 - w (w > 2^31)
    if (b == 0.0f) return 0.0f;  // u = 0: beta = 0
    return exp2f((low ? e : -e) * __log2f(b));
#else
    const bool low = w <= 0x80000000u;
    const float b = (float)(low ? w : 0u - w) * 0x1.0p-31f;  // 2u, or 2(1-u) = (2^32 - w) 2^-31
    return ex2_ftz((low ? e : -e) * lg2_ftz(b));
#endif
}

template <class T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// Block-cooperative polynomial mutation.  Every thread holds a 64-bit mask of
// the genes [w0, w0 + 64) its child mutates; the block numbers all tasks by an
// exclusive scan of the mask popcounts and, round by round, the owners post
// blockDim tasks to shared memory and thread k runs task k on the owner's
// staged row with the owner's Philox key (~1 round per block: PM picks ~1 of
// d genes per child).  Must be reached by every thread of the block.
template <class VP>
__device__ __forceinline__ void pm_tasks(const VP& p, unsigned long long mmask, int w0, float4* sm4,
                                         unsigned gen, unsigned pid, int i0) {
    __shared__ unsigned task[128];  // (owner thread << 16) | gene
    __shared__ int wsum[4];
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int cnt = __popcll(mmask);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int base = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
        base += w < wid ? wsum[w] : 0;
        total += wsum[w];
    }
    const int excl = base + incl - cnt, inc = base + incl;
    const int bs = blockDim.x;
    for (int r0 = 0; r0 < total; r0 += bs) {
        if (excl < r0 + bs && inc > r0) {  // post my tasks with index in [r0, r0 + bs)
            unsigned long long mm = mmask;
            for (int t = excl; t < inc && t < r0 + bs; ++t) {
                const int b = __ffsll((long long)mm) - 1;
                mm &= mm - 1ull;
                if (t >= r0) task[t - r0] = ((unsigned)tid << 16) | (unsigned)(w0 + b);
            }
        }
        __syncthreads();
        if (r0 + tid < total) {
            const unsigned tk = task[tid];
            const int row = (int)(tk >> 16), j = (int)(tk & 0xffffu);
            float* x = reinterpret_cast<float*>(sm4 + row * p.srs4);
            const unsigned slot = (unsigned)(p.slot_base + i0 + row);
            const float lo = p.P.lob(j), hi = p.P.hib(j);
            const u32x4 mu = philox4x32_10(slot, gen, philox_tag(pid, STREAM_MU), (unsigned)j, p.key);
            x[j] = clamp_ref(pm_apply(x[j], lo, hi, mu.x, p.pm_e1, p.pm_einv), lo, hi);
        }
        __syncthreads();
    }
}

// Warp-cooperative polynomial mutation for windows of <= 32 genes: the
// warp's mutation tasks are numbered by an inclusive scan of the lanes' mask
// popcounts; in each round lane t takes task t, finds its owner lane by a
// 5-step binary search over the scanned counts and its gene as the k-th set
// bit of the owner's mask (__fns), then mutates the owner's staged row.  No
// shared task list and no block barrier.
template <class VP>
__device__ __forceinline__ void pm_tasks_warp(const VP& p, unsigned mask, int w0, float4* sm4, unsigned gen,
                                              unsigned pid, int i0) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wbase = threadIdx.x & ~31;
    const int cnt = __popc(mask);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    __syncwarp();  // the lanes' staged rows are visible to the warp
    for (int r0 = 0; r0 < total; r0 += 32) {
        const int t = r0 + lane;
        int owner = 0;  // lanes [0, owner) have incl <= t
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const int v = __shfl_sync(FULL, incl, owner + step - 1);
            if (v <= t) owner += step;
        }
        owner = min(owner, 31);
        const int ex = __shfl_sync(FULL, incl - cnt, owner);
        const unsigned mo = __shfl_sync(FULL, mask, owner);
        if (t < total) {
            const int j = w0 + (int)__fns(mo, 0u, t - ex + 1);
            const int row = wbase + owner;
            float* x = reinterpret_cast<float*>(sm4 + row * p.srs4);
            const unsigned slot = (unsigned)(p.slot_base + i0 + row);
            const float lo = p.P.lob(j), hi = p.P.hib(j);
            const u32x4 mu = philox4x32_10(slot, gen, philox_tag(pid, STREAM_MU), (unsigned)j, p.key);
            x[j] = clamp_ref(pm_apply(x[j], lo, hi, mu.x, p.pm_e1, p.pm_einv), lo, hi);
        }
    }
    __syncwarp();
}

// One thread per (slot, population); block rows are staged in shared memory.
// Phase 1 writes the child genes (before mutation), 64 genes per window, and
// records which genes the PM coin selects; phase 2 applies polynomial
// mutation + clipping to those genes only, so a warp pays for the mutation
// arithmetic once per mutated gene of its busiest lane instead of once per
// gene that any lane mutates (PM picks ~1 of d genes per child); phase 3
// streams the final genes through the problem evaluator; phase 4 stores the
// block's rows as one contiguous coalesced copy.
#ifndef GMPEA_VARY_MINBLOCKS
#define GMPEA_VARY_MINBLOCKS 8
#endif
#ifndef GMPEA_TMA_STORE
#define GMPEA_TMA_STORE 0  // whole-line rows by per-thread cp.async.bulk (A/B switch; phase 4)
#endif
#ifndef GMPEA_MUT_ONLY_CHECK
#define GMPEA_MUT_ONLY_CHECK 0  // phase 3 bounds test on the mutated genes only (A/B switch)
#endif
#ifndef GMPEA_DE_ONECOPY
#define GMPEA_DE_ONECOPY 1  // DE kernels: every gene group through one run-time-count copy (A/B: vary LIRCMOP13 -0.9 %, LIRCMOP14 -0.4 %; 2896 -> 2544 SASS)
#endif
#ifndef GMPEA_VARY_MINBLOCKS_MW
#define GMPEA_VARY_MINBLOCKS_MW 10  // MW kernels (d = 15): 48 registers
#endif
#ifndef GMPEA_DE_GAPS
#define GMPEA_DE_GAPS 0  // DE kernels: PM by gaps instead of per-gene coins (A/B switch)
#endif
#ifndef GMPEA_PREFETCH
#define GMPEA_PREFETCH 1  // bit 0: neighbourhood row to L1 before the picks; bit 1: parent lines to L2 (A/B)
#endif
#ifndef GMPEA_SBX_FULLGROUPS
#define GMPEA_SBX_FULLGROUPS 1  // streaming kernels: compile-time full groups + tail (A/B switch)
#endif
#ifndef GMPEA_VARY_MINBLOCKS_DE
#define GMPEA_VARY_MINBLOCKS_DE GMPEA_VARY_MINBLOCKS
#endif
// DC > 0 compiles the kernel for a fixed decision dimension (the registered
// suites: LIRCMOP 30, MW 15, DTLZ 7/12) so the gene loops unroll completely.
// TOUR: tournament parent picks (the comparison algorithms' instantiation;
// the GMPEA kernels carry no tournament code)
// (the DE kernels used to keep a dead run-time tournament branch, which once
// bought a better register allocation; with one gene-group copy its removal
// is -0.8 % LIRCMOP13 vary and 2544 -> 2136 SASS instructions, A/B in DESIGN.md)
#ifndef GMPEA_TOUR_COND
#define GMPEA_TOUR_COND (TOUR)
#endif
template <class Ev, int MODE, int OP, int DC = 0, bool UB = false, bool TOUR = false>
__device__ __forceinline__ void vary_body(const VaryParams& p, const int bx, const int by) {
    extern __shared__ float4 sm4[];
    DevState* st = p.st;
    if (st->stop) return;
    const int pi = by;
    const int tid = threadIdx.x;
    const int i0 = p.row0 + bx * blockDim.x;
    const int i = i0 + tid;
    const bool active = i < p.row_end;
    const int d = DC > 0 ? DC : p.P.d;
    const int rs4 = p.rs4;
    const unsigned gen = p.fixed_gen >= 0 ? (unsigned)p.fixed_gen : (unsigned)st->gen;
    const unsigned slot = (unsigned)(p.slot_base + i);
    const unsigned pid = (unsigned)p.pop_id[pi];
    const ProbDev& P = p.P;
    // UB: every gene shares [ulo, uhi] (all registered suites), no per-gene loads
    const float ulo = P.ulo, uhi = P.uhi;
#define GMPEA_LO(j) (UB ? ulo : P.lob(j))
#define GMPEA_HI(j) (UB ? uhi : P.hib(j))
    float4* my4 = sm4 + tid * p.srs4;
    // Ev::kStream: no staged row.  The child's genes go from registers to its
    // global row and, in the same pass, through the evaluator, which keeps its
    // per-thread state in shared memory (one column per thread); mutation is
    // applied inline (PM picks ~1 of d genes and d is large for these).
    constexpr bool ST = !Ev::kStream;
    float4* const grow = p.out[pi] + (long long)i * rs4;  // this child's global row
    float4* const wr4 = ST ? my4 : grow;
    Ev ev;
    ev.bind(sm4, tid, (int)blockDim.x);
    const bool stream_eval = !ST && MODE == MODE_VARY && p.eval && active;
    if (stream_eval) ev.begin(p.P);

    double f[kMaxM] = {0.0, 0.0, 0.0};
    bool bad = false;
    // a child's genes outside [lo, hi] can only be mutated ones: crossover /
    // DE children of in-bounds parents are finite and clipped, so only the
    // reference's PM hazard (a NaN, gmpea.cpp:146-150) fails the bounds test
    // of evaluate (problems.cpp:554-561).  With the whole mutation mask in one
    // window (d <= 64, compile-time d) phase 3 tests the mutated genes only.
    constexpr bool kMutOnly = GMPEA_MUT_ONLY_CHECK && MODE == MODE_VARY && DC > 0 && DC <= 64 && !Ev::kStream;
    unsigned long long mut_all = 0ull;
    {
        if (MODE == MODE_EVAL) {
            if (ST && active) {
                const float4* __restrict__ row = p.parX[pi] + (long long)i * rs4;
                for (int q = 0; q < rs4; ++q) my4[q] = row[q];
            }
        } else {
            // the whole warp stays in this branch (pm_tasks is warp-cooperative);
            // lanes past the end only skip the per-slot work
            // parents as one base pointer plus 32-bit row offsets (float4 units;
            // n * rs4 < 2^32) to keep the group loop's live set small
            const float4* __restrict__ PX = p.parX[pi];
            unsigned oa = 0u, ob = 0u;
            const unsigned oc = (unsigned)i * (unsigned)rs4;
            int jrand = -1;
            bool cross = true;
            if (MODE == MODE_VARY && active) {
#if GMPEA_PREFETCH & 1
                // the neighbourhood row arrives while the picks are drawn
                if (!GMPEA_TOUR_COND) asm volatile("prefetch.global.L1 [%0];" ::"l"(p.B[pi] + (long long)i * p.t[pi]));
#endif
                PickStream ps{slot, gen, philox_tag(pid, STREAM_PICK), p.key, 0u, {}};
                if (GMPEA_TOUR_COND) {
                    auto tournament = [&]() {
                        const unsigned a = ps.index(p.un), b = ps.index(p.un);
                        if (p.tour == 1) {
                            const long long ra = p.trank[pi][a], rb = p.trank[pi][b];
                            if (ra != rb) return ra < rb ? a : b;
                            const double ca = p.tkey[pi][a], cb = p.tkey[pi][b];
                            if (ca != cb) return ca > cb ? a : b;
                            return a;
                        }
                        return p.tkey[pi][a] <= p.tkey[pi][b] ? a : b;
                    };
                    const unsigned a = tournament();
                    const unsigned b = tournament();
                    oa = a * (unsigned)rs4;
                    ob = b * (unsigned)rs4;
                } else {
                    const int t = p.t[pi];
                    unsigned a = ps.index(p.ui[pi]);
                    unsigned b = ps.index(p.ui[pi]);
                    while (t > 1 && b == a) b = ps.index(p.ui[pi]);
                    const int* Brow = p.B[pi] + (long long)i * t;
                    oa = (unsigned)Brow[a] * (unsigned)rs4;
                    ob = (unsigned)Brow[b] * (unsigned)rs4;
                }
                if (OP == OP_SBX) {
                    cross = (unsigned long long)ps.next() < p.sbx_T;  // the per-child coin (gmpea.cpp:117)
                } else {
                    jrand = (int)ps.index(p.uid);
                }
            }
#if GMPEA_PREFETCH & 2
            // the parents' lines, all at once, before the first group needs them
            if (MODE == MODE_VARY && active) {
                for (int q = 0; q < rs4; q += 8) {
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(PX + oa + q));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(PX + ob + q));
                }
            }
#endif
            const bool de_all = p.de_T >= 0xffffffffll;
            const bool even_rows = (rs4 & 1) == 0;  // rows 32 B aligned
            const PhiloxKey& K = p.key;
            // the mutated genes, in ascending order (gaps, MutCursor)
            MutCursor mc{slot, gen, philox_tag(pid, STREAM_MSKIP), 0u, {}, -1};
            if ((OP == OP_SBX || GMPEA_DE_GAPS) && MODE == MODE_VARY && active && p.pm_T >= 0)
                mc.advance(K, p.pm_gap, d, p.pm_glog);
            else
                mc.next = d;
            for (int w0 = 0; w0 < d; w0 += 64) {
                const int w1 = min(d, w0 + 64);
                // genes of this window PM selects (32 bits suffice for d <= 32)
                using Mask = typename std::conditional<(DC > 0 && DC <= 32), unsigned, unsigned long long>::type;
                Mask mmask = 0;
                while (mc.next < w1) {
                    mmask |= (Mask)1 << (mc.next - w0);
                    mc.advance(K, p.pm_gap, d, p.pm_glog);
                }
                // SBX per-gene crossover bits of the window (gmpea.cpp:119): one
                // XCOIN counter holds 128 genes' bits
                unsigned long long xwin = 0ull;
                if (OP == OP_SBX && MODE == MODE_VARY && active && cross) {
                    const u32x4 xw = philox4x32_10(slot, gen, philox_tag(pid, STREAM_XCOIN), (unsigned)(w0 >> 7), K);
                    const int wi = (w0 & 127) >> 5;
                    xwin = (unsigned long long)pick_word(xw, wi) | ((unsigned long long)pick_word(xw, wi + 1) << 32);
                }
                if (MODE == MODE_INIT) {
                    for (int jb = w0; jb < (active ? w1 : w0); jb += 4) {  // 64-bit pair (j % 2) of counter j / 2
                        const u32x4 xa = philox4x32_10(slot, 0u, philox_tag(pid, STREAM_INIT), (unsigned)(jb >> 1), K);
                        const u32x4 xb =
                            philox4x32_10(slot, 0u, philox_tag(pid, STREAM_INIT), (unsigned)(jb >> 1) + 1u, K);
                        float v[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int j = jb + k;
                            if (j >= w1) {
                                v[k] = 0.0f;
                                continue;
                            }
                            const u32x4& w = k < 2 ? xa : xb;
                            const double u = (k & 1) ? u53(w.z, w.w) : u53(w.x, w.y);
                            const double lo = GMPEA_LO(j), hi = GMPEA_HI(j);
                            v[k] = (float)(lo + (hi - lo) * u);
                        }
                        wr4[jb >> 2] = make_float4(v[0], v[1], v[2], v[3]);
                    }
                } else {
                    // eight genes per group: their crossover and mutation bits from the
                    // window masks, two XU counters (32-bit spread uniforms); DE's CR
                    // coin (CR < 1 only) one XCOIN counter of 16-bit heads.  NGC > 0
                    // makes the group's gene count a compile-time constant (DC suites),
                    // so the per-gene code carries no bounds tests
                    auto group = [&](const int jb, auto ngc) {
                        constexpr int NGC = decltype(ngc)::value;
                        const int ng = NGC > 0 ? NGC : min(8, w1 - jb);
                        const bool two = NGC > 0 ? (NGC > 4) : (jb + 4 < w1);
                        const int q = jb >> 2;
                        u32x4 xc{0, 0, 0, 0}, xu0{0, 0, 0, 0}, xu1{0, 0, 0, 0}, pmc{0, 0, 0, 0};
                        const unsigned idx8 = (unsigned)(jb >> 3);
                        const unsigned gmask = (2u << (ng - 1)) - 1u;
                        const unsigned xg = (unsigned)(xwin >> (jb - w0)) & gmask;
                        if (OP == OP_SBX && xg) {  // spread uniforms only for a group that crosses
                            xu0 = philox4x32_10(slot, gen, philox_tag(pid, STREAM_XU), (unsigned)q, K);
                            if (two) xu1 = philox4x32_10(slot, gen, philox_tag(pid, STREAM_XU), (unsigned)q + 1u, K);
                        }
                        if (OP == OP_DE && !de_all) xc = philox4x32_10(slot, gen, philox_tag(pid, STREAM_XCOIN), idx8, K);
                        if (OP == OP_DE && !GMPEA_DE_GAPS && p.pm_T >= 0)
                            pmc = philox4x32_10(slot, gen, philox_tag(pid, STREAM_MCOIN), idx8, K);
                        float4 a4[2], b4[2], c4[2];
                        if (two && even_rows) {  // one 32 B sector per parent: 256-bit loads
                            ldg256(PX + (oa + q), a4[0], a4[1]);
                            ldg256(PX + (ob + q), b4[0], b4[1]);
                            if (OP == OP_DE) {
                                ldg256(PX + (oc + q), c4[0], c4[1]);
                            } else {
                                c4[0] = a4[0];
                                c4[1] = a4[1];
                            }
                        } else {
                        a4[0] = PX[oa + q];
                        b4[0] = PX[ob + q];
                        c4[0] = OP == OP_DE ? PX[oc + q] : a4[0];
                        if (two) {
                            a4[1] = PX[oa + q + 1];
                            b4[1] = PX[ob + q + 1];
                            c4[1] = OP == OP_DE ? PX[oc + q + 1] : a4[1];
                        } else {
                            a4[1] = b4[1] = c4[1] = make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                        }
                        // per-gene SBX crossover bit (gmpea.cpp:119), DE CR coin, PM gene
                        const unsigned xbits =
                            OP == OP_SBX ? xg
                                         : (de_all ? (1u << ng) - 1u
                                                   : coins8(xc, p.de_T, ng, slot, gen, philox_tag(pid, STREAM_XREF),
                                                                   (unsigned)jb, K));
                        const unsigned mbits =
                            OP == OP_DE && !GMPEA_DE_GAPS
                                ? coins8(pmc, p.pm_coinT, ng, slot, gen, philox_tag(pid, STREAM_MREF), (unsigned)jb, K)
                                        : (unsigned)(mmask >> (jb - w0)) & gmask;
                        float v[8];
                        auto comp = [](const float4& f, int kk) {
                            return kk == 0 ? f.x : (kk == 1 ? f.y : (kk == 2 ? f.z : f.w));
                        };
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            if (k >= ng) {
                                v[k] = 0.0f;
                                continue;
                            }
                            const int kk = k & 3;
                            const float av = comp(a4[k >> 2], kk);
                            const float bv = comp(b4[k >> 2], kk);
                            if (OP == OP_SBX) {
#if GMPEA_SBX_BRANCHY
                                if ((xbits >> k) & 1u) {
                                    const float beta = sbx_beta(pick_word(k < 4 ? xu0 : xu1, kk), p.sbx_e);
                                    v[k] = 0.5f * ((1.0f + beta) * av + (1.0f - beta) * bv);
                                } else {
                                    v[k] = av;
                                }
#else
                                // every gene of a crossing group through the branch-free
                                // spread, the crossover bit selects (a warp's lanes cross
                                // some gene k almost surely: a branch costs all of them)
                                const float beta = sbx_beta(pick_word(k < 4 ? xu0 : xu1, kk), p.sbx_e);
                                const float cv = 0.5f * ((1.0f + beta) * av + (1.0f - beta) * bv);
                                v[k] = ((xbits >> k) & 1u) ? cv : av;
#endif
                            } else {
                                v[k] = comp(c4[k >> 2], kk) + p.de_f * (av - bv);
                            }
                        }
                        if (OP == OP_DE) {
                            // genes that neither win the CR coin nor are jrand keep the
                            // target's value (gmpea.cpp:196-199); none when CR = 1
                            unsigned take = xbits;
                            const int jr = jrand - jb;
                            if (jr >= 0 && jr < ng) take |= 1u << jr;
                            if (take != (1u << ng) - 1u) {
#pragma unroll
                                for (int k = 0; k < 8; ++k)
                                    if (k < ng && !((take >> k) & 1u)) v[k] = comp(c4[k >> 2], k & 3);
                            }
                        }
                        // clip (gmpea.cpp:202-203; children are finite here, so min/max
                        // equals std::clamp); mutated genes are clipped after PM (phase 2)
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            if (k < ng && !((mbits >> k) & 1u))
                                v[k] = fminf(fmaxf(v[k], GMPEA_LO(jb + k)), GMPEA_HI(jb + k));
                        if constexpr (ST) {
                            if (OP == OP_DE && !GMPEA_DE_GAPS) mmask |= (Mask)mbits << (jb - w0);  // the DE kernels' coins
                        } else {
                            // inline polynomial mutation + clip, then the evaluator, as
                            // rolled loops over the group: one code copy of the PM draw
                            // and of the evaluator's gene step instead of eight (the
                            // unrolled copies overflowed the instruction cache: the WTA
                            // kernel's top stall was "no instruction").  Genes are read
                            // from and written to v[] by compile-time-indexed selects.
                            auto sel = [&](const int k) {
                                float x = v[0];
#pragma unroll
                                for (int kk = 1; kk < 8; ++kk) x = k == kk ? v[kk] : x;
                                return x;
                            };
                            unsigned mb = mbits & ((2u << (ng - 1)) - 1u);
#pragma unroll 1
                            while (mb) {
                                const int k = __ffs(mb) - 1;
                                mb &= mb - 1u;
                                const int j = jb + k;
                                const float lo = GMPEA_LO(j), hi = GMPEA_HI(j);
                                const u32x4 mu = philox4x32_10(slot, gen, philox_tag(pid, STREAM_MU), (unsigned)j, K);
                                const float y = clamp_ref(pm_apply(sel(k), lo, hi, mu.x, p.pm_e1, p.pm_einv), lo, hi);
#pragma unroll
                                for (int kk = 0; kk < 8; ++kk)
                                    if (kk == k) v[kk] = y;
                            }
                            if (stream_eval) {
                                // bounds test and candidate mask on the group's registers;
                                // the evaluator visits the candidates only
                                unsigned cand = 0u;
#pragma unroll
                                for (int k = 0; k < 8; ++k) {
                                    if (k >= ng) continue;
                                    if (!(v[k] >= GMPEA_LO(jb + k) && v[k] <= GMPEA_HI(jb + k))) bad = true;
                                    if (Ev::candidate(v[k])) cand |= 1u << k;
                                }
                                ev.group(p.P, ng, cand, sel);
                            }
                        }
                        wr4[q] = make_float4(v[0], v[1], v[2], v[3]);
                        if (two) wr4[q + 1] = make_float4(v[4], v[5], v[6], v[7]);
                    };
                    if (active) {
                        // SBX kernels run every group, the tail included, through one
                        // run-time-count copy: their second (tail) copy cost more in
                        // instruction fetch than the bounds tests it saves (A/B:
                        // DAS-CMOP9 vary -4.2 %, DAS-CMOP7 -3.3 %, MW1 -0.9 %, MW7 +0.3 %);
                        // so do the DE kernels (GMPEA_DE_ONECOPY)
                        if (DC > 0 && DC <= 64 && OP != OP_SBX && !GMPEA_DE_ONECOPY) {  // one window, full groups then the tail
#pragma unroll 1
                            for (int jb = 0; jb + 8 <= DC; jb += 8) group(jb, std::integral_constant<int, 8>{});
                            if (DC % 8) group(DC / 8 * 8, std::integral_constant<int, (DC % 8)>{});
                        } else if (GMPEA_SBX_FULLGROUPS && DC == 0 && !ST) {
                            // streaming evaluators (WTA, d in the hundreds): full groups
                            // with a compile-time count, then the run-time tail
#pragma unroll 1
                            for (int jb = w0; jb + 8 <= w1; jb += 8) group(jb, std::integral_constant<int, 8>{});
                            if ((w1 - w0) & 7) group(w1 - ((w1 - w0) & 7), std::integral_constant<int, 0>{});
                        } else {
#pragma unroll 1
                            for (int jb = w0; jb < w1; jb += 8) group(jb, std::integral_constant<int, 0>{});
                        }
                    }
                }
                // phase 2: polynomial mutation then clip (gmpea.cpp:202-203).
                // The warp's mutation tasks (lane, gene) are dealt round-robin
                // over its lanes, ~1 task per lane per round.
                if (ST && MODE == MODE_VARY) {
                    if (DC > 0 && DC <= 32)
                        pm_tasks_warp(p, (unsigned)mmask, w0, sm4, gen, pid, i0);
                    else
                        pm_tasks(p, (unsigned long long)mmask, w0, sm4, gen, pid, i0);
                }
                if (kMutOnly) mut_all = (unsigned long long)mmask;
            }
        }
        if (p.eval && active) {
            // phase 3: bounds check (problems.cpp:554-561) + streamed evaluation
            // (already done in the gene loop for streaming evaluators)
            // MW / DAS-CMOP: the staged row through one rolled gene loop (one
            // copy of the evaluator's gene step instead of d: instruction fetch;
            // A/B vary: MW1 -4.6 %, MW7 -2.6 %, DAS-CMOP7 -1.4 %, DAS-CMOP9 -4.3 %,
            // C1-DTLZ1 -1.1 %;
            // the LIRCMOP kernels lose 8-11 % rolled and keep the unrolled loop)
            constexpr bool ROLL_EVAL = ST && (is_mw<Ev>::value || is_das<Ev>::value || is_dtlz<Ev>::value);
            if constexpr (ROLL_EVAL) {
                ev.begin(p.P);
                const float* rd = reinterpret_cast<const float*>(my4);
                // MW: two genes per trip (A/B: vary MW1 -2.2 %, MW7 -0.9 %;
                // DAS-CMOP9 +0.8 % and C1-DTLZ1 +0.2 % keep one)
                constexpr int EU = is_mw<Ev>::value ? 2 : 1;
#pragma unroll EU
                for (int j = 0; j < d; ++j) {
                    const float x = rd[j];
                    if (!kMutOnly && !(x >= GMPEA_LO(j) && x <= GMPEA_HI(j))) bad = true;
                    ev.gene(p.P, j, x);
                }
            } else if (!stream_eval) {
                ev.begin(p.P);
                const float4* rd4 = ST ? my4 : grow;
                for (int jb = 0; jb < d; jb += 4) {
                    const float4 v4 = rd4[jb >> 2];
                    const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int j = jb + k;
                        if (j >= d) break;
                        if (!kMutOnly && !(v[k] >= GMPEA_LO(j) && v[k] <= GMPEA_HI(j))) bad = true;
                        ev.gene(p.P, j, v[k]);
                    }
                }
            }
            if (kMutOnly) {
                const float* rd = reinterpret_cast<const float*>(my4);
                for (unsigned long long mm = mut_all; mm; mm &= mm - 1ull) {
                    const int j = __ffsll((long long)mm) - 1;
                    if (!(rd[j] >= GMPEA_LO(j) && rd[j] <= GMPEA_HI(j))) bad = true;
                }
            }
            if (bad) {
                int k = atomicAdd(&st->n_bad[pi], 1);
                if (k < p.bad_cap) p.bad_rows[pi][k] = p.slot_base + i;  // the population's row index
                if (atomicCAS(&st->err, 0, ERR_EVAL_OOB) == 0) st->err_gen = (int)gen;
                // the reference throws here (gmpea.cpp:469-471): the rest of the run is a no-op
                if (MODE == MODE_VARY) halt(st);
            } else {
                Emitter em{reinterpret_cast<float*>(wr4) + d, {}, 0.0, false};
                em.cv.init(p.P.nin);
                ev.finish(p.P, f, em);
                float4 o;
                o.x = (float)f[0];
                o.y = (float)f[1];
                o.z = p.P.m > 2 ? (float)f[2] : 0.0f;
                o.w = (float)em.result();
                p.outFcv[pi][i] = o;
            }
        }
    }
    // phase 4: the block's rows leave shared memory as one contiguous,
    // coalesced copy of rows [i0, i0 + rows).  GMPEA_TMA_STORE sends rows of
    // whole 128 B lines (rs4 % 8 == 0, LIRCMOP1-13) through the bulk-copy
    // engine instead (per-thread cp.async.bulk, UBLKCP, after a proxy fence
    // and one barrier): LIRCMOP13 vary -1.9 % when it was measured, +2.2 %
    // since the kernel's hot code shrank (one group copy, no tournament
    // branch: its operand loop over the lanes now costs more than it saves);
    // rows that straddle lines cost MW7 +6 %, DAS-CMOP9 +2 %, C1-DTLZ1 +13 %
    // (A/B in DESIGN.md)
    if (ST && GMPEA_TMA_STORE && (rs4 & 7) == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (active) {
            const unsigned saddr = (unsigned)__cvta_generic_to_shared(my4);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(grow), "r"(saddr),
                         "r"(rs4 * 16)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    } else if (ST) {
        __syncthreads();
        const int rows = min((int)blockDim.x, p.row_end - i0);
        const int total = rows * rs4;
        float4* __restrict__ dst = p.out[pi] + (long long)i0 * rs4;
        const float inv = 1.0f / (float)rs4;  // exact floor for e < 2^20
        if ((rs4 & 1) == 0) {  // float4 pairs: 256-bit stores (rows 32 B aligned)
            for (int e = 2 * tid; e < total; e += 2 * blockDim.x) {
                const int r = (int)(((float)e + 0.5f) * inv);
                const float4* src = sm4 + r * p.srs4 + (e - r * rs4);
                const float4 a = src[0], b = src[1];
                asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + e), "f"(a.x), "f"(a.y),
                             "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
                             : "memory");
            }
        } else {
            for (int e = tid; e < total; e += blockDim.x) {
                const int r = (int)(((float)e + 0.5f) * inv);
                dst[e] = sm4[r * p.srs4 + (e - r * rs4)];
            }
        }
    }
    if (!p.update_z || !p.eval) return;
    // ideal point: block min per objective, one atomic per block only when
    // the block improves on the current z (update_ideal, gmpea.cpp:102-109)
    __shared__ unsigned smin[kMaxM][4];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kMaxM; ++k) {
        unsigned v = (active && !bad && k < p.P.m) ? float_to_ordered((float)f[k]) : 0xffffffffu;
        v = warp_min(v);
        if (lane == 0) smin[k][wid] = v;
    }
    __syncthreads();
    if (threadIdx.x < kMaxM && (int)threadIdx.x < p.P.m) {
        const int k = threadIdx.x;
        unsigned v = smin[k][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = smin[k][w] < v ? smin[k][w] : v;
        if (v < *(volatile unsigned*)&st->zbits[k]) atomicMin(&st->zbits[k], v);
    }
}
#undef GMPEA_LO
#undef GMPEA_HI

// blocks per SM: 8 (63 registers); the MW kernel (d = 15, smaller rows and
// evaluator state) runs faster at 10 (48 registers) despite a small spill,
// LIRCMOP13 slower (A/B)
template <class Ev, int OP, int DC>
constexpr int vary_minblocks() {
    return DC == 15 && is_mw<Ev>::value ? GMPEA_VARY_MINBLOCKS_MW : (OP == OP_DE ? GMPEA_VARY_MINBLOCKS_DE : GMPEA_VARY_MINBLOCKS);
}

template <class Ev, int MODE, int OP, int DC = 0, bool UB = false, bool TOUR = false>
__global__ void __launch_bounds__(128, (vary_minblocks<Ev, OP, DC>())) vary_eval_kernel(VaryParams p) {
    vary_body<Ev, MODE, OP, DC, UB, TOUR>(p, blockIdx.x, blockIdx.y);
}

}  // namespace gmpea_b200
