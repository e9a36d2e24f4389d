// Selection-side kernels of one GMPEA generation (proj/src/gmpea.cpp:248-390,
// :457-489): PBI keys, OP1 offspring cooperation, the pull-based OP2 + OP3
// select kernel, the loop bookkeeping (end_gen), the time-budget undo
// (restore) and the generation-0 feasible count.  Included by engine.cu only.
#pragma once
#include "kernels.cuh"

namespace gmpea_b200 {

// ---- PBI in fp32 on unit reference vectors (scalarize.cpp:72-89):
// d1 = |(f - z) . u|, d2 = |(f - z) - d1 u|, g = d1 + theta d2.  Unused lanes
// of f, u and z are zero for m = 2.  d2 uses the MUFU square root
// (sqrt.approx, ~1 ulp): the keys are fp32 already, every PBI of a run goes
// through this one function (op1 and select agree), and select's claimant
// loop is latency-bound on it (-7.5 % select time vs the IEEE sqrtf).
__device__ __forceinline__ float pbi(const float4 f, const float4 u, const float3 z, float theta) {
    const float a = f.x - z.x, b = f.y - z.y, c = f.z - z.z;
    const float d1 = fabsf(a * u.x + b * u.y + c * u.z);
    const float r0 = a - d1 * u.x, r1 = b - d1 * u.y, r2 = c - d1 * u.z;
    float d2;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(d2) : "f"(r0 * r0 + r1 * r1 + r2 * r2));
    return d1 + theta * d2;
}

// ---- aggregation of a subproblem key.  AGG_PBI is the reference's (and the
// default); AGG_TCH is the weighted Tchebycheff function the north-star names
// (no reference counterpart, parity unpinned: checked against the oracle's
// f64 restatement): g = max_k max(w_k, 1e-6) |f_k - z_k| on the lattice
// weight w.  With the unit vector u = w / |w| (and u.w = 1e-6 / |w|, set at
// setup) the kernel computes g / |w| -- a positive per-slot scale, so every
// comparison (OP1 at slot i, OP2/OP3 at slot j) decides as on g itself.
enum : int { AGG_PBI = 0, AGG_TCH = 1 };

template <int AGG>
__device__ __forceinline__ float agg_key(const float4 f, const float4 u, const float3 z, float theta) {
    if (AGG == AGG_TCH) {
        const float a = fabsf(f.x - z.x), b = fabsf(f.y - z.y), c = fabsf(f.z - z.z);
        const float t = fmaxf(fmaxf(fmaxf(u.x, u.w) * a, fmaxf(u.y, u.w) * b), fmaxf(u.z, u.w) * c);
        return isnan(a + b + c) ? a + b + c : t;  // fmaxf would drop a NaN (OP1 rejects it)
    }
    return pbi(f, u, z, theta);
}

__device__ __forceinline__ float3 load_z(const DevState* st, int m) {
    float3 z;
    z.x = ordered_to_float(st->zbits[0]);
    z.y = ordered_to_float(st->zbits[1]);
    z.z = m > 2 ? ordered_to_float(st->zbits[2]) : 0.0f;
    return z;
}

struct Op1Params {
    int row0, row_end;
    int m;
    float theta;
    const float4* U;
    const float4* oFcv[2];
    float4* eff[2];
    unsigned char* srcbits;
    DevState* st;
};

// OP1 (gmpea.cpp:248-279).  s1: stream 1 takes off2 (FPR-preferred),
// s2: stream 2 takes off1 (PBI-preferred).  The reference builds both from
// Heaviside masks over differences, which reject non-finite inputs.
template <int AGG>
__device__ __forceinline__ void op1_body(const Op1Params& p, const int bx) {
    // a shard's error arrives as a zero go flag with the ideal-point exchange
    if (p.st->stop || p.st->zbits[3] == 0u) {
        if (bx == 0 && threadIdx.x == 0) halt(p.st);
        return;
    }
    const int i = p.row0 + bx * blockDim.x + threadIdx.x;
    if (i >= p.row_end) return;
    const float3 z = load_z(p.st, p.m);
    const float4 a = p.oFcv[0][i], b = p.oFcv[1][i], u = p.U[i];
    const float g1 = agg_key<AGG>(a, u, z, p.theta), g2 = agg_key<AGG>(b, u, z, p.theta);
    if (!isfinite(a.w - b.w) || !isfinite(g1 - g2)) {
        atomicCAS(&p.st->err, 0, ERR_NONFINITE);
        halt(p.st);
        return;
    }
    const bool s1 = b.w < a.w || (a.w == b.w && g1 > g2);
    const bool s2 = g2 > g1;
    p.eff[0][i] = s1 ? b : a;
    p.eff[1][i] = s2 ? a : b;
    p.srcbits[i] = (unsigned char)((s1 ? 1 : 0) | (s2 ? 2 : 0));
}

template <int AGG>
__global__ void __launch_bounds__(256) op1_kernel(Op1Params p) { op1_body<AGG>(p, blockIdx.x); }

struct SelParams {
    int n, rs4, m;       // n: local rows (winner code c | n + c)
    int row0, row_end;   // parent slots [row0, row_end) selected by this launch
    float theta;
    const float4* U;
    float4* X[2];        // parent rows, updated in place
    float4* Fcv[2];
    const float4* oX[2]; // offspring rows
    const float4* oFcv[2];
    const float4* eff[2];
    const unsigned char* srcbits;
    const int* R[2];     // reverse neighbourhood, R[k*ldr + j] ascending in k
    const uint2* Rp[2];  // the same packed: claimants 4q..4q+3 of j as int16 offsets c - j in Rp[q*ldr + j]
    const int* Rdeg[2];
    long long ldr;
    int* winner[2];      // optional: -1 parent, c: off1 row c, n + c: off2 row c
    int apply;           // copy winner rows into the parents
    // undo log for the time budget (gmpea.cpp:481-486)
    float4* uX[2];
    float4* uFcv[2];
    int* ustamp[2];
    DevState* st;
    DevRecord* rec;      // optional: feasible count of pop1 for this generation
    // the last block to finish runs the generation's bookkeeping (end_gen)
    // and publishes the stop flag, saving two launches per generation
    unsigned* done;
    volatile int* host_flag;
};

// L1 policy of the select kernel (GMPEA_SELECT_L1HINTS): the claimants' keys
// are gathered many times by neighbouring slots and should stay in L1; the
// per-slot streams (parent key, weight, in-degree, reverse rows) and the
// winner rows are touched once, so they bypass / leave L1 first
#ifndef GMPEA_SELECT_L1HINTS
#define GMPEA_SELECT_L1HINTS 1
#endif
// GMPEA_SELECT_L1HINTS 1: ld.global.cs (evict first in L1 and L2); 2: only
// L1::no_allocate (L2 policy untouched)
__device__ __forceinline__ float4 ld_once(const float4* p) {
#if GMPEA_SELECT_L1HINTS == 2
    float4 v;
    asm("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
#elif GMPEA_SELECT_L1HINTS == 1
    return __ldcs(p);
#else
    return *p;
#endif
}
__device__ __forceinline__ int ld_once(const int* p) {
#if GMPEA_SELECT_L1HINTS == 2
    int v;
    asm("ld.global.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#elif GMPEA_SELECT_L1HINTS == 1
    return __ldcs(p);
#else
    return *p;
#endif
}
__device__ __forceinline__ uint2 ld_once(const uint2* p) {
#if GMPEA_SELECT_L1HINTS == 2
    uint2 v;
    asm("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
#elif GMPEA_SELECT_L1HINTS == 1
    return __ldcs(p);
#else
    return *p;
#endif
}
// 256-bit load that does not allocate in L1 (winner rows)
__device__ __forceinline__ void ldg256_na(const float4* p, float4& a, float4& b) {
#if GMPEA_SELECT_L1HINTS
    asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
#else
    ldg256(p, a, b);
#endif
}

// 128-bit load that does not allocate in L1 (winner rows of odd-float4 strides)
#ifndef GMPEA_COPY_NA
#define GMPEA_COPY_NA 1  // (A/B switch)
#endif
__device__ __forceinline__ float4 ldg128_na(const float4* p) {
    float4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ void copy_row(float4* __restrict__ dst, const float4* __restrict__ src, int rs4) {
    if ((rs4 & 1) == 0) {  // rows 32 B aligned: 256-bit loads and stores
        for (int q0 = 0; q0 < rs4; q0 += 8) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; u += 2)
                if (q0 + u < rs4) ldg256_na(src + q0 + u, v[u], v[u + 1]);
#pragma unroll
            for (int u = 0; u < 8; u += 2)
                if (q0 + u < rs4)
                    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + q0 + u),
                                 "f"(v[u].x), "f"(v[u].y), "f"(v[u].z), "f"(v[u].w), "f"(v[u + 1].x),
                                 "f"(v[u + 1].y), "f"(v[u + 1].z), "f"(v[u + 1].w)
                                 : "memory");
        }
        return;
    }
    for (int q0 = 0; q0 < rs4; q0 += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (q0 + u < rs4) v[u] = GMPEA_COPY_NA ? ldg128_na(src + q0 + u) : src[q0 + u];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (q0 + u < rs4) dst[q0 + u] = v[u];
    }
}

// PACK: claimants come from Rp (one 8 B coalesced load per four claimants,
// half the bytes of R); the engine packs only when every |c - j| < 2^15.
__device__ __forceinline__ void unpack_claims(const uint2 w, const int j, const int left, int cc[4]) {
    cc[0] = left > 0 ? j + (int)(short)(w.x & 0xffffu) : -1;
    cc[1] = left > 1 ? j + ((int)w.x >> 16) : -1;
    cc[2] = left > 2 ? j + (int)(short)(w.y & 0xffffu) : -1;
    cc[3] = left > 3 ? j + ((int)w.y >> 16) : -1;
}

template <int POP, bool PACK = false, int NBP = 4, int AGG = AGG_PBI>
__device__ __forceinline__ bool select_slot(const SelParams& p, int j, const float3 z, bool& feas) {
    // claimants per batch: 4 (R), NBP (4 or 8) from the packed Rp
    constexpr int NB = PACK ? NBP : 4;
    constexpr int NW = NB / 4;
    // only the parent's cv and PBI stay live (the full keys are re-read at the
    // end), which keeps select small: 40 registers at 6 blocks of 256 per SM
    const float4 par4 = ld_once(&p.Fcv[POP][j]);
    const float4 u4 = ld_once(&p.U[j]);
    const float gp = agg_key<AGG>(par4, u4, z, p.theta);
    const float pw = par4.w;
    const int deg = ld_once(&p.Rdeg[POP][j]);
    const int* __restrict__ R = p.R[POP];
    const uint2* __restrict__ Rp = p.Rp[POP] + j;
    const float4* __restrict__ eff = p.eff[POP];
    bool have = false;
    float bw = pw;
    float bg = 0.0f;
    int bc = -1;
    bool negcv = false;
    // batches of NB claimants; the next batch's indices are loaded while
    // this batch's keys are gathered (one memory round trip per batch)
    int cc[NB];
    uint2 wn[NW];
    if (PACK) {
#pragma unroll
        for (int h = 0; h < NW; ++h) wn[h] = 4 * h < deg ? ld_once(&Rp[(long long)h * p.ldr]) : make_uint2(0u, 0u);
#pragma unroll
        for (int h = 0; h < NW; ++h) unpack_claims(wn[h], j, deg - 4 * h, cc + 4 * h);
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) cc[u] = u < deg ? R[(long long)u * p.ldr + j] : -1;
    }
    for (int k0 = 0; k0 < deg; k0 += NB) {
        float4 ee[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u)
            if (cc[u] >= 0) ee[u] = eff[cc[u]];
        int cn[4];
        if (PACK) {
#pragma unroll
            for (int h = 0; h < NW; ++h)
                if (k0 + NB + 4 * h < deg) wn[h] = ld_once(&Rp[(long long)((k0 + NB) / 4 + h) * p.ldr]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) cn[u] = k0 + 4 + u < deg ? R[(long long)(k0 + 4 + u) * p.ldr + j] : -1;
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int c = cc[u];
            if (c < 0) continue;
            const float4 e = ee[u];
            const float g = agg_key<AGG>(e, u4, z, p.theta);
            bool mark;
            if (POP == 0) {  // fpr_better (scalarize.cpp:91-96)
                negcv |= (e.w < 0.0f) || (pw < 0.0f);
                mark = (e.w == pw) ? (g < gp) : (e.w < pw);
            } else {
                mark = g < gp;
            }
            if (!mark) continue;
            bool better;
            if (!have)
                better = true;
            else if (POP == 0)
                better = e.w < bw || (e.w == bw && (g < bg || (g == bg && c < bc)));
            else
                better = g < bg || (g == bg && c < bc);
            if (better) {
                have = true;
                bw = e.w;
                bg = g;
                bc = c;
            }
        }
        if (PACK) {
#pragma unroll
            for (int h = 0; h < NW; ++h) unpack_claims(wn[h], j, deg - k0 - NB - 4 * h, cc + 4 * h);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) cc[u] = cn[u];
        }
    }
    if (negcv) {
        atomicCAS(&p.st->err, 0, ERR_NEG_CV);
        halt(p.st);
    }
    // The reference puts the parent into the argmin at index mex(claims)
    // (gmpea.cpp:343-371), where that index decides only an exact key tie
    // between the parent and the best claimant.  Every claimant marked j, i.e.
    // is strictly better than the parent under the same key function (OP2's
    // fpr_better / PBI, recomputed identically in OP3), so the best claimant is
    // too: the tie never occurs and an offspring wins iff some claimant marked j.
    const bool off_wins = have;
    int code = -1;
    if (off_wins) {
        const unsigned char sb = p.srcbits[bc];
        const bool from2 = POP == 0 ? (sb & 1) : !(sb & 2);
        code = from2 ? p.n + bc : bc;
    }
    if (p.winner[POP]) p.winner[POP][j] = code;
    feas = (off_wins ? bw : pw) == 0.0f;
    if (!off_wins || !p.apply) return off_wins;
    const int src = code >= p.n ? 1 : 0;
    float4* dst = p.X[POP] + (long long)j * p.rs4;
    if (p.ustamp[POP]) {
        copy_row(p.uX[POP] + (long long)j * p.rs4, dst, p.rs4);
        p.uFcv[POP][j] = p.Fcv[POP][j];
        p.ustamp[POP][j] = p.st->gen;
    }
    copy_row(dst, p.oX[src] + (long long)bc * p.rs4, p.rs4);  // copy_row, gmpea.cpp:372-377
    p.Fcv[POP][j] = eff[bc];
    return true;
}

#ifndef GMPEA_SELECT_MINBLOCKS
#define GMPEA_SELECT_MINBLOCKS 6  // 40 registers (a small spill): select -3 % against 5 blocks (48)
#endif
#ifndef GMPEA_SELECT_NBP
#define GMPEA_SELECT_NBP 4  // packed claimants gathered per batch (4 or 8)
#endif
template <bool PACK = false, int NBP = 4, int AGG = AGG_PBI>
__device__ __forceinline__ void select_body(const SelParams& p, const int bx, const int by) {
    if (p.st->stop) return;
    const int j = p.row0 + bx * blockDim.x + threadIdx.x;
    const float3 z = load_z(p.st, p.m);
    bool feas = false, off_taken = false;
    if (j < p.row_end) {
        // blockIdx.y = 0 is pop2 (~4x the claimants per slot): the long
        // blocks are dispatched first and pop1's short ones fill the tail
        if (by == 1)
            off_taken = select_slot<0, PACK, NBP, AGG>(p, j, z, feas);
        else
            off_taken = select_slot<1, PACK, NBP, AGG>(p, j, z, feas);
    }
    if (p.rec == nullptr) return;
    // feasible_ratio of pop1 (gmpea.cpp:411-417) and the replacement count
    // (diagnostic): block counts, one atomic each
    __shared__ unsigned cnt[8], rep[8];
    const unsigned b = __popc(__ballot_sync(0xffffffffu, by == 1 && feas && j < p.row_end));
    const unsigned r = __popc(__ballot_sync(0xffffffffu, off_taken));
    if ((threadIdx.x & 31) == 0) {
        cnt[threadIdx.x >> 5] = b;
        rep[threadIdx.x >> 5] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned s = 0, t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            s += cnt[w];
            t += rep[w];
        }
        const int k = rec_slot(p.st, p.st->gen);
        if (k >= 0) {
            if (s) atomicAdd(&p.rec[k].feasible, s);
            if (t) atomicAdd(&p.rec[k].replaced, t);
        }
    }
}

// loop-time bookkeeping after a generation (gmpea.cpp:480-488)
__device__ __forceinline__ void end_gen_body(DevState* st, DevRecord* rec) {
    if (st->stop || st->follower) return;  // a follower takes rank 0's clock (follow_kernel)
    const unsigned long long now = globaltimer();
    st->loop_ns += now - st->t_gen_start;
    if (st->budget_ns && st->loop_ns >= st->budget_ns) {
        st->discard = 1;  // the generation that crossed the deadline is discarded
        st->stop = 1;
        return;
    }
    const int k = rec_slot(st, st->gen);
    if (k >= 0) rec[k].loop_ns = st->loop_ns;
    st->gens_done += 1;
    st->gen += 1;
    if (rec_slot(st, st->gen) < 0) {  // the host did not drain the records: fail loudly
        atomicCAS(&st->err, 0, ERR_RECORDS);
        halt(st);
        return;
    }
    st->t_gen_start = globaltimer();
}

#ifndef GMPEA_SELECT_BS
#define GMPEA_SELECT_BS 128  // threads per select block (A/B: 128 select -2..-4 % against 256, 64 slower)
#endif
constexpr int kSelectBS = GMPEA_SELECT_BS;
template <bool PACK = false, int AGG = AGG_PBI>
__global__ void __launch_bounds__(kSelectBS, GMPEA_SELECT_MINBLOCKS * 256 / kSelectBS) select_kernel(SelParams p) {
    select_body<PACK, GMPEA_SELECT_NBP, AGG>(p, blockIdx.x, blockIdx.y);
    if (p.done == nullptr) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();  // this block's rows, keys and record counts are visible
        const unsigned nblocks = gridDim.x * gridDim.y;
        if (atomicAdd(p.done, 1u) == nblocks - 1) {
            __threadfence();
            end_gen_body(p.st, p.rec);
            if (p.host_flag) *p.host_flag = p.st->stop | (p.st->err ? 2 : 0);
            *p.done = 0u;  // re-armed for the next generation (stream order)
        }
    }
}

__global__ void end_gen_kernel(DevState* st, DevRecord* rec) { end_gen_body(st, rec); }

__global__ void mark_start_kernel(DevState* st) { st->t_gen_start = globaltimer(); }

struct RestoreParams {
    int row0, row_end, rs4;
    float4* X[2];
    float4* Fcv[2];
    const float4* uX[2];
    const float4* uFcv[2];
    const int* ustamp[2];
    DevState* st;
};

__device__ __forceinline__ void restore_body(const RestoreParams& p, const int bx, const int by) {
    if (!p.st->discard) return;
    const int j = p.row0 + bx * blockDim.x + threadIdx.x;
    const int q = by;
    if (j >= p.row_end || p.ustamp[q][j] != p.st->gen) return;
    copy_row(p.X[q] + (long long)j * p.rs4, p.uX[q] + (long long)j * p.rs4, p.rs4);
    p.Fcv[q][j] = p.uFcv[q][j];
}

__global__ void restore_kernel(RestoreParams p) { restore_body(p, blockIdx.x, blockIdx.y); }

// feasible count of pop1 (generation-0 record)
__global__ void count_feasible_kernel(const float4* Fcv, int row0, int row_end, unsigned* out) {
    const int j = row0 + blockIdx.x * blockDim.x + threadIdx.x;
    const bool f = j < row_end && Fcv[j].w == 0.0f;
    unsigned b = __popc(__ballot_sync(0xffffffffu, f));
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(out, b);
}

}  // namespace gmpea_b200
