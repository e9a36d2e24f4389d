// Common device definitions for the GMPEA-B200 engine (sm_100a).
//
// Layout conventions (DESIGN.md §3 "Data layout in HBM"):
//   * individuals are padded fp32 rows [x_0..x_{d-1} | g_0..g_{nc-1} | pad] of
//     rs4 float4, and the selection keys are packed per slot as
//     Fcv[i] = float4{f0, f1, f2, cv} (m <= 3; unused lanes are 0).
//   * reference vectors are kept twice: exact fp64 lattice values only during
//     setup (neighbourhoods are decided by fp64 distances, gmpea.cpp:84-97),
//     and U[i] = float4{w/|w|} for the PBI hot path.
//   * neighbourhoods: B[i*t + l] (int32, row-major, gmpea.hpp:45-51) for the
//     variation gathers, and the reverse neighbourhood padded SoA
//     R[k*ld + j] / Rdeg[j] (ascending offspring ids) for the pull-based
//     selection (one writer per parent slot, no atomics on data).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gmpea_b200 {

constexpr int kMaxM = 3;          // objectives handled by the packed Fcv key
constexpr int kMaxBadRows = 1024; // out-of-bounds rows remembered per run

// engine-wide error codes (mirrored in include/gmpea_b200.h)
enum : int {
    ERR_NONE = 0,
    ERR_EVAL_OOB = 1,     // evaluate: out-of-bounds (incl. NaN) rows
    ERR_NONFINITE = 2,    // heaviside: non-finite mask source (OP1)
    ERR_NEG_CV = 3,       // fpr_better: negative constraint violation
    ERR_RECORDS = 4,      // the generation-record buffer was not drained in time
};

// Per-run device state; one instance per engine (and per operator call).
struct DevState {
    unsigned zbits[4];          // ideal point, order-preserving float encoding
    int gen;                    // generation currently being produced (1-based)
    int stop;                   // nonzero: every kernel of the generation is a no-op
    int discard;                // the generation that crossed the deadline is undone
    int err;                    // first error code
    int err_gen;
    int n_bad[2];               // out-of-bounds rows per offspring population
    int bad_rows[2][kMaxBadRows];
    unsigned long long t_gen_start;
    unsigned long long loop_ns;  // accumulated loop time (gmpea.cpp:443,480)
    unsigned long long budget_ns; // 0 = no time budget
    int gens_done;
    int rec_base;               // generation of record slot 0 (the host drains older records)
    int rec_cap;                // record slots on the device
    int follower;               // a sharded time-budget run's shard > 0: rank 0 keeps the loop clock
};

// stops the run after an error.  zbits[3] (no objective uses it; 0x80000000
// otherwise) doubles as the shards' go flag: the ideal-point MIN exchange of
// a sharded run carries a 0 to every shard, whose OP1 then stops too.
__device__ __forceinline__ void halt(DevState* st) {
    st->stop = 1;
    st->zbits[3] = 0u;
}

// record slot of generation g, or -1 outside the device window
__host__ __device__ inline int rec_slot(const DevState* st, int g) {
    const int k = g - st->rec_base;
    return (k >= 0 && k < st->rec_cap) ? k : -1;
}

// per-generation record (gmpea.hpp:129-136); evals is derived on the host
struct DevRecord {
    unsigned feasible;  // rows of pop1 with cv == 0 after the generation
    unsigned replaced;  // slots of both populations that took an offspring (OP3)
    unsigned long long loop_ns;
};

// ---- order-preserving float <-> uint (atomicMin on floats of either sign)
__host__ __device__ inline unsigned float_to_ordered(float f) {
#ifdef __CUDA_ARCH__
    unsigned u = __float_as_uint(f);
#else
    unsigned u;
    __builtin_memcpy(&u, &f, 4);
#endif
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ inline float ordered_to_float(unsigned u) {
    unsigned v = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
#ifdef __CUDA_ARCH__
    return __uint_as_float(v);
#else
    float f;
    __builtin_memcpy(&f, &v, 4);
    return f;
#endif
}

// ---- Philox4x32-10 (Salmon et al. SC'11), the counter-based generator of the
// engine.  Key schema (shared with oracle/philox.h, the test checker):
//   key = {(u32)seed, (u32)(seed >> 32)}, ctr = {slot, gen, tag(pop, stream), index}
// Draw schema v2 (oracle/philox.h is the checker's copy of the contract)
enum : unsigned {
    STREAM_INIT = 1,   // initial population, pair of 64-bit draws per counter
    STREAM_PICK = 2,   // 32-bit words, four per counter: picks a, b (b == a redrawn), DE jrand / SBX child coin
    STREAM_XCOIN = 5,  // SBX per-gene crossover bit (128 genes per counter); DE CR coin heads (CR < 1)
    STREAM_XU = 6,     // per-gene SBX spread uniform, 4 genes per counter
    STREAM_MCOIN = 7,  // DE kernels' per-gene PM coin: 16-bit heads, 8 genes per counter
    STREAM_MU = 8,     // PM direction uniform, one counter per mutated gene
    STREAM_XREF = 9,   // low 16 bits of a DE CR coin whose head ties the threshold
    STREAM_MREF = 10,  // low 16 bits of a PM coin whose head ties the threshold
    STREAM_MSKIP = 11, // SBX kernels' PM gaps between mutated genes, 32-bit words, four per counter
};

__host__ __device__ inline unsigned philox_tag(unsigned pop, unsigned stream) {
    return (pop << 28) | (stream << 20);
}

struct u32x4 {
    unsigned x, y, z, w;
};

__device__ __forceinline__ u32x4 philox4x32_10(unsigned c0, unsigned c1, unsigned c2, unsigned c3,
                                               unsigned k0, unsigned k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        unsigned lo0 = 0xD2511F53u * c0;
        unsigned hi0 = __umulhi(0xD2511F53u, c0);
        unsigned lo1 = 0xCD9E8D57u * c2;
        unsigned hi1 = __umulhi(0xCD9E8D57u, c2);
        unsigned n0 = hi1 ^ c1 ^ k0;
        unsigned n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return {c0, c1, c2, c3};
}

// Philox key with the ten round keys precomputed on the host: kept in the
// kernel's parameter space, every round key is a constant-bank operand of the
// round's LOP3 instead of a live register (or a per-round add)
struct PhiloxKey {
    unsigned k[20];  // (k0, k1) of round r at [2r], [2r + 1]
};

__host__ inline PhiloxKey make_philox_key(unsigned long long seed) {
    PhiloxKey K;
    unsigned k0 = (unsigned)seed, k1 = (unsigned)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        K.k[2 * r] = k0;
        K.k[2 * r + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return K;
}

__device__ __forceinline__ u32x4 philox4x32_10(unsigned c0, unsigned c1, unsigned c2, unsigned c3,
                                               const PhiloxKey& K) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        unsigned lo0 = 0xD2511F53u * c0;
        unsigned hi0 = __umulhi(0xD2511F53u, c0);
        unsigned lo1 = 0xCD9E8D57u * c2;
        unsigned hi1 = __umulhi(0xCD9E8D57u, c2);
        unsigned n0 = hi1 ^ c1 ^ K.k[2 * r];
        unsigned n2 = hi0 ^ c3 ^ K.k[2 * r + 1];
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return {c0, c1, c2, c3};
}

__device__ __forceinline__ double u53(unsigned lo, unsigned hi) {
    unsigned long long v = ((unsigned long long)hi << 32) | lo;
    return (double)(v >> 11) * 0x1.0p-53;
}

// ---- misc
__host__ __device__ inline long long round_up(long long v, long long a) { return (v + a - 1) / a * a; }

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

}  // namespace gmpea_b200
