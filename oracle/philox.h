/* oracle/philox.h — TEST INFRASTRUCTURE ONLY (the checker, never shipped).
 *
 * Independent CPU restatement of Philox4x32-10 (Salmon et al., SC'11; the
 * algorithm cuRAND ships as curand_Philox4x32_10) and of the GMPEA-B200 draw
 * key schema.  The product kernels carry their own implementation
 * (paper_2509_19821_b200/csrc/common.cuh); tests/test_oracle_pins.py pins this
 * one to the published Random123 known-answer vectors, and the GPU parity
 * tests compare the two draw for draw.
 *
 * Key schema (shared contract between the CUDA engine and this oracle):
 *   key = { (u32)seed, (u32)(seed >> 32) }
 *   ctr = { slot, gen, tag(pop, stream), index }
 *   tag(pop, stream) = (pop << 28) | (stream << 20)
 * streams (draw schema v2):
 *   INIT   initial population, gen = 0; two 64-bit draws per counter
 *   PICK   a sequence of 32-bit words, four per counter: the neighbour picks a,
 *          b (rejection sampling, b == a redrawn), then DE's jrand or SBX's
 *          per-child coin (taken iff w < ceil(pc 2^32))
 *   XCOIN  SBX per-gene crossover bit: gene j is bit j%32 of word (j%128)/32 of
 *          index j/128 (crosses iff 1); DE's CR coin when CR < 1: the 32-bit
 *          coin w = (h << 16) | l, head h = 16-bit half j%8 of index j/8
 *          (word (j%8)/2, low half first), tail l = low 16 bits of word 0 of
 *          index j of XREF
 *   XU     SBX spread uniform: gene j = word j%4 of index j/4, u = w * 2^-32
 *   MSKIP  SBX operator's PM gaps: word t (index t/4, word t%4) is the t-th gap
 *          between mutated genes, gap = max k in [0, d] with
 *          w <= ceil((1-pm)^k 2^32) - 1
 *   MCOIN  DE operator's PM coin of gene j: the 32-bit coin (as XCOIN's for CR,
 *          tail from MREF); mutates iff pm > 0 and w 2^-32 <= pm
 *   MU     PM direction of a mutated gene j: index j, word 0
 */
#ifndef GMPEA_ORACLE_PHILOX_H
#define GMPEA_ORACLE_PHILOX_H
#include <stdint.h>

enum {
    ORC_STREAM_INIT = 1, ORC_STREAM_PICK = 2, ORC_STREAM_CHILD = 3,
    ORC_STREAM_XCOIN = 5, ORC_STREAM_XU = 6, ORC_STREAM_MCOIN = 7, ORC_STREAM_MU = 8,
    ORC_STREAM_XREF = 9, ORC_STREAM_MREF = 10, ORC_STREAM_MSKIP = 11  /* CHILD: draw schema v1 */
};

static inline uint32_t orc_tag(uint32_t pop, uint32_t stream) {
    return (pop << 28) | (stream << 20);
}

static inline void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                                     uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

#endif
