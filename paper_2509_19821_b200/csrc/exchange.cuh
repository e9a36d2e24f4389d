// Shard exchange of a weight-region sharded run (the ideal-point
// all-reduce between update_ideal and selection, gmpea.cpp:474-478).  The
// engine runs it inside each generation's CUDA graph, over NCCL (one process
// per GPU) or over peer memory (one process driving several devices):
//
//   after vary_eval   ideal point: MIN over the shards of zbits[0..3] (word 3
//                     is the go flag, zeroed by halt(): errors stop all shards)
//   after select      time budget only: rank 0's loop clock and stop /
//                     discard decision (LeadState) replace every follower's
//   after select      the 2r boundary parent rows, to each neighbour (copies
//                     or NCCL send / recv; no keys: only X of halo rows is read)
#pragma once
#include "common.cuh"

namespace gmpea_b200 {

constexpr int kMaxShards = 16;

struct PeerStates {
    const DevState* st[kMaxShards];
    int n;
};

// zbits <- MIN over every shard's zbits (peer loads over NVLink, or the same
// device).  Racing with a peer's own update is harmless: a peer's words only
// move from its partial minimum to the global one.
__global__ void z_peers_kernel(DevState* mine, PeerStates peers) {
    const int k = threadIdx.x;
    if (k >= 4) return;
    unsigned v = mine->zbits[k];
    for (int j = 0; j < peers.n; ++j) v = min(v, *(volatile const unsigned*)&peers.st[j]->zbits[k]);
    mine->zbits[k] = v;
}

// rank 0's loop state after a generation (end_gen_body)
struct LeadState {
    int gen, gens_done, stop, discard;
    unsigned long long loop_ns;
};

__global__ void lead_pack_kernel(const DevState* st, LeadState* out) {
    out->gen = st->gen;
    out->gens_done = st->gens_done;
    out->stop = st->stop;
    out->discard = st->discard;
    out->loop_ns = st->loop_ns;
}

// a follower shard adopts rank 0's generation count, clock and deadline
// decision (so every shard keeps or discards the same generation)
__global__ void follow_kernel(DevState* st, const LeadState* lead, volatile int* host_flag) {
    const volatile LeadState* L = lead;  // another device's memory (multi-device handle) or NCCL's copy
    st->gen = L->gen;
    st->gens_done = L->gens_done;
    st->loop_ns = L->loop_ns;
    st->discard = L->discard;
    if (L->stop) st->stop = 1;
    if (host_flag) *host_flag = st->stop | (st->err ? 2 : 0);
}

// boundary rows of both populations from a neighbour shard (peer loads over
// NVLink, or the same device): dst[q][i] = src[q][i], i < n4 float4
struct HaloCopy {
    float4* dst[2];
    const float4* src[2];
    long long n4;
};

__global__ void __launch_bounds__(256) halo_pull_kernel(HaloCopy h) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (int q = 0; q < 2; ++q)
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < h.n4; i += stride)
            h.dst[q][i] = h.src[q][i];
}

}  // namespace gmpea_b200
