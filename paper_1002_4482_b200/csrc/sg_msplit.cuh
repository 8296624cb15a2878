// sg_msplit.cuh -- block multisplit of 64-bit pairs into bins by ballots.
//
// Used by the edge partition (sg_cc.cu) and by the ranking's window passes
// (sg_list.cu).  Shared-memory atomics cost ~2 cycles per lane on this part
// (B300_MICROARCH.md: ATOMS spread-addr), which made one per element the
// bottleneck of a scatter pass; here a warp groups its 32 elements by bin
// with nbits ballots (lanes with equal bins = peers), so every (warp, bin)
// has one leader that updates a warp-private counter -- no atomics inside
// the block -- and one global atomic per (tile, bin) claims the tile's slots.
#pragma once

#include "sg_internal.cuh"

namespace sg {

constexpr int MS_THREADS = 256;
constexpr int MS_WARPS = MS_THREADS / 32;
constexpr int MS_MAXB = 1024;

// lanes (among `valid` ones) holding the same nbits-bit key as this lane
__device__ __forceinline__ unsigned ms_peers(uint32_t key, bool valid, int nbits) {
    unsigned m = __ballot_sync(0xffffffffu, valid);
    for (int b = 0; b < nbits; ++b) {
        const bool bit = (key >> b) & 1u;
        const unsigned bb = __ballot_sync(0xffffffffu, bit);
        m &= bit ? bb : ~bb;
    }
    return m;
}

// One tile: elements [e0, e1) in steps of MS_THREADS (coalesced).
// get(e, pair, bin, want_pair) -> false to skip an element; bins < nb <= MS_MAXB,
// nbits = ceil(log2 nb).  slot(bin) = {first slot, capacity}; cursor[bin]
// (global, u64) counts slots already claimed.  Returns true if a bin
// overflowed (only for inputs that break the caller's size contract).
template <int ITEMS, class Get, class Slot>
__device__ __forceinline__ bool ms_tile(Get get, Slot slot, unsigned long long e0, unsigned long long e1, uint32_t nb,
                                        int nbits, unsigned long long* __restrict__ cursor,
                                        unsigned long long* __restrict__ out) {
    __shared__ uint32_t s_w[MS_WARPS][MS_MAXB];
    __shared__ unsigned long long s_base[MS_MAXB];
    const uint32_t lane = lane_id();
    const int w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (uint32_t b = lane; b < nb; b += 32) s_w[w][b] = 0;
    __syncwarp();
    // phase A: per-warp bin counts
    for (int j = 0; j < ITEMS; ++j) {
        const unsigned long long e = e0 + (unsigned long long)j * MS_THREADS + threadIdx.x;
        unsigned long long pr;
        uint32_t b = 0;
        const bool ok = e < e1 && get(e, pr, b, false) && b < nb;
        const unsigned peers = ms_peers(b, ok, nbits);
        if (ok && (peers & lt) == 0) s_w[w][b] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // warp offsets per bin, tile slots per bin
    for (uint32_t b = threadIdx.x; b < nb; b += MS_THREADS) {
        uint32_t acc = 0;
#pragma unroll
        for (int k = 0; k < MS_WARPS; ++k) {
            const uint32_t c = s_w[k][b];
            s_w[k][b] = acc;
            acc += c;
        }
        s_base[b] = acc ? atomicAdd(cursor + b, (unsigned long long)acc) : 0ull;
    }
    __syncthreads();
    // phase B: place
    bool over = false;
    for (int j = 0; j < ITEMS; ++j) {
        const unsigned long long e = e0 + (unsigned long long)j * MS_THREADS + threadIdx.x;
        unsigned long long pr = 0;
        uint32_t b = 0;
        const bool ok = e < e1 && get(e, pr, b, true) && b < nb;
        const unsigned peers = ms_peers(b, ok, nbits);
        if (ok) {
            const unsigned long long pos = s_base[b] + s_w[w][b] + __popc(peers & lt);
            const ulonglong2 sc = slot(b);
            if (pos < sc.y)
                out[sc.x + pos] = pr;
            else
                over = true;
        }
        __syncwarp();
        if (ok && (peers & lt) == 0) s_w[w][b] += __popc(peers);
        __syncwarp();
    }
    return over;
}

}  // namespace sg
