// sg_msplit.cuh -- block multisplit of 64-bit pairs into bins.
//
// Used by the edge partition (sg_cc.cu) and by the ranking's window passes
// (sg_list.cu).  A tile of MS_THREADS x MS_ITEMS elements is
//   1. loaded up front (all loads of a thread in flight at once),
//   2. ranked per bin in the warp: lanes with equal bins ("peers", one
//      match.any per element) elect one leader per (warp, bin) that updates a
//      warp-private counter -- no shared-memory atomics, which cost ~2 cycles
//      per lane on this part (B300_MICROARCH.md, ATOMS spread-addr),
//   3. sorted by bin through shared memory, and
//   4. written out bin run by bin run: consecutive threads store consecutive
//      slots, so every run leaves the SM as full sectors.
// One global atomic per (tile, bin) claims the tile's slots of a bin.
#pragma once

#include "sg_internal.cuh"

namespace sg {

constexpr int MS_THREADS = 256;
constexpr int MS_WARPS = MS_THREADS / 32;
constexpr int MS_ITEMS = 8;
constexpr int MS_TILE = MS_THREADS * MS_ITEMS;
constexpr int MS_MAXB = 1024;

// dynamic shared memory layout for nb bins
struct MsSmem {
    unsigned long long* buf;    // [MS_TILE] the tile, sorted by bin
    unsigned long long* base;   // [nb] first global slot claimed for the bin
    uint32_t* w;                // [MS_WARPS][nb] per-warp counts, then per-warp offsets
    uint32_t* start;            // [nb] first buffer slot of each bin in the tile

    static size_t bytes(uint32_t nb) { return (size_t)MS_TILE * 8 + (size_t)nb * 8 + (size_t)nb * 4 * (MS_WARPS + 1); }
    __device__ static MsSmem carve(unsigned char* p, uint32_t nb) {
        MsSmem s;
        s.buf = reinterpret_cast<unsigned long long*>(p);
        s.base = s.buf + MS_TILE;
        s.w = reinterpret_cast<uint32_t*>(s.base + nb);
        s.start = s.w + (size_t)MS_WARPS * nb;
        return s;
    }
};

// One tile: elements [e0, e1), element (j, t) = e0 + j*MS_THREADS + t.
// get(e, pair, bin) -> false to skip; bins < nb <= MS_MAXB, nbits =
// ceil(log2 nb).  slot(bin) = {first slot, capacity}; cursor[bin] (global
// u64) counts the bin's slots already claimed.  bin_of(pair) recovers the bin
// when writing out.  Returns true if a bin overflowed (only for inputs that
// break the caller's size contract).  Needs MsSmem::bytes(nb) of dynamic smem.
template <class Get, class BinOf, class Slot>
__device__ __forceinline__ bool ms_tile(Get get, BinOf bin_of, Slot slot, unsigned long long e0,
                                        unsigned long long e1, uint32_t nb, int nbits,
                                        unsigned long long* __restrict__ cursor,
                                        unsigned long long* __restrict__ out, MsSmem& sm) {
    const uint32_t lane = lane_id();
    const int w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    unsigned long long pr[MS_ITEMS];
    uint32_t bn[MS_ITEMS];  // bin, or MS_MAXB for a skipped element
    unsigned peers[MS_ITEMS];
#pragma unroll
    for (int j = 0; j < MS_ITEMS; ++j) {
        const unsigned long long e = e0 + (unsigned long long)j * MS_THREADS + threadIdx.x;
        uint32_t b = 0;
        pr[j] = 0;
        const bool ok = e < e1 && get(e, pr[j], b) && b < nb;
        bn[j] = ok ? b : (uint32_t)MS_MAXB;
    }
    for (uint32_t b = lane; b < nb; b += 32) sm.w[w * nb + b] = 0;
    __syncwarp();
    // per-warp counts
#pragma unroll
    for (int j = 0; j < MS_ITEMS; ++j) {
        peers[j] = __match_any_sync(0xffffffffu, bn[j]);
        if (bn[j] < nb && (peers[j] & lt) == 0) sm.w[w * nb + bn[j]] += __popc(peers[j]);
        __syncwarp();
    }
    __syncthreads();
    // bin totals -> tile-local bin starts, warp offsets, global slots
    uint32_t tot = 0;
    const uint32_t b0 = threadIdx.x * ((nb + MS_THREADS - 1) / MS_THREADS);
    const uint32_t b1 = min(b0 + (nb + MS_THREADS - 1) / MS_THREADS, nb);
    for (uint32_t b = b0; b < b1; ++b) {
        uint32_t acc = 0;
#pragma unroll
        for (int k = 0; k < MS_WARPS; ++k) {
            const uint32_t c = sm.w[k * nb + b];
            sm.w[k * nb + b] = acc;
            acc += c;
        }
        sm.start[b] = acc;  // bin size for now
        sm.base[b] = acc ? atomicAdd(cursor + b, (unsigned long long)acc) : 0ull;
        tot += acc;
    }
    // exclusive scan of the bin sizes (thread-contiguous bin ranges)
    uint32_t incl = tot;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += v;
    }
    __shared__ uint32_t s_warp[MS_WARPS];
    if (lane == 31) s_warp[w] = incl;
    __syncthreads();
    uint32_t wpre = 0;
    for (int k = 0; k < w; ++k) wpre += s_warp[k];
    uint32_t run = wpre + incl - tot;
    for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t c = sm.start[b];
        sm.start[b] = run;
        run += c;
    }
    __syncthreads();
    // rank and place into the sorted tile
#pragma unroll
    for (int j = 0; j < MS_ITEMS; ++j) {
        const bool ok = bn[j] < nb;
        if (ok) sm.buf[sm.start[bn[j]] + sm.w[w * nb + bn[j]] + __popc(peers[j] & lt)] = pr[j];
        __syncwarp();
        if (ok && (peers[j] & lt) == 0) sm.w[w * nb + bn[j]] += __popc(peers[j]);
        __syncwarp();
    }
    __syncthreads();
    // write out, run by run
    uint32_t total = 0;
    for (int k = 0; k < MS_WARPS; ++k) total += s_warp[k];
    bool over = false;
    for (uint32_t i = threadIdx.x; i < total; i += MS_THREADS) {
        const unsigned long long p = sm.buf[i];
        const uint32_t b = bin_of(p);
        const unsigned long long pos = sm.base[b] + (i - sm.start[b]);
        const ulonglong2 sc = slot(b);
        if (pos < sc.y)
            out[sc.x + pos] = p;
        else
            over = true;
    }
    __syncthreads();  // the smem is reused by the next tile
    return over;
}

}  // namespace sg
