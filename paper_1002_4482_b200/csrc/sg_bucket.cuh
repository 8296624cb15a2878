// sg_bucket.cuh -- bucket scatter of 64-bit pairs into bins whose slot ranges
// are known up front (one global cursor per bin, one atomic per bin per tile;
// ranks inside a tile come from shared-memory atomic counters).
// Shared by the ranking's window passes (sg_list.cu) and the edge partition
// (sg_cc.cu).
#pragma once

#include "sg_internal.cuh"

namespace sg {

constexpr int BK_THREADS = 256;
constexpr int BK_ITEMS = 64;
constexpr int BK_TILE = BK_THREADS * BK_ITEMS;
constexpr int BK_MAXB = 2048;

// One tile of a bucket scatter.  get(e, pair, bin, want_pair) yields element
// e's pair and its bin (false: skip); bins are [bin0, bin0 + nb).  slot(bin)
// gives {first slot, capacity} of a bin; cursor[bin] counts slots handed out.
// Returns true if a bin overflowed (only for invalid inputs).
template <class Get, class Slot>
__device__ __forceinline__ bool bucket_tile(Get get, Slot slot, unsigned long long e0, unsigned long long e1,
                                            uint32_t nb, unsigned long long bin0, uint32_t* __restrict__ cursor,
                                            unsigned long long* __restrict__ out) {
    __shared__ uint32_t s_cnt[BK_MAXB];
    __shared__ uint32_t s_base[BK_MAXB];
    for (uint32_t b = threadIdx.x; b < nb; b += BK_THREADS) s_cnt[b] = 0;
    __syncthreads();
    constexpr int U = 4;  // loads of U elements in flight before their counter updates
    for (int j = 0; j < BK_ITEMS; j += U) {
        uint32_t b[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned long long e = e0 + (unsigned long long)(j + u) * BK_THREADS + threadIdx.x;
            unsigned long long pr;
            b[u] = 0;
            ok[u] = e < e1 && get(e, pr, b[u], false) && b[u] < nb;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (ok[u]) atomicAdd(&s_cnt[b[u]], 1u);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nb; b += BK_THREADS) {
        const uint32_t c = s_cnt[b];
        s_base[b] = c ? atomicAdd(cursor + bin0 + b, c) : 0u;
        s_cnt[b] = 0;
    }
    __syncthreads();
    bool over = false;
    for (int j = 0; j < BK_ITEMS; j += U) {
        uint32_t b[U];
        bool ok[U];
        unsigned long long pr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned long long e = e0 + (unsigned long long)(j + u) * BK_THREADS + threadIdx.x;
            b[u] = 0;
            ok[u] = e < e1 && get(e, pr[u], b[u], true) && b[u] < nb;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (ok[u]) {
                const unsigned long long pos = (unsigned long long)s_base[b[u]] + atomicAdd(&s_cnt[b[u]], 1u);
                const ulonglong2 sc = slot(bin0 + b[u]);  // {first slot, capacity}
                if (pos < sc.y)
                    out[sc.x + pos] = pr[u];
                else
                    over = true;
            }
        }
    }
    return over;
}

}  // namespace sg
