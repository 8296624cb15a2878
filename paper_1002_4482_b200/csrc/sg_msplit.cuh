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

#include <stdlib.h>

#include "sg_internal.cuh"

namespace sg {

constexpr int MS_THREADS = 256;
constexpr int MS_WARPS = MS_THREADS / 32;
constexpr int MS_ITEMS = 8;
constexpr int MS_TILE = MS_THREADS * MS_ITEMS;
constexpr int MS_MAXB = 1024;

// peer ranking: 0 match.any, 1 ballots, 2 alternate per item (SG_MS_PEERS)
static __constant__ int g_ms_peers = 1;

// pushes the SG_MS_PEERS switch to the device: once per device and tuning
// generation, and only when it differs from the default
static inline void ms_configure() {
    const Tuning tu = tuning();
    if (tu.ms_peers == 1 && tu.generation == 1) return;
    static thread_local uint32_t done_gen[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || done_gen[dev] == tu.generation) return;
    done_gen[dev] = tu.generation;
    const int v = (int)tu.ms_peers;
    cudaMemcpyToSymbol(g_ms_peers, &v, sizeof(int));
}

// dynamic shared memory layout for nb bins
struct MsSmem {
    unsigned long long* buf;    // [MS_TILE] the tile, sorted by bin
    unsigned long long* base;   // [nb] first global slot claimed for the bin, then the tile -> global delta
    unsigned long long* endp;   // [nb] end of the bin's global slots
    uint32_t* w;                // [MS_WARPS][nb] per-warp counts, then per-warp offsets
    uint32_t* start;            // [nb] first buffer slot of each bin in the tile

    static size_t bytes(uint32_t nb, uint32_t tile = MS_TILE) {
        return (size_t)tile * 8 + (size_t)nb * 16 + (size_t)nb * 4 * (MS_WARPS + 1);
    }
    __device__ static MsSmem carve(unsigned char* p, uint32_t nb, uint32_t tile = MS_TILE) {
        MsSmem s;
        s.buf = reinterpret_cast<unsigned long long*>(p);
        s.base = s.buf + tile;
        s.endp = s.base + nb;
        s.w = reinterpret_cast<uint32_t*>(s.endp + nb);
        s.start = s.w + (size_t)MS_WARPS * nb;
        return s;
    }
};

// The split of one tile already in registers: element j of thread t is
// pr[j] with bin bn[j] (>= nb: skip).  slot(bin) = {first slot, capacity};
// cursor[bin] (global u64) counts the bin's slots already claimed.
// bin_of(pair) recovers the bin when writing out.  Returns true if a bin
// overflowed (only for inputs that break the caller's size contract).
// pair(j) yields element j's value; it is first needed when the tile is
// placed, after the ranking, so a value that waits on a gather can arrive
// while the ballots run.
template <int ITEMS, int NBITS, class PairFn, class BinOf, class Slot>
__device__ __forceinline__ bool ms_split_fn(PairFn pair, const uint32_t (&bn)[ITEMS], BinOf bin_of, Slot slot,
                                            uint32_t nb, unsigned long long* __restrict__ cursor,
                                            unsigned long long* __restrict__ out, MsSmem& sm) {
    const uint32_t lane = lane_id();
    const int w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    uint32_t rk[ITEMS];  // rank among the warp's elements of the same bin
    for (uint32_t b = lane; b < nb; b += 32) sm.w[w * nb + b] = 0;
    __syncwarp();
    // per-warp counts; the leader of each peer group (lanes with equal bins)
    // bumps the warp's counter and hands the old value to its peers
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        // peers: lanes with the same bin
        unsigned peers;
        if (g_ms_peers == 0 || (g_ms_peers == 2 && (j & 1))) {  // 2: alternate, MIO and ALU side by side
            peers = __match_any_sync(0xffffffffu, bn[j]);
        } else {
            // bit-by-bit ballots over the NBITS bin bits (VOTE is an ALU op;
            // match.any queues on MIO).  Bits above nb's width are 0 in every
            // lane and leave the mask unchanged.
            const bool valid = bn[j] < nb;
            const unsigned vb = __ballot_sync(0xffffffffu, valid);
            peers = valid ? vb : ~vb;
#pragma unroll
            for (int k = 0; k < NBITS; ++k) {
                const unsigned b = __ballot_sync(0xffffffffu, (bn[j] >> k) & 1u);
                const unsigned m = 0u - ((bn[j] >> k) & 1u);
                peers &= ~(b ^ m);
            }
        }
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (bn[j] < nb && (int)lane == leader) {
            old = sm.w[w * nb + bn[j]];
            sm.w[w * nb + bn[j]] = old + __popc(peers);
        }
        rk[j] = __shfl_sync(0xffffffffu, old, leader) + __popc(peers & lt);
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
        const ulonglong2 sc = slot(b);
        // global slot of tile position i in bin b: delta + i; valid while < end
        sm.base[b] = sc.x + sm.base[b] - run;
        sm.endp[b] = sc.x + sc.y;
        sm.start[b] = run;
        run += c;
    }
    __syncthreads();
    // place into the sorted tile
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
        if (bn[j] < nb) sm.buf[sm.start[bn[j]] + sm.w[w * nb + bn[j]] + rk[j]] = pair(j);
    __syncthreads();
    // write out, run by run
    uint32_t total = 0;
    for (int k = 0; k < MS_WARPS; ++k) total += s_warp[k];
    bool over = false;
    for (uint32_t i = threadIdx.x; i < total; i += MS_THREADS) {
        const unsigned long long p = sm.buf[i];
        const uint32_t b = bin_of(p);
        const unsigned long long pos = sm.base[b] + i;
        if (pos < sm.endp[b])
            __stcs(out + pos, p);
        else
            over = true;
    }
    __syncthreads();  // the smem is reused by the next tile
    return over;
}

template <int ITEMS, int NBITS, class BinOf, class Slot>
__device__ __forceinline__ bool ms_split(const unsigned long long (&pr)[ITEMS], const uint32_t (&bn)[ITEMS],
                                         BinOf bin_of, Slot slot, uint32_t nb,
                                         unsigned long long* __restrict__ cursor,
                                         unsigned long long* __restrict__ out, MsSmem& sm) {
    return ms_split_fn<ITEMS, NBITS>([&](int j) { return pr[j]; }, bn, bin_of, slot, nb, cursor, out, sm);
}

// One tile: elements [e0, e1), element (j, t) = e0 + j*MS_THREADS + t.
// get(e, pair, bin) -> false to skip; bins < nb <= MS_MAXB.  Needs
// MsSmem::bytes(nb) of dynamic smem.
template <class Get, class BinOf, class Slot>
__device__ __forceinline__ bool ms_tile(Get get, BinOf bin_of, Slot slot, unsigned long long e0,
                                        unsigned long long e1, uint32_t nb, int nbits,
                                        unsigned long long* __restrict__ cursor,
                                        unsigned long long* __restrict__ out, MsSmem& sm) {
    (void)nbits;
    unsigned long long pr[MS_ITEMS];
    uint32_t bn[MS_ITEMS];
#pragma unroll
    for (int j = 0; j < MS_ITEMS; ++j) {
        const unsigned long long e = e0 + (unsigned long long)j * MS_THREADS + threadIdx.x;
        uint32_t b = 0;
        pr[j] = 0;
        const bool ok = e < e1 && get(e, pr[j], b) && b < nb;
        bn[j] = ok ? b : (uint32_t)MS_MAXB;
    }
    return ms_split<MS_ITEMS, 10>(pr, bn, bin_of, slot, nb, cursor, out, sm);
}

// ---------------------------------------------------------------------------
// TMA bulk staging: a persistent CTA streams its next input tile into shared
// memory (cp.async.bulk, completion on an mbarrier) while it splits the
// current one, so the loads never stall the sort.
constexpr int MS2_ITEMS = 16;
constexpr int MS2_TILE = MS_THREADS * MS2_ITEMS;  // 4096 elements

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// bytes: multiple of 16, src/dst 16-B aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// L2 eviction policies: streams that are read or written once go first, small
// gather tables that the streams would otherwise flush out of L2 go last
__device__ __forceinline__ unsigned long long l2_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, unsigned long long* bar,
                                              unsigned long long pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ uint32_t ld_hint(const uint32_t* p, unsigned long long pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "SG_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra SG_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

}  // namespace sg
