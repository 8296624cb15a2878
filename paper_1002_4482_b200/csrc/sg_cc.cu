// sg_cc.cu -- connected components on sm_100a.
//
// Reference: concomp.sv_components (concomp.py:208-246), Shiloach-Vishkin
// with six kernels per round over a doubly-stored edge list.  Here the
// stored edge list (each undirected edge once, core.py:97-110) is streamed
// as (u,v) u32 pairs and both orientations are handled in registers.
//
// Invariant for every variant: D[i] <= i and D[i] is connected to i.  A root
// is therefore the minimum of its tree, and after the final shortcut the
// labels are the component minima -- bit-identical to the reference's
// canonical labels (core.py:240-257) with no relabel pass.
//
//  * SG_CC_UF (default): one hook sweep.  Each edge finds both roots with
//    path halving and hooks the larger root under the smaller one with a CAS
//    that only succeeds on a root (ECL-CC style lock-free union-find).
//    Every edge has been united when the sweep ends, so one sweep + one
//    shortcut sweep is the whole algorithm (rounds = 1).
//  * SG_CC_SV: synchronous min-hook rounds.  Hook: for an edge whose
//    endpoints sit in different stars, atomicMin(D[larger root], smaller
//    root) (conditional hooking, concomp.py:136-154).  Shortcut: every
//    vertex chases its root (one sweep reaches stars; concomp.py:88-103).
//    Rounds repeat until a hook sweep changes nothing (the converge-OR of
//    sv5, concomp.py:183-205).  Hooks only lower parents (min-monotone), so
//    per-GPU proposals merge exactly with a min all-reduce (multi-GPU path).
#include <stdlib.h>
#include <string.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "sg_internal.cuh"
#include "sg_msplit.cuh"

namespace sg {

constexpr int HOOK_THREADS = 256;
constexpr int COMP_THREADS = 256;

// ---------------------------------------------------------------------------
// edge views: pair i -> (u, v) widened so that negative / >= n endpoints fail
// the range check

struct EdgesU32 {
    static constexpr uint32_t kBytes = 8;
    const uint2* e;
    __device__ static void decode(const void* p, uint32_t i, unsigned long long& u, unsigned long long& v) {
        const uint2 x = reinterpret_cast<const uint2*>(p)[i];
        u = x.x;
        v = x.y;
    }
    __device__ __forceinline__ void load(unsigned long long i, unsigned long long& u, unsigned long long& v) const {
        const uint2 x = __ldcs(e + i);
        u = x.x;
        v = x.y;
    }
};
struct EdgesI32 {
    static constexpr uint32_t kBytes = 8;
    const int2* e;
    __device__ static void decode(const void* p, uint32_t i, unsigned long long& u, unsigned long long& v) {
        const int2 x = reinterpret_cast<const int2*>(p)[i];
        u = (unsigned long long)(long long)x.x;
        v = (unsigned long long)(long long)x.y;
    }
    __device__ __forceinline__ void load(unsigned long long i, unsigned long long& u, unsigned long long& v) const {
        const int2 x = __ldcs(e + i);
        u = (unsigned long long)(long long)x.x;
        v = (unsigned long long)(long long)x.y;
    }
};
struct EdgesI64 {
    static constexpr uint32_t kBytes = 16;
    const longlong2* e;
    __device__ static void decode(const void* p, uint32_t i, unsigned long long& u, unsigned long long& v) {
        const longlong2 x = reinterpret_cast<const longlong2*>(p)[i];
        u = (unsigned long long)x.x;
        v = (unsigned long long)x.y;
    }
    __device__ __forceinline__ void load(unsigned long long i, unsigned long long& u, unsigned long long& v) const {
        const longlong2 x = __ldcs(e + i);
        u = (unsigned long long)x.x;
        v = (unsigned long long)x.y;
    }
};

// flags layout (device, u64): [0] changed, [1] ~first out-of-range row,
// [2] ~first self-loop row (0 = none; atomicMax of ~row keeps the minimum row)
__device__ __forceinline__ bool edge_ok(unsigned long long u, unsigned long long v, unsigned long long n,
                                        unsigned long long row, unsigned long long* flags) {
    if (u >= n || v >= n) {
        atomicMax(flags + 1, ~row);
        return false;
    }
    if (u == v) {
        atomicMax(flags + 2, ~row);
        return false;
    }
    return true;
}

// ---------------------------------------------------------------------------
// union-find hook

// root of x given p = D[x]; halves the path on the way (benign races: only
// ever writes an ancestor, never touches a root)
//
// Parent reads go through L1: a stale value is still an ancestor (pointers
// only ever move up), so finds stay correct; the CAS below is L2-coherent and
// returns the true parent when a stale root was hooked meanwhile.  Reading
// through L2 only would funnel every find of the giant component into the one
// L2 sector that holds its root.
__device__ __forceinline__ uint32_t ld_parent(const uint32_t* p) { return *p; }

__device__ __forceinline__ uint32_t find_from(uint32_t* D, uint32_t x, uint32_t p) {
    while (p != x) {
        const uint32_t gp = ld_parent(D + p);
        if (gp == p) return p;
        D[x] = gp;
        x = gp;
        p = ld_parent(D + x);
    }
    return x;
}

__device__ __forceinline__ bool unite(uint32_t* D, uint32_t u, uint32_t pu, uint32_t v, uint32_t pv) {
    uint32_t ru = find_from(D, u, pu);
    uint32_t rv = find_from(D, v, pv);
    while (ru != rv) {
        const uint32_t hi = ru > rv ? ru : rv;
        const uint32_t lo = ru > rv ? rv : ru;
        const uint32_t old = atomicCAS(D + hi, hi, lo);
        if (old == hi) return true;
        // hi was hooked by someone else: continue from its new tree
        ru = find_from(D, old, ld_parent(D + old));
        rv = lo;
    }
    return false;
}

template <class E, bool kValidate>
__global__ void __launch_bounds__(HOOK_THREADS) k_cc_hook_uf(E edges, unsigned long long m, unsigned long long row0,
                                                             unsigned long long n, uint32_t* D,
                                                             unsigned long long* flags,
                                                             const unsigned long long* rng) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    bool any = false;
    unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (rng != nullptr) {  // partition [rng[0], rng[1]) of a partitioned edge list
        i += rng[0];
        m = rng[1];
    }
    // HU edges per iteration: 2*HU independent parent loads in flight (2 beats 4 and 8:
    // fewer unions racing for the same roots, measured)
#ifndef CC_HOOK_HU
#define CC_HOOK_HU 2
#endif
    constexpr int HU = CC_HOOK_HU;
    for (; i + (HU - 1) * stride < m; i += HU * stride) {
        unsigned long long u[HU], v[HU];
        bool ok[HU];
#pragma unroll
        for (int k = 0; k < HU; ++k) edges.load(i + k * stride, u[k], v[k]);
#pragma unroll
        for (int k = 0; k < HU; ++k) ok[k] = !kValidate || edge_ok(u[k], v[k], n, row0 + i + k * stride, flags);
        uint32_t pu[HU], pv[HU];
#pragma unroll
        for (int k = 0; k < HU; ++k) {
            pu[k] = ok[k] ? ld_parent(D + u[k]) : 0;
            pv[k] = ok[k] ? ld_parent(D + v[k]) : 0;
        }
#pragma unroll
        for (int k = 0; k < HU; ++k)
            if (ok[k] && pu[k] != pv[k]) any |= unite(D, (uint32_t)u[k], pu[k], (uint32_t)v[k], pv[k]);
    }
    for (; i < m; i += stride) {
        unsigned long long u, v;
        edges.load(i, u, v);
        if (!kValidate || edge_ok(u, v, n, row0 + i, flags)) {
            const uint32_t pu = ld_parent(D + u), pv = ld_parent(D + v);
            if (pu != pv) any |= unite(D, (uint32_t)u, pu, (uint32_t)v, pv);
        }
    }
    if (__any_sync(0xffffffffu, any) && lane_id() == 0) flags[0] = 1ull;
}

// ---------------------------------------------------------------------------
// synchronous SV min-hook

template <class E, bool kValidate>
__global__ void __launch_bounds__(HOOK_THREADS) k_cc_hook_sv(E edges, unsigned long long m, unsigned long long row0,
                                                             unsigned long long n, uint32_t* D,
                                                             unsigned long long* flags,
                                                             const unsigned long long* rng) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    bool any = false;
    unsigned long long i0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (rng != nullptr) {
        i0 += rng[0];
        m = rng[1];
    }
    for (unsigned long long i = i0; i < m; i += stride) {
        unsigned long long u, v;
        edges.load(i, u, v);
        if (kValidate && !edge_ok(u, v, n, row0 + i, flags)) continue;
        const uint32_t du = ld_parent(D + u), dv = ld_parent(D + v);
        if (du != dv) {
            const uint32_t hi = du > dv ? du : dv;
            const uint32_t lo = du > dv ? dv : du;
            if (atomicMin(D + hi, lo) > lo) any = true;
        }
    }
    if (__any_sync(0xffffffffu, any) && lane_id() == 0) flags[0] = 1ull;
}

// ---------------------------------------------------------------------------
// init / shortcut / labels

__global__ void __launch_bounds__(COMP_THREADS) k_cc_init(uint32_t* D, unsigned long long n) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        D[i] = (uint32_t)i;
}

// D[i] = root(i) for i in [lo, hi); counts roots; optionally writes labels
template <class OutT>
__global__ void __launch_bounds__(COMP_THREADS) k_cc_compress(uint32_t* D, unsigned long long lo, unsigned long long hi,
                                                              unsigned long long* roots, OutT* out) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    uint32_t nroots = 0;
    for (unsigned long long i = lo + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += stride) {
        uint32_t r = ld_parent(D + i);
        if (r == (uint32_t)i) {
            ++nroots;
        } else {
            for (;;) {
                const uint32_t p = ld_parent(D + r);  // roots do not move during the shortcut
                if (p == r) break;
                r = p;
            }
            __stcg(D + i, r);
        }
        if (out != nullptr) out[i] = (OutT)r;
    }
    for (int o = 16; o > 0; o >>= 1) nroots += __shfl_xor_sync(0xffffffffu, nroots, o);
    if (lane_id() == 0 && nroots && roots != nullptr) atomicAdd(roots, (unsigned long long)nroots);
}

// the same over four consecutive vertices per thread (16-B loads and stores
// of D, four root chases in flight per thread); [lo, hi) starts 16-B aligned.
// C5: 0.161 -> 0.089 ms (SG_CC_COMP4=1, default; pass x8)
template <class OutT>
__global__ void __launch_bounds__(COMP_THREADS) k_cc_compress4(uint32_t* D, unsigned long long lo,
                                                               unsigned long long hi, unsigned long long* roots,
                                                               OutT* out) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long t0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long nq = (hi - lo) >> 2;
    uint4* D4 = reinterpret_cast<uint4*>(D + lo);
    uint32_t nroots = 0;
    for (unsigned long long q = t0; q < nq; q += stride) {
        const uint4 p = D4[q];
        const uint32_t i0 = (uint32_t)(lo + 4 * q);
        uint32_t r[4] = {p.x, p.y, p.z, p.w};
        bool live[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            live[j] = r[j] != i0 + (uint32_t)j;
            nroots += live[j] ? 0u : 1u;
        }
        for (;;) {  // roots do not move during the shortcut
            bool any = false;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (live[j]) {
                    const uint32_t pp = ld_parent(D + r[j]);
                    if (pp == r[j])
                        live[j] = false;
                    else
                        r[j] = pp;
                }
                any |= live[j];
            }
            if (!any) break;
        }
        if (r[0] != p.x || r[1] != p.y || r[2] != p.z || r[3] != p.w) __stcg(D4 + q, make_uint4(r[0], r[1], r[2], r[3]));
        if (out != nullptr) {
#pragma unroll
            for (int j = 0; j < 4; ++j) out[lo + 4 * q + j] = (OutT)r[j];
        }
    }
    for (unsigned long long i = lo + 4 * nq + t0; i < hi; i += stride) {  // the < 4 trailing vertices
        uint32_t r = ld_parent(D + i);
        if (r == (uint32_t)i) {
            ++nroots;
        } else {
            for (;;) {
                const uint32_t pp = ld_parent(D + r);
                if (pp == r) break;
                r = pp;
            }
            __stcg(D + i, r);
        }
        if (out != nullptr) out[i] = (OutT)r;
    }
    for (int o = 16; o > 0; o >>= 1) nroots += __shfl_xor_sync(0xffffffffu, nroots, o);
    if (lane_id() == 0 && nroots && roots != nullptr) atomicAdd(roots, (unsigned long long)nroots);
}

template <class OutT>
__global__ void __launch_bounds__(COMP_THREADS) k_cc_labels(const uint32_t* __restrict__ D, unsigned long long n,
                                                            OutT* __restrict__ out) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (OutT)D[i];
}

// ---------------------------------------------------------------------------
// Stable partition of the edge list by the window of its larger endpoint.
//
// Stored rows are (u, v) with the random endpoint v (gen.py:215-217 sorts by
// u), so the parent gathers D[v] scatter over all of D -- 256 MiB at n = 2^26,
// twice the L2.  Hooking one window of v at a time keeps those gathers (and
// the CAS / path-halving writes they lead to) in an L2-resident slice of D,
// while D[u] and the edges stream.  Invalid rows are reported (first
// offending original row, core.py:196-206) and dropped here.

constexpr int PART_THREADS = 256;
constexpr int PART_ITEMS = 16;
constexpr int PART_TILE = PART_THREADS * PART_ITEMS;
constexpr int MAX_PARTS = 16;

template <class E>
__device__ __forceinline__ int part_of(E edges, unsigned long long e, unsigned long long m, unsigned long long n,
                                       uint32_t shift, unsigned long long* flags, bool validate, uint2& uv) {
    if (e >= m) return -1;
    unsigned long long u, v;
    edges.load(e, u, v);
    if (u >= n || v >= n) {
        if (validate) atomicMax(flags + 1, ~e);
        return -1;
    }
    if (u == v) {
        if (validate) atomicMax(flags + 2, ~e);
        return -1;
    }
    uv = make_uint2((uint32_t)u, (uint32_t)v);
    return (int)((u > v ? u : v) >> shift);
}

// partition sizes: persistent CTAs; per 32 edges a warp takes five ballots
// (valid + 4 partition bits) and lane p keeps partition p's count in a
// register; one atomic per partition per CTA at the end.  Validates rows.
// NB = ceil(log2 P) partition bits (ballots per edge); kNarrow: 32-bit ids
// (u32 edges, or int32 edges with n <= 2^31, where a negative id reads as
// >= 2^31 >= n), so the checks run in 32-bit
template <class E, int NB, bool kNarrow>
__global__ void __launch_bounds__(PART_THREADS) k_cc_part_count(E edges, unsigned long long m, unsigned long long n,
                                                                unsigned long long row0,
                                                                uint32_t shift, int P,
                                                                unsigned long long* __restrict__ totals,
                                                                unsigned long long* flags) {
    __shared__ unsigned long long s_cnt[MAX_PARTS];
    if (threadIdx.x < MAX_PARTS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t lane = lane_id();
    unsigned long long mine = 0;  // edges of partition `lane` seen by this warp
    const unsigned long long ntiles = (m + PART_TILE - 1) / PART_TILE;
    constexpr int H = PART_ITEMS / 2;  // half a tile in flight: fewer registers, more resident warps
    for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
            const unsigned long long e0 = tile * PART_TILE + (unsigned long long)half * H * PART_THREADS + threadIdx.x;
            unsigned long long uu[H], vv[H];
#pragma unroll
            for (int j = 0; j < H; ++j) {  // all loads in flight before any validation atomic
                const unsigned long long e = e0 + (unsigned long long)j * PART_THREADS;
                uu[j] = n;
                vv[j] = n;
                if (e < m) edges.load(e, uu[j], vv[j]);
            }
#pragma unroll
            for (int j = 0; j < H; ++j) {
                const unsigned long long e = e0 + (unsigned long long)j * PART_THREADS;
                bool ok = false;
                if (e < m) {
                    const bool oob = kNarrow ? ((uint32_t)uu[j] >= (uint32_t)n || (uint32_t)vv[j] >= (uint32_t)n)
                                             : (uu[j] >= n || vv[j] >= n);
                    if (oob)
                        atomicMax(flags + 1, ~(row0 + e));
                    else if ((uint32_t)uu[j] == (uint32_t)vv[j])
                        atomicMax(flags + 2, ~(row0 + e));
                    else
                        ok = true;
                }
                // valid ids fit 32 bits (n < 2^32): the partition math runs in 32-bit
                const uint32_t p = max((uint32_t)uu[j], (uint32_t)vv[j]) >> shift;
                unsigned msk = __ballot_sync(0xffffffffu, ok);
#pragma unroll
                for (int k = 0; k < NB; ++k) {
                    const unsigned b = __ballot_sync(0xffffffffu, (p >> k) & 1u);
                    msk &= ((lane >> k) & 1u) ? b : ~b;
                }
                mine += __popc(msk);
            }
        }
    }
    if (lane < (uint32_t)P && mine) atomicAdd(&s_cnt[lane], mine);
    __syncthreads();
    if (threadIdx.x < (uint32_t)P && s_cnt[threadIdx.x]) atomicAdd(totals + threadIdx.x, s_cnt[threadIdx.x]);
}

// off_part = exclusive prefix of the P totals (off_part[P] = valid edges)
__global__ void k_cc_part_offsets(const unsigned long long* __restrict__ totals, int P,
                                  unsigned long long* __restrict__ off_part) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned long long acc = 0;
        for (int p = 0; p < P; ++p) {
            off_part[p] = acc;
            acc += totals[p];
        }
        off_part[P] = acc;
    }
}

// Scatter every valid edge into its partition (block multisplit,
// sg_msplit.cuh; one global atomic per partition per 4096-edge tile).
template <class E>
__global__ void __launch_bounds__(MS_THREADS, 4) k_cc_part_scatter(E edges, unsigned long long m, unsigned long long n,
                                                                uint32_t shift, int P,
                                                                const unsigned long long* __restrict__ off_part,
                                                                unsigned long long* __restrict__ cursor,
                                                                uint2* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char ms_raw[];
    MsSmem sm = MsSmem::carve(ms_raw, (uint32_t)P);
    int nbits = 0;
    while ((1 << nbits) < P) ++nbits;
    auto get = [&](unsigned long long e, unsigned long long& pr, uint32_t& b) -> bool {
        uint2 uv;
        const int p = part_of(edges, e, m, n, shift, nullptr, false, uv);
        if (p < 0) return false;
        pr = ((unsigned long long)uv.y << 32) | uv.x;
        b = (uint32_t)p;
        return true;
    };
    auto bin_of = [&](unsigned long long pr) {
        const uint32_t u = (uint32_t)pr, v = (uint32_t)(pr >> 32);
        return (u > v ? u : v) >> shift;
    };
    auto slot = [&](uint32_t b) { return make_ulonglong2(off_part[b], off_part[b + 1] - off_part[b]); };
    for (unsigned long long e0 = (unsigned long long)blockIdx.x * MS_TILE; e0 < m;
         e0 += (unsigned long long)gridDim.x * MS_TILE)
        ms_tile(get, bin_of, slot, e0, min(e0 + MS_TILE, m), (uint32_t)P, nbits, cursor,
                reinterpret_cast<unsigned long long*>(out), sm);
}

// TMA-staged scatter (persistent, 2 CTAs per SM): the next 4096-edge tile
// streams into shared memory while the current one is split.
constexpr int PART2_CTAS_PER_SM = 2;

template <class E, int NB, bool kNarrow>  // kNarrow: as in k_cc_part_count
__global__ void __launch_bounds__(MS_THREADS, PART2_CTAS_PER_SM) k_cc_part_scatter2(
    E edges, unsigned long long m, unsigned long long n, uint32_t shift, int P,
    const unsigned long long* __restrict__ off_part, unsigned long long* __restrict__ cursor, uint2* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char ms_raw[];
    unsigned char* stage = ms_raw;
    MsSmem sm = MsSmem::carve(ms_raw + MS2_TILE * E::kBytes, (uint32_t)P, MS2_TILE);
    __shared__ unsigned long long bar;
    const unsigned long long ntiles = (m + MS2_TILE - 1) / MS2_TILE;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    auto issue = [&](unsigned long long tile) {
        if (threadIdx.x == 0 && tile < ntiles) {
            const unsigned long long e0 = tile * MS2_TILE;
            const uint32_t cnt = (uint32_t)min((unsigned long long)MS2_TILE, m - e0);
            const uint32_t full = cnt * E::kBytes & ~15u;  // whole 16-B units by bulk copy, the rest below
            if (full) {
                mbar_expect_tx(&bar, full);
                bulk_g2s(stage, reinterpret_cast<const unsigned char*>(edges.e) + e0 * E::kBytes, full, &bar);
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
            }
        }
    };
    auto bin_of = [&](unsigned long long pr) {
        const uint32_t u = (uint32_t)pr, v = (uint32_t)(pr >> 32);
        return (u > v ? u : v) >> shift;
    };
    auto slot = [&](uint32_t b) { return make_ulonglong2(off_part[b], off_part[b + 1] - off_part[b]); };
    uint32_t phase = 0;
    issue(blockIdx.x);
    for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const unsigned long long e0 = tile * MS2_TILE;
        const uint32_t cnt = (uint32_t)min((unsigned long long)MS2_TILE, m - e0);
        const uint32_t staged = (cnt * E::kBytes & ~15u) / E::kBytes;
        mbar_wait(&bar, phase);
        phase ^= 1u;
        unsigned long long pr[MS2_ITEMS];
        uint32_t bn[MS2_ITEMS];
#pragma unroll
        for (int j = 0; j < MS2_ITEMS; ++j) {
            const uint32_t e = j * MS_THREADS + threadIdx.x;
            unsigned long long u = n, v = n;
            if (e < staged)
                E::decode(stage, e, u, v);
            else if (e < cnt)
                edges.load(e0 + e, u, v);  // the odd tail element of the last tile
            const bool ok = kNarrow ? ((uint32_t)u < (uint32_t)n && (uint32_t)v < (uint32_t)n && (uint32_t)u != (uint32_t)v)
                                    : (u < n && v < n && u != v);
            pr[j] = ((unsigned long long)(uint32_t)v << 32) | (uint32_t)u;
            bn[j] = ok ? max((uint32_t)u, (uint32_t)v) >> shift : (uint32_t)MS_MAXB;
        }
        __syncthreads();  // staging consumed: refill it behind the split
        issue(tile + gridDim.x);
        ms_split<MS2_ITEMS, NB>(pr, bn, bin_of, slot, (uint32_t)P, cursor, reinterpret_cast<unsigned long long*>(out), sm);
    }
}

// ---------------------------------------------------------------------------
// One-pass partition into per-window chunk lists.
//
// Every edge is read once and written once, with no count pass and no
// shared-memory sort.  Each CTA keeps, per window, a reservation counter in
// shared memory over its own stream of chunks (CC_CHUNK rows, 8 KiB each).
// Per 32 edges a warp groups its lanes by window (one match.any, kMatch, the
// default; or NB + 1 ballots) and each group's leader reserves the group's
// rows with one shared atomic.  Chunk k + 1 of a window is claimed from a
// global bump allocator when chunk k starts filling (its id published in a
// shared-memory ring and in the CTA's chunk list), so a writer never waits on
// a claim's atomic; chunk k joins the window's directory when its first row
// is reserved.  Every lane then stores its edge straight into its chunk -- a
// warp's stores are at most P contiguous runs.  No barriers inside the loop:
// warps stream independently.  The identity forest D[i] = i (cc_init) is
// written by the same launch.
// At the end each CTA pads its open chunks with (0, 0) rows, which the hook
// skips (equal parents), so a window is a whole number of chunks and the
// hook walks its directory as one virtual contiguous range (EdgesChunked).
//
// The edge order inside a window is the claim order of the chunks: the warps
// walk 64-row groups grid-stride, so it is the input order up to the ~grid x
// 64 x warps rows in flight and the D[u] side of the hook stays a streaming
// window of D.  (A tile-local sort written back in place, r02a/b, left
// ~65k short slices per window for the hook and lost 1.1 ms there:
// profiles/r02_cc_partition.txt.)
constexpr int CC_CHUNK_BITS = 10;
constexpr uint32_t CC_CHUNK = 1u << CC_CHUNK_BITS;
constexpr int PD_THREADS = 256;
#ifndef CC_PD_CTAS
#define CC_PD_CTAS 5
#endif
#ifndef CC_PD_G16
#define CC_PD_G16 4
#endif
constexpr int PD_CTAS_PER_SM = CC_PD_CTAS;
constexpr uint32_t PD_RING = 16;  // chunk ids of the last PD_RING chunks per window, in shared memory
// 64-row groups per warp iteration: 4 rows per lane in flight (8 rows with 4
// CTAs per SM measured slower: 1.60 vs 1.09 ms at C5)
constexpr int PD_GROUPS = 2;

struct EdgesChunked {
    static constexpr uint32_t kBytes = 8;
    const uint2* e;       // chunk c = rows [c*CC_CHUNK, (c+1)*CC_CHUNK)
    const uint32_t* dir;  // the window's chunk ids in claim order
    __device__ __forceinline__ void load(unsigned long long i, unsigned long long& u, unsigned long long& v) const {
        const uint32_t c = __ldg(dir + (i >> CC_CHUNK_BITS));
        const uint2 x = __ldcs(e + (((unsigned long long)c << CC_CHUNK_BITS) | (i & (CC_CHUNK - 1))));
        u = x.x;
        v = x.y;
    }
};

template <class E, int NB, bool kNarrow, bool kMatch, bool kV16 = false>
__global__ void __launch_bounds__(PD_THREADS, PD_CTAS_PER_SM) k_cc_part_chunks(
    E edges, unsigned long long m, unsigned long long n, unsigned long long row0, uint32_t shift, int P,
    uint2* __restrict__ out, uint32_t* __restrict__ dir, unsigned long long dir_stride,
    uint32_t* __restrict__ counts /* [MAX_PARTS] chunks per window, [MAX_PARTS] chunks claimed */,
    uint32_t* __restrict__ cta_list /* [grid][P][kmax] the CTA's chunks per window */, uint32_t kmax,
    unsigned long long* flags, uint32_t* __restrict__ Dinit, unsigned long long ninit) {
    __shared__ uint32_t s_fill[MAX_PARTS];
    __shared__ unsigned long long s_ring[MAX_PARTS][PD_RING];  // (k + 1) << 32 | chunk id
    const uint32_t lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    uint32_t* my_list = cta_list + (size_t)blockIdx.x * P * kmax;
    for (uint32_t i = threadIdx.x; i < MAX_PARTS * PD_RING; i += PD_THREADS) (&s_ring[0][0])[i] = 0ull;
    if (Dinit != nullptr) {  // the identity forest D[i] = i (cc_init), streamed out beside the partition
        const unsigned long long gt = (unsigned long long)blockIdx.x * PD_THREADS + threadIdx.x;
        const unsigned long long nt = (unsigned long long)gridDim.x * PD_THREADS;
        uint4* D4 = reinterpret_cast<uint4*>(Dinit);
        for (unsigned long long q = gt; q < ninit / 4; q += nt) {
            const uint32_t b = (uint32_t)(q * 4);
            __stcs(D4 + q, make_uint4(b, b + 1, b + 2, b + 3));
        }
        if (gt < (ninit & 3)) Dinit[(ninit & ~3ull) + gt] = (uint32_t)((ninit & ~3ull) + gt);
    }
    __syncthreads();
    // chunk k + 1 of a window is claimed when chunk k starts filling, so a
    // writer finds its chunk id already published (no wait on the claim's
    // atomic); chunk 0 is claimed here
    auto preclaim = [&](uint32_t w, uint32_t k) {
        const uint32_t c = atomicAdd(counts + MAX_PARTS, 1u);
        my_list[w * kmax + k] = c;
        __threadfence_block();
        *reinterpret_cast<volatile unsigned long long*>(&s_ring[w][k % PD_RING]) =
            ((unsigned long long)(k + 1) << 32) | c;
    };
    if (threadIdx.x < (uint32_t)P) {
        s_fill[threadIdx.x] = 0;
        preclaim(threadIdx.x, 0);
    }
    __syncthreads();
    auto chunk_of = [&](uint32_t w, uint32_t k) -> uint32_t {
        const volatile unsigned long long* slot = &s_ring[w][k % PD_RING];
        for (;;) {  // published when chunk k - 1 started: at most a short wait
            const unsigned long long x = *slot;
            const uint32_t tag = (uint32_t)(x >> 32);
            if (tag == k + 1) return (uint32_t)x;
            if (tag > k + 1) return *reinterpret_cast<volatile uint32_t*>(my_list + w * kmax + k);  // slot reused
        }
    };
    // chunk k of window w takes its first row: it joins the window's directory
    // (the hook's order) and chunk k + 1 is claimed
    auto activate = [&](uint32_t w, uint32_t k) {
        const uint32_t c = chunk_of(w, k);
        const uint32_t d = atomicAdd(counts + w, 1u);
        dir[w * dir_stride + d] = c;
        preclaim(w, k + 1);
    };
    // invalid rows (range / self-loop, core.py:196-206) are flagged off the fast path
    auto flag_bad = [&](unsigned long long e, unsigned long long u, unsigned long long v) {
        const bool oob = kNarrow ? ((uint32_t)u >= (uint32_t)n || (uint32_t)v >= (uint32_t)n) : (u >= n || v >= n);
        if (oob)
            atomicMax(flags + 1, ~(row0 + e));
        else if ((uint32_t)u == (uint32_t)v)
            atomicMax(flags + 2, ~(row0 + e));
    };
    const uint32_t n32 = (uint32_t)min(n, 0xFFFFFFFFull);
    // ok: valid row (range and self-loop checks done by the caller for four rows at once)
    auto place = [&](bool ok, unsigned long long u, unsigned long long v) {
        const uint32_t b = ok ? max((uint32_t)u, (uint32_t)v) >> shift : 0xFFFFFFFFu;
        uint32_t base = 0, q = 0;
        if (kMatch) {
            // peers by match.any; the group leader reserves the group's rows with one shared atomic
            const unsigned peers = __match_any_sync(0xffffffffu, b);
            const int leader = __ffs(peers) - 1;
            if (ok && (int)lane == leader) {
                const uint32_t cnt = __popc(peers);
                base = atomicAdd(&s_fill[b], cnt);
                if ((base & (CC_CHUNK - 1)) == 0)
                    activate(b, base >> CC_CHUNK_BITS);
                else if (((base + cnt - 1) >> CC_CHUNK_BITS) != (base >> CC_CHUNK_BITS))
                    activate(b, (base + cnt - 1) >> CC_CHUNK_BITS);
            }
            q = __shfl_sync(0xffffffffu, base, leader) + __popc(peers & lt);
        } else {
            // peers by NB + 1 ballots; lane w reserves window w's rows
            const unsigned vb = __ballot_sync(0xffffffffu, ok);
            unsigned peers = vb, mine = vb;  // peers: lanes of my window; mine: lanes of window `lane`
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                const unsigned bk = __ballot_sync(0xffffffffu, (b >> k) & 1u);
                peers &= ((b >> k) & 1u) ? bk : ~bk;
                mine &= ((lane >> k) & 1u) ? bk : ~bk;
            }
            const uint32_t cnt = lane < (uint32_t)P ? __popc(mine) : 0u;
            if (cnt) {
                base = atomicAdd(&s_fill[lane], cnt);
                if ((base & (CC_CHUNK - 1)) == 0)
                    activate(lane, base >> CC_CHUNK_BITS);
                else if (((base + cnt - 1) >> CC_CHUNK_BITS) != (base >> CC_CHUNK_BITS))
                    activate(lane, (base + cnt - 1) >> CC_CHUNK_BITS);
            }
            q = __shfl_sync(0xffffffffu, base, b & 31u) + __popc(peers & lt);
        }
        if (ok) {
            const uint32_t k = q >> CC_CHUNK_BITS;
            const unsigned long long x = *reinterpret_cast<volatile unsigned long long*>(&s_ring[b][k % PD_RING]);
            const uint32_t c = (uint32_t)(x >> 32) == k + 1 ? (uint32_t)x : chunk_of(b, k);
            __stcs(out + (((unsigned long long)c << CC_CHUNK_BITS) | (q & (CC_CHUNK - 1))),
                   make_uint2((uint32_t)u, (uint32_t)v));
        }
    };
    // warps take 64-row groups grid-stride, G groups (2 G rows per lane) in flight.
    // kV16 (8-B rows, 16-B aligned): a lane loads rows 2l, 2l + 1 of a group
    // with one 16-B load, so four groups (eight rows, 64 B per lane) are in
    // flight for the registers the 8-B path spends on two
    constexpr int G = kV16 ? CC_PD_G16 : PD_GROUPS;
    constexpr int RL = 2 * G;
    const unsigned long long nw = (unsigned long long)gridDim.x * (PD_THREADS / 32);
    const unsigned long long ng = (m + 63) / 64;
    for (unsigned long long g = (unsigned long long)blockIdx.x * (PD_THREADS / 32) + (threadIdx.x >> 5); g < ng;
         g += G * nw) {
        unsigned long long ee[RL], uu[RL], vv[RL];
        bool ok[RL], any_bad = false;
        if (kV16) {
#pragma unroll
            for (int k = 0; k < G; ++k) {
                const unsigned long long r = (g + k * nw) * 64 + 2 * lane;
                ee[2 * k] = r;
                ee[2 * k + 1] = r + 1;
                uu[2 * k] = vv[2 * k] = uu[2 * k + 1] = vv[2 * k + 1] = n;
                if (r + 1 < m) {
                    const uint4 x = __ldcs(reinterpret_cast<const uint4*>(edges.e) + (r >> 1));
                    uu[2 * k] = x.x;
                    vv[2 * k] = x.y;
                    uu[2 * k + 1] = x.z;
                    vv[2 * k + 1] = x.w;
                } else if (r < m) {
                    edges.load(r, uu[2 * k], vv[2 * k]);
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < RL; ++j) {
                ee[j] = (g + (j >> 1) * nw) * 64 + (j & 1) * 32 + lane;
                uu[j] = n;
                vv[j] = n;
                if (ee[j] < m) edges.load(ee[j], uu[j], vv[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < RL; ++j) {
            const bool in = ee[j] < m;
            ok[j] = in && (kNarrow ? ((uint32_t)uu[j] < n32 && (uint32_t)vv[j] < n32) : (uu[j] < n && vv[j] < n)) &&
                    (uint32_t)uu[j] != (uint32_t)vv[j];
            any_bad |= in && !ok[j];
        }
        if (__any_sync(0xffffffffu, any_bad)) {  // invalid rows are flagged off the fast path
#pragma unroll
            for (int j = 0; j < RL; ++j)
                if (ee[j] < m && !ok[j]) flag_bad(ee[j], uu[j], vv[j]);
        }
#pragma unroll
        for (int j = 0; j < RL; ++j) place(ok[j], uu[j], vv[j]);
    }
    __syncthreads();
    // pad the open chunks with (0, 0) rows: the hook skips them (equal parents)
    for (int w = 0; w < P; ++w) {
        const uint32_t tot = s_fill[w], r = tot & (CC_CHUNK - 1);
        if (r == 0) continue;  // (chunk tot >> CC_CHUNK_BITS was only pre-claimed: not in the directory)
        const uint32_t c = *reinterpret_cast<volatile uint32_t*>(my_list + w * kmax + (tot >> CC_CHUNK_BITS));
        for (uint32_t q = r + threadIdx.x; q < CC_CHUNK; q += PD_THREADS)
            out[((unsigned long long)c << CC_CHUNK_BITS) | q] = make_uint2(0u, 0u);
    }
}

// hook range of window k: [0, chunks_k * CC_CHUNK).  (One hook launch over all
// windows laid end to end measured 4.27 vs 2.87 ms at C5: without the launch
// boundary the fast warps run into the next windows and the parent gathers
// spill out of L2.)
__global__ void k_cc_chunk_ranges(const uint32_t* __restrict__ counts, int P, unsigned long long* __restrict__ rng) {
    const int k = threadIdx.x;
    if (k < P) {
        rng[2 * k] = 0;
        rng[2 * k + 1] = (unsigned long long)counts[k] << CC_CHUNK_BITS;
    }
}

// ---------------------------------------------------------------------------
// sparse merge of the sharded rounds (dist.py): after the dense merge of
// round 1 every replica is identical, so later rounds only exchange the
// entries a rank's hook sweep lowered

__global__ void k_cc_changes(const uint32_t* __restrict__ Dold, const uint32_t* __restrict__ D, unsigned long long n,
                             uint32_t* __restrict__ idx, uint32_t* __restrict__ val, unsigned long long cap,
                             unsigned long long* __restrict__ count) {
    const uint32_t lane = lane_id();
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i0 = (unsigned long long)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const unsigned long long i = i0 + threadIdx.x;
        const uint32_t d = i < n ? D[i] : 0u;
        const bool ch = i < n && d != Dold[i];
        const unsigned m = __ballot_sync(0xffffffffu, ch);
        if (m == 0) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (ch) {
            const unsigned long long k = base + __popc(m & ((1u << lane) - 1u));
            if (k < cap) {
                idx[k] = (uint32_t)i;
                val[k] = d;
            }
        }
    }
}

__global__ void k_cc_apply_min(uint32_t* __restrict__ D, const uint32_t* __restrict__ idx,
                               const uint32_t* __restrict__ val, unsigned long long k) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride)
        atomicMin(D + idx[i], val[i]);
}

// ---------------------------------------------------------------------------
// host side

static uint32_t hook_grid(unsigned long long m) { return grid_for(m, HOOK_THREADS, 4, sm_count() * 8); }
static uint32_t vtx_grid(unsigned long long n) { return grid_for(n, COMP_THREADS, 1, sm_count() * 8); }

template <class E>
static int launch_hook(E view, unsigned long long m, unsigned long long row0, unsigned long long n, uint32_t* D,
                       int variant, bool validate, unsigned long long* flags, cudaStream_t s,
                       const unsigned long long* rng = nullptr) {
    if (m == 0) return SG_OK;
    const uint32_t g = hook_grid(m);
    if (variant == SG_CC_UF) {
        if (validate)
            k_cc_hook_uf<E, true><<<g, HOOK_THREADS, 0, s>>>(view, m, row0, n, D, flags, rng);
        else
            k_cc_hook_uf<E, false><<<g, HOOK_THREADS, 0, s>>>(view, m, row0, n, D, flags, rng);
    } else {
        if (validate)
            k_cc_hook_sv<E, true><<<g, HOOK_THREADS, 0, s>>>(view, m, row0, n, D, flags, rng);
        else
            k_cc_hook_sv<E, false><<<g, HOOK_THREADS, 0, s>>>(view, m, row0, n, D, flags, rng);
    }
    SG_LAUNCH_CHECK();
    return SG_OK;
}

static int hook_dispatch(const void* edges, int dt, unsigned long long m, unsigned long long row0,
                         unsigned long long n, uint32_t* D, int variant, bool validate, unsigned long long* flags,
                         cudaStream_t s) {
    switch (dt) {
        case SG_U32: return launch_hook(EdgesU32{(const uint2*)edges}, m, row0, n, D, variant, validate, flags, s);
        case SG_I32: return launch_hook(EdgesI32{(const int2*)edges}, m, row0, n, D, variant, validate, flags, s);
        case SG_I64: return launch_hook(EdgesI64{(const longlong2*)edges}, m, row0, n, D, variant, validate, flags, s);
        default: return SG_ERR_VALUE;
    }
}

struct CcPlan {
    int parts = 1;
    uint32_t shift = 31;
    unsigned long long ntiles = 0;
};

static CcPlan plan_cc(unsigned long long n, unsigned long long m) {
    CcPlan p;
    const uint32_t tw = tuning().cc_wbits;  // tests force small windows with SG_CC_WBITS
    uint32_t wbits = tw ? tw : 23u;         // window of 2^23 vertices = 32 MiB of D
    if (wbits < 10) wbits = 10;
    if (wbits > 31) wbits = 31;
    unsigned long long parts = (n + (1ull << wbits) - 1) >> wbits;
    while (parts > MAX_PARTS) {
        ++wbits;
        parts = (n + (1ull << wbits) - 1) >> wbits;
    }
    if (parts <= 1 || m < (1ull << 16)) return p;
    p.parts = (int)parts;
    p.shift = wbits;
    p.ntiles = (m + PART_TILE - 1) / PART_TILE;
    return p;
}

struct CcPartBufs {
    unsigned long long* totals = nullptr;   // [MAX_PARTS]
    unsigned long long* cursor = nullptr;   // [MAX_PARTS]
    unsigned long long* off_part = nullptr; // [MAX_PARTS + 2]
    uint32_t* counts = nullptr;             // [2 * MAX_PARTS] chunk layout: chunks per window, chunks claimed
    uint32_t* dir = nullptr;                // [parts][dir_stride] chunk ids per window
    unsigned long long* rng = nullptr;      // [2 * MAX_PARTS] hook range per window
    unsigned long long dir_stride = 0;
    uint32_t* cta_list = nullptr;           // [grid][parts][kmax] chunk ids per CTA and window
    uint32_t kmax = 0;
    uint2* edges = nullptr;
    bool chunked = false;                   // which layout partition_edges produced
};

// partition mode: one pass into per-window chunk lists (default), or count +
// scatter (SG_CC_PART=count; also taken for input rows that are not 16-B
// aligned, which the bulk copies need).  A reused partition (sg_cc_hook_part,
// reuse = 1) re-derives its layout from the same test.
static bool use_chunks(const void*) { return !tuning().cc_part_count; }
static uint32_t chunk_grid(unsigned long long m) {
    const unsigned long long warps = (m + 64 * PD_GROUPS - 1) / (64 * PD_GROUPS);  // PD_GROUPS groups per warp at least
    const unsigned long long ctas = (warps + PD_THREADS / 32 - 1) / (PD_THREADS / 32);
    const unsigned long long g = (unsigned long long)sm_count() * PD_CTAS_PER_SM;
    return (uint32_t)(ctas < g ? ctas : g);
}
// chunks the layout can claim: every full chunk, plus per (CTA, window) one
// partial chunk and one pre-claimed chunk that may stay unused
static unsigned long long max_chunks(unsigned long long m, int parts) {
    return ((m + CC_CHUNK - 1) >> CC_CHUNK_BITS) + 2ull * parts * chunk_grid(m);
}
// chunks one CTA can fill per window: its warps' groups, whole chunks, plus the open one
static uint32_t chunk_kmax(unsigned long long m) {
    const unsigned long long nw = (unsigned long long)chunk_grid(m) * (PD_THREADS / 32);
    const unsigned long long ng = (m + 63) / 64;
    const unsigned long long rows = ((ng + nw - 1) / nw + 1) * 64 * (PD_THREADS / 32);
    return (uint32_t)((rows >> CC_CHUNK_BITS) + 3);  // + the open chunk + the pre-claimed one
}

static bool carve_part(Carver& c, unsigned long long m, const CcPlan& p, CcPartBufs& b) {
    b.totals = c.take<unsigned long long>(MAX_PARTS);
    b.cursor = c.take<unsigned long long>(MAX_PARTS);
    b.off_part = c.take<unsigned long long>((size_t)MAX_PARTS + 2);
    b.counts = c.take<uint32_t>(2 * MAX_PARTS);
    b.rng = c.take<unsigned long long>(2 * MAX_PARTS);
    const unsigned long long mc = max_chunks(m, p.parts);
    b.dir_stride = mc;
    b.dir = c.take<uint32_t>((size_t)(mc * p.parts));
    b.kmax = chunk_kmax(m);
    b.cta_list = c.take<uint32_t>((size_t)chunk_grid(m) * p.parts * b.kmax);
    b.edges = c.take<uint2>((size_t)(mc << CC_CHUNK_BITS));  // >= m: also holds the count + scatter layout
    return c.ok;
}

template <class E>
static int partition_edges(E view, unsigned long long m, unsigned long long n, const CcPlan& p, CcPartBufs& b,
                           unsigned long long* flags, cudaStream_t s, unsigned long long row0 = 0,
                           uint32_t* Dinit = nullptr) {
    const uint32_t nt = (uint32_t)p.ntiles;
    b.chunked = false;
    if (use_chunks(view.e)) {
        int nbits = 0;
        while ((1 << nbits) < p.parts) ++nbits;
        const bool narrow = E::kBytes == 8 && n <= 0x80000000ull;
        using KT = void (*)(E, unsigned long long, unsigned long long, unsigned long long, uint32_t, int, uint2*,
                            uint32_t*, unsigned long long, uint32_t*, uint32_t*, uint32_t, unsigned long long*,
                            uint32_t*, unsigned long long);
        KT kt;
        const bool v16 = E::kBytes == 8 && narrow && ((uintptr_t)view.e & 15) == 0;
        if (!tuning().cc_rank_ballot)  // match.any peers (default)
            kt = v16 ? k_cc_part_chunks<E, 4, true, true, (E::kBytes == 8)>
                     : (narrow ? k_cc_part_chunks<E, 4, true, true> : k_cc_part_chunks<E, 4, false, true>);
        else
            kt = narrow ? (nbits <= 1 ? k_cc_part_chunks<E, 1, true, false>
                           : nbits == 2 ? k_cc_part_chunks<E, 2, true, false>
                           : nbits == 3 ? k_cc_part_chunks<E, 3, true, false> : k_cc_part_chunks<E, 4, true, false>)
                        : (nbits <= 1 ? k_cc_part_chunks<E, 1, false, false>
                           : nbits == 2 ? k_cc_part_chunks<E, 2, false, false>
                           : nbits == 3 ? k_cc_part_chunks<E, 3, false, false> : k_cc_part_chunks<E, 4, false, false>);
        SG_CUDA(cudaMemsetAsync(b.counts, 0, sizeof(uint32_t) * 2 * MAX_PARTS, s));
        kt<<<chunk_grid(m), PD_THREADS, 0, s>>>(view, m, n, row0, p.shift, p.parts, b.edges, b.dir, b.dir_stride,
                                                b.counts, b.cta_list, b.kmax, flags, Dinit, Dinit ? n : 0ull);
        SG_LAUNCH_CHECK();
        k_cc_chunk_ranges<<<1, 32, 0, s>>>(b.counts, p.parts, b.rng);
        SG_LAUNCH_CHECK();
        b.chunked = true;
        return SG_OK;
    }
    if (Dinit != nullptr) {
        k_cc_init<<<vtx_grid(n), COMP_THREADS, 0, s>>>(Dinit, n);
        SG_LAUNCH_CHECK();
    }
    SG_CUDA(cudaMemsetAsync(b.totals, 0, sizeof(unsigned long long) * MAX_PARTS, s));
    SG_CUDA(cudaMemsetAsync(b.cursor, 0, sizeof(unsigned long long) * MAX_PARTS, s));
    const uint32_t cg = nt < sm_count() * 8 ? nt : sm_count() * 8;
    int nbits = 0;
    while ((1 << nbits) < p.parts) ++nbits;
    const bool narrow = E::kBytes == 8 && n <= 0x80000000ull;  // (u32 ids are < 2^32 - 1 = n's cap anyway)
    auto kc = narrow ? (nbits <= 1 ? k_cc_part_count<E, 1, true>
                        : nbits == 2 ? k_cc_part_count<E, 2, true>
                        : nbits == 3 ? k_cc_part_count<E, 3, true> : k_cc_part_count<E, 4, true>)
                     : (nbits <= 1 ? k_cc_part_count<E, 1, false>
                        : nbits == 2 ? k_cc_part_count<E, 2, false>
                        : nbits == 3 ? k_cc_part_count<E, 3, false> : k_cc_part_count<E, 4, false>);
    kc<<<cg, PART_THREADS, 0, s>>>(view, m, n, row0, p.shift, p.parts, b.totals, flags);
    SG_LAUNCH_CHECK();
    k_cc_part_offsets<<<1, 32, 0, s>>>(b.totals, p.parts, b.off_part);
    SG_LAUNCH_CHECK();
    if (((uintptr_t)view.e & 15) == 0) {
        const size_t smem = (size_t)MS2_TILE * E::kBytes + MsSmem::bytes((uint32_t)p.parts, MS2_TILE);
        auto ks = narrow ? (nbits <= 1 ? k_cc_part_scatter2<E, 1, true>
                            : nbits == 2 ? k_cc_part_scatter2<E, 2, true>
                            : nbits == 3 ? k_cc_part_scatter2<E, 3, true> : k_cc_part_scatter2<E, 4, true>)
                         : (nbits <= 1 ? k_cc_part_scatter2<E, 1, false>
                            : nbits == 2 ? k_cc_part_scatter2<E, 2, false>
                            : nbits == 3 ? k_cc_part_scatter2<E, 3, false> : k_cc_part_scatter2<E, 4, false>);
        SG_CUDA(set_smem_max(ks, smem));
        const unsigned long long ntile = (m + MS2_TILE - 1) / MS2_TILE;
        const uint32_t ns = (uint32_t)(ntile < (unsigned long long)sm_count() * PART2_CTAS_PER_SM ? ntile
                                                                                            : sm_count() * PART2_CTAS_PER_SM);
        ks<<<ns, MS_THREADS, smem, s>>>(view, m, n, p.shift, p.parts, b.off_part, b.cursor, b.edges);
    } else {
        const size_t smem = MsSmem::bytes((uint32_t)p.parts);
        SG_CUDA(set_smem_max(k_cc_part_scatter<E>, smem));
        const unsigned long long ntile = (m + MS_TILE - 1) / MS_TILE;
        const uint32_t ns = (uint32_t)(ntile < (unsigned long long)sm_count() * 4 ? ntile : sm_count() * 4);
        k_cc_part_scatter<E><<<ns, MS_THREADS, smem, s>>>(view, m, n, p.shift, p.parts, b.off_part, b.cursor, b.edges);
    }
    SG_LAUNCH_CHECK();
    return SG_OK;
}

static int partition_dispatch(const void* edges, int dt, unsigned long long m, unsigned long long n, const CcPlan& p,
                              CcPartBufs& b, unsigned long long* flags, cudaStream_t s, unsigned long long row0 = 0,
                              uint32_t* Dinit = nullptr) {
    switch (dt) {
        case SG_U32: return partition_edges(EdgesU32{(const uint2*)edges}, m, n, p, b, flags, s, row0, Dinit);
        case SG_I32: return partition_edges(EdgesI32{(const int2*)edges}, m, n, p, b, flags, s, row0, Dinit);
        case SG_I64: return partition_edges(EdgesI64{(const longlong2*)edges}, m, n, p, b, flags, s, row0, Dinit);
        default: return SG_ERR_VALUE;
    }
}

// one hook sweep over a partitioned edge list, window by window
// a full shortcut sweep between hook launches: the later edges then find most
// roots one step away.  Unpartitioned UF (D in L2, n <= 2^23): after the
// first m / 8 rows (SG_CC_SPLIT=3, default): C4 hook 0.345 -> 0.262 ms incl.
// the sweep (~0.014 ms); after m / 4: 0.279 ms, m / 16: 0.32 ms, a second
// sweep (SG_CC_SPLIT2) no gain (passes x2-x4).  Partitioned (SG_CC_SPLITW=k, after k windows;
// experiment, off): C5 hook 2.89 -> 3.02-3.08 ms for k = 2, 4, 6 -- the sweep
// over 256 MiB of D costs more than the shorter finds save (pass x2)
static void mid_shortcut(uint32_t* D, unsigned long long n, cudaStream_t s) {
    k_cc_compress<uint32_t><<<vtx_grid(n), COMP_THREADS, 0, s>>>(D, 0, n, nullptr, nullptr);
}

static int hook_partitions(const CcPlan& p, const CcPartBufs& b, unsigned long long m, unsigned long long n,
                           uint32_t* D, int variant, unsigned long long* flags, cudaStream_t s) {
    const unsigned long long per = m / p.parts + 1;
    const uint32_t split = variant == SG_CC_UF ? tuning().cc_splitw : 0u;  // shortcut after this many windows
    if (b.chunked) {  // one launch per window: the launch boundary keeps the window's parents in L2
        for (int k = 0; k < p.parts; ++k) {
            if (split && k == (int)split) mid_shortcut(D, n, s);
            int rc = launch_hook(EdgesChunked{b.edges, b.dir + (size_t)k * b.dir_stride}, per, 0, n, D, variant, false,
                                 flags, s, b.rng + 2 * k);
            if (rc != SG_OK) return rc;
        }
        return SG_OK;
    }
    for (int k = 0; k < p.parts; ++k) {
        int rc = launch_hook(EdgesU32{b.edges}, per, 0, n, D, variant, false, flags, s, b.off_part + k);
        if (rc != SG_OK) return rc;
    }
    return SG_OK;
}

static int compress_dispatch(uint32_t* D, unsigned long long lo, unsigned long long hi, unsigned long long* roots,
                             void* out, int odt, cudaStream_t s) {
    if (hi <= lo) return SG_OK;
    const uint32_t g = vtx_grid(hi - lo);
    if (tuning().cc_comp4 && ((uintptr_t)(D + lo) & 15) == 0) {  // four vertices per thread
        const uint32_t g4 = vtx_grid((hi - lo + 3) / 4);
        if (out == nullptr || odt == SG_U32 || odt == SG_I32)
            k_cc_compress4<uint32_t><<<g4, COMP_THREADS, 0, s>>>(D, lo, hi, roots,
                                                                 out == (void*)D ? nullptr : (uint32_t*)out);
        else if (odt == SG_I64)
            k_cc_compress4<int64_t><<<g4, COMP_THREADS, 0, s>>>(D, lo, hi, roots, (int64_t*)out);
        else
            return SG_ERR_VALUE;
        SG_LAUNCH_CHECK();
        return SG_OK;
    }
    if (out == nullptr || odt == SG_U32 || odt == SG_I32) {
        // u32 / i32 labels share D's bit pattern (ids < 2^31 for i32)
        k_cc_compress<uint32_t><<<g, COMP_THREADS, 0, s>>>(D, lo, hi, roots,
                                                           out == (void*)D ? nullptr : (uint32_t*)out);
    } else if (odt == SG_I64) {
        k_cc_compress<int64_t><<<g, COMP_THREADS, 0, s>>>(D, lo, hi, roots, (int64_t*)out);
    } else {
        return SG_ERR_VALUE;
    }
    SG_LAUNCH_CHECK();
    return SG_OK;
}

struct CcHostFlags {
    unsigned long long f[4];
    unsigned long long roots;
};

static int read_flags(const unsigned long long* dev, CcHostFlags& h, cudaStream_t s) {
    SG_CUDA(cudaMemcpyAsync(&h, dev, sizeof(CcHostFlags), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    return SG_OK;
}

// pinned host copy of the flags, enqueued behind the last kernel so a call
// synchronises once
static CcHostFlags* pinned_flags() {
    static thread_local CcHostFlags* p = nullptr;
    if (!p && cudaMallocHost(&p, sizeof(CcHostFlags)) != cudaSuccess) p = nullptr;
    return p;
}

static int graph_violation(const CcHostFlags& h, sg_violation* v) {
    if (h.f[1]) {
        if (v) {
            v->kind = SG_GRAPH_OUT_OF_RANGE;
            v->index = (int64_t)~h.f[1];
        }
        return SG_ERR_INVALID_GRAPH;
    }
    if (h.f[2]) {
        if (v) {
            v->kind = SG_GRAPH_SELF_LOOP;
            v->index = (int64_t)~h.f[2];
        }
        return SG_ERR_INVALID_GRAPH;
    }
    return SG_OK;
}

}  // namespace sg

using namespace sg;

extern "C" {

static bool carve_cc(Carver& c, uint64_t n, uint64_t m, const CcPlan& p, unsigned long long*& flags, uint32_t*& Dws,
                     CcPartBufs& b) {
    flags = c.take<unsigned long long>(8);  // [0..3] flags, [4] roots
    Dws = c.take<uint32_t>(n);
    if (p.parts > 1) carve_part(c, m, p, b);
    return c.ok;
}

size_t sg_cc_workspace_bytes(uint64_t n, uint64_t m) {
    const CcPlan p = plan_cc(n, m);
    Carver c(nullptr, 0);
    unsigned long long* f;
    uint32_t* d;
    CcPartBufs b;
    carve_cc(c, n, m, p, f, d, b);
    return c.off + 256;
}

int sg_cc(const void* edges, int edge_dtype, uint64_t m, uint64_t n, void* labels, int label_dtype, int variant,
          int round_bound, void* ws, size_t ws_bytes, void* stream, sg_stats* st, sg_violation* viol) {
    if (n == 0) return SG_ERR_INVALID_GRAPH;
    if (n >= 0x7FFFFFFFull) return SG_ERR_CAPABILITY;
    if (variant != SG_CC_UF && variant != SG_CC_SV) return SG_ERR_VALUE;
    if (label_dtype != SG_U32 && label_dtype != SG_I32 && label_dtype != SG_I64) return SG_ERR_VALUE;
    ::sg::apply_tuning();
    cudaStream_t s = (cudaStream_t)stream;
    if (st) memset(st, 0, sizeof(sg_stats));
    if (viol) {
        viol->kind = SG_GRAPH_OK;
        viol->index = -1;
        viol->pad = 0;
    }
    const CcPlan plan = plan_cc(n, m);
    ms_configure();
    Carver c(ws, ws_bytes);
    unsigned long long* flags;
    uint32_t* Dws;
    CcPartBufs pb;
    if (!carve_cc(c, n, m, plan, flags, Dws, pb)) return SG_ERR_WORKSPACE;
    // u32/i32 labels: run in place in the output buffer
    uint32_t* D = (label_dtype == SG_I64) ? Dws : (uint32_t*)labels;
    unsigned long long* roots = flags + 4;

    Recorder rec(st, s);
    SG_CUDA(cudaMemsetAsync(flags, 0, 8 * sizeof(unsigned long long), s));
    const uint32_t gv = vtx_grid(n);
    const bool parted = plan.parts > 1;
    if (!parted) {  // (partitioned: the partition pass writes the identity forest beside the edges)
        rec.begin(K_CC_INIT, 0, gv, COMP_THREADS, n);
        k_cc_init<<<gv, COMP_THREADS, 0, s>>>(D, n);
        rec.end();
        SG_LAUNCH_CHECK();
    }
    if (st) {
        st->roots_per_round[0] = n;
        st->n_roots = 1;
        st->vertex_sweeps = 1;
    }
    int rc;
    if (parted) {
        rec.begin(K_CC_PARTITION, 0, (uint32_t)plan.ntiles, PART_THREADS, m);
        rc = partition_dispatch(edges, edge_dtype, m, n, plan, pb, flags, s, 0, D);
        rec.end();
        if (rc != SG_OK) return rc;
        if (st) st->edge_sweeps = 0;
    }
    if (variant == SG_CC_UF) {
        rec.begin(K_CC_HOOK_UF, 1, hook_grid(m), HOOK_THREADS, m);
        const uint32_t split = tuning().cc_split;
        if (parted) {
            rc = hook_partitions(plan, pb, m, n, D, SG_CC_UF, flags, s);
        } else if (split && split < 32 && m >= (1ull << 16)) {  // (smaller sweeps are launch-bound)
            // hook the first m / 2^f rows (SG_CC_SPLIT=f), shortcut, hook the rest
            // (SG_CC_SPLIT2=f2 < f: a second shortcut after m / 2^f2 rows)
            const uint32_t split2 = tuning().cc_split2;
            unsigned long long cut[3] = {m >> split, m, m};
            if (split2 && split2 < split) cut[1] = m >> split2;
            const size_t esz = edge_dtype == SG_I64 ? 16 : 8;
            unsigned long long r0 = 0;
            rc = SG_OK;
            for (int k = 0; k < 3 && rc == SG_OK && r0 < m; ++k) {
                if (k > 0) {
                    mid_shortcut(D, n, s);
                    if (st) st->vertex_sweeps += 1;
                }
                rc = hook_dispatch((const char*)edges + r0 * esz, edge_dtype, cut[k] - r0, r0, n, D, SG_CC_UF, true,
                                   flags, s);
                r0 = cut[k];
            }
        } else {
            rc = hook_dispatch(edges, edge_dtype, m, 0, n, D, SG_CC_UF, true, flags, s);
        }
        rec.end();
        if (rc != SG_OK) return rc;
        rec.begin(K_CC_COMPRESS, 1, gv, COMP_THREADS, n);
        rc = compress_dispatch(D, 0, n, roots, labels, label_dtype, s);
        rec.end();
        if (rc != SG_OK) return rc;
        CcHostFlags* hp = pinned_flags();
        CcHostFlags hloc;
        if (hp) SG_CUDA(cudaMemcpyAsync(hp, flags, sizeof(CcHostFlags), cudaMemcpyDeviceToHost, s));
        SG_CUDA(rec.finish());  // the one synchronisation of a UF call
        if (!hp) {
            rc = read_flags(flags, hloc, s);
            if (rc != SG_OK) return rc;
        }
        const CcHostFlags& h = hp ? *hp : hloc;
        rc = graph_violation(h, viol);
        if (rc != SG_OK) return rc;
        if (st) {
            st->rounds = 1;
            st->edge_sweeps = m ? 1 : 0;
            st->vertex_sweeps += 1;
            st->roots_per_round[1] = h.roots;
            st->n_roots = 2;
        }
        return SG_OK;
    }
    // SV rounds
    int r = 0;
    for (;;) {
        ++r;
        if (r > round_bound) return SG_ERR_RUNTIME;
        SG_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned long long), s));
        SG_CUDA(cudaMemsetAsync(roots, 0, sizeof(unsigned long long), s));
        rec.begin(K_CC_HOOK_SV, r, hook_grid(m), HOOK_THREADS, m);
        rc = parted ? hook_partitions(plan, pb, m, n, D, SG_CC_SV, flags, s)
                    : hook_dispatch(edges, edge_dtype, m, 0, n, D, SG_CC_SV, r == 1, flags, s);
        rec.end();
        if (rc != SG_OK) return rc;
        rec.begin(K_CC_COMPRESS, r, gv, COMP_THREADS, n);
        rc = compress_dispatch(D, 0, n, roots, nullptr, SG_U32, s);
        rec.end();
        if (rc != SG_OK) return rc;
        CcHostFlags h;
        rc = read_flags(flags, h, s);
        if (rc != SG_OK) return rc;
        if (r == 1 || parted) {
            rc = graph_violation(h, viol);
            if (rc != SG_OK) return rc;
        }
        if (st) {
            st->edge_sweeps += m ? 1 : 0;
            st->vertex_sweeps += 1;
            if (st->n_roots < SG_MAX_ROUNDS) st->roots_per_round[st->n_roots++] = h.roots;
            st->rounds = (uint32_t)r;
        }
        if (!h.f[0]) break;
    }
    if (label_dtype == SG_I64) {
        rec.begin(K_CC_LABELS, r, gv, COMP_THREADS, n);
        k_cc_labels<int64_t><<<gv, COMP_THREADS, 0, s>>>(D, n, (int64_t*)labels);
        rec.end();
        SG_LAUNCH_CHECK();
    }
    SG_CUDA(rec.finish());
    return SG_OK;
}

int sg_cc_init(uint32_t* D, uint64_t n, void* stream) {
    if (n == 0) return SG_OK;
    k_cc_init<<<vtx_grid(n), COMP_THREADS, 0, (cudaStream_t)stream>>>(D, n);
    SG_LAUNCH_CHECK();
    return SG_OK;
}

int sg_cc_hook(const void* edges, int edge_dtype, uint64_t m, uint64_t row0, uint64_t n, uint32_t* D, int variant,
               int validate, uint64_t* flags, void* stream) {
    if (variant != SG_CC_UF && variant != SG_CC_SV) return SG_ERR_VALUE;
    return hook_dispatch(edges, edge_dtype, m, row0, n, D, variant, validate != 0, (unsigned long long*)flags,
                         (cudaStream_t)stream);
}

size_t sg_cc_hook_workspace_bytes(uint64_t n, uint64_t m) {
    const CcPlan p = plan_cc(n, m);
    if (p.parts <= 1) return 256;
    Carver c(nullptr, 0);
    CcPartBufs b;
    carve_part(c, m, p, b);
    return c.off + 256;
}

int sg_cc_hook_part(const void* edges, int edge_dtype, uint64_t m, uint64_t row0, uint64_t n, uint32_t* D,
                    int variant, int validate, uint64_t* flags, void* ws, size_t ws_bytes, int reuse, void* stream) {
    if (variant != SG_CC_UF && variant != SG_CC_SV) return SG_ERR_VALUE;
    const CcPlan p = plan_cc(n, m);
    cudaStream_t s = (cudaStream_t)stream;
    if (p.parts <= 1)
        return hook_dispatch(edges, edge_dtype, m, row0, n, D, variant, validate != 0, (unsigned long long*)flags, s);
    ms_configure();
    Carver c(ws, ws_bytes);
    CcPartBufs b;
    if (!carve_part(c, m, p, b)) return SG_ERR_WORKSPACE;
    b.chunked = use_chunks(edges);
    if (!reuse) {  // rows are validated while they are partitioned (flags hold ~global row)
        int rc = partition_dispatch(edges, edge_dtype, m, n, p, b, (unsigned long long*)flags, s, row0);
        if (rc != SG_OK) return rc;
    }
    return hook_partitions(p, b, m, n, D, variant, (unsigned long long*)flags, s);
}

int sg_cc_changes(const uint32_t* Dold, const uint32_t* D, uint64_t n, uint32_t* idx, uint32_t* val, uint64_t cap,
                  uint64_t* count, void* stream) {
    if (n == 0) return SG_OK;
    // count is accumulated: the caller zeroes it
    k_cc_changes<<<vtx_grid(n), COMP_THREADS, 0, (cudaStream_t)stream>>>(Dold, D, n, idx, val, cap,
                                                                          (unsigned long long*)count);
    SG_LAUNCH_CHECK();
    return SG_OK;
}

int sg_cc_apply_min(uint32_t* D, const uint32_t* idx, const uint32_t* val, uint64_t k, void* stream) {
    if (k == 0) return SG_OK;
    k_cc_apply_min<<<vtx_grid(k), COMP_THREADS, 0, (cudaStream_t)stream>>>(D, idx, val, k);
    SG_LAUNCH_CHECK();
    return SG_OK;
}

int sg_cc_compress(uint32_t* D, uint64_t lo, uint64_t hi, uint64_t* roots, void* stream) {
    return compress_dispatch(D, lo, hi, (unsigned long long*)roots, nullptr, SG_U32, (cudaStream_t)stream);
}

int sg_cc_labels(const uint32_t* D, uint64_t n, void* out, int out_dtype, void* stream) {
    if (n == 0) return SG_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t g = vtx_grid(n);
    switch (out_dtype) {
        case SG_U32: k_cc_labels<uint32_t><<<g, COMP_THREADS, 0, s>>>(D, n, (uint32_t*)out); break;
        case SG_I32: k_cc_labels<int32_t><<<g, COMP_THREADS, 0, s>>>(D, n, (int32_t*)out); break;
        case SG_I64: k_cc_labels<int64_t><<<g, COMP_THREADS, 0, s>>>(D, n, (int64_t*)out); break;
        default: return SG_ERR_VALUE;
    }
    SG_LAUNCH_CHECK();
    return SG_OK;
}

}  // extern "C"
