// sg_list.cu -- list ranking on sm_100a.
//
//  * Wyllie pointer jumping (reference: listrank.py:75-155) over packed
//    64-bit {rank:32 | succ:32} words, updated in place.  Asynchronous
//    in-place jumping is sound because a word is always read and written as
//    one 64-bit access: whichever version of w[s] a node sees, its
//    (distance, pointer) pair stays consistent and its pointer distance at
//    least doubles per launch, so ceil(log2 n) launches still suffice.
//    Converged nodes (pointer at the tail) are skipped without a gather.
//
//  * Recursive sparse ruling set (reference RS1..RS5: listrank.py:197-408)
//    for scattered layouts.  Level 0 walks the input list from a hashed
//    ruling set (every ~2^kbits-th node id, Fibonacci hashing, node 0 always
//    included): one dependent random load (succ[cur]) per node, and one
//    {cur, sid, local} record streamed out; one {next ruler, sublist weight}
//    pair per ruler.  The ruler list is ranked the same way (weighted, in
//    place) until it fits one CTA, which finishes it with weighted pointer
//    jumping; expand passes turn inclusive suffix sums back into ranks, and
//    TMA-staged multisplit passes put the level-0 ranks in node order.
//
//  * Tile contraction for local layouts (ordered or locally shuffled lists):
//    in-tile segments are ranked in shared memory, the segment list is
//    ranked by the levels above, a streaming pass expands.
//
// Validation happens inside the pipeline (no host round trip): range / tail
// census in the first pass, and "the head's weighted pointer reaches the
// tail with inclusive sum n" at the top level -- together equivalent to
// core.validate_list (core.py:148-167).  A walk that exceeds the hop cap
// (a cycle without rulers, or a pathological layout) makes the host re-run
// the list with Wyllie, which terminates on any input.
#include <cub/block/block_load.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/block/block_store.cuh>

#include <cooperative_groups.h>
#include <stdlib.h>
#include <type_traits>
#include <string.h>

#include <atomic>

#include "sg_internal.cuh"
#include "sg_msplit.cuh"

namespace sg {

constexpr uint32_t PHI = 0x9E3779B9u;
constexpr int TILE_THREADS = 256;
constexpr int TILE_ITEMS = 16;
constexpr int TILE = TILE_THREADS * TILE_ITEMS;
constexpr uint32_t FINAL_CAP = 8192;          // ruler list handled by one CTA
constexpr uint32_t WALK_CAP_HOPS = 1u << 16;  // longer walk => Wyllie fallback
constexpr int WALK_THREADS = 256;
constexpr int JUMP_THREADS = 256;

// ---------------------------------------------------------------------------
// element access helpers

template <class T>
__device__ __forceinline__ unsigned long long as_index(T v);
template <>
__device__ __forceinline__ unsigned long long as_index<uint32_t>(uint32_t v) { return v; }
template <>
__device__ __forceinline__ unsigned long long as_index<int32_t>(int32_t v) {
    return (unsigned long long)(long long)v;
}
template <>
__device__ __forceinline__ unsigned long long as_index<int64_t>(int64_t v) {
    return (unsigned long long)v;
}

__device__ __forceinline__ bool is_ruler(uint32_t i, uint32_t kbits, uint32_t salt) {
    return i == 0u || ((i * PHI + salt) >> (32u - kbits)) == 0u;
}

template <class T>
__device__ __forceinline__ T ld_mode(const T* p, int mode) {
    switch (mode) {
        case 1: return __ldcg(p);   // L2 only
        case 2: return __ldcv(p);   // volatile (no cache)
        case 3: return *p;          // default (L1 + L2)
        default: return __ldg(p);   // read-only path
    }
}

// level-0 view: node i -> (successor, weight 1)
template <class SuccT>
struct Level0 {
    const SuccT* succ;
    int mode;
    __device__ __forceinline__ void load(uint32_t i, unsigned long long& nx, uint32_t& w) const {
        nx = as_index<SuccT>(ld_mode(succ + i, mode));
        w = 1u;
    }
};

// level-k view: ruler i -> (next ruler, sublist weight); next == i at the tail
struct LevelK {
    const uint2* lvl;
    __device__ __forceinline__ void load(uint32_t i, unsigned long long& nx, uint32_t& w) const {
        uint2 e = lvl[i];
        nx = e.x;
        w = e.y;
    }
};

// ---------------------------------------------------------------------------
// status

__global__ void k_status_init(ListStatus* st, unsigned long long n) {
    if (threadIdx.x == 0) {
        st->oor_first = NONE64;
        st->loop_first = NONE64;
        st->loop_count = 0;
        st->overflow = 0;
        st->head_sum = 0;
        st->head_ok = 0;
        st->bad = 0;
        st->local = 0;
        st->chunks = 0;
        st->top_live[0] = st->top_live[1] = st->top_live[2] = 0;
    }
    if (threadIdx.x <= SG_MAX_LEVELS) {
        st->R[threadIdx.x] = threadIdx.x == 0 ? n : 0;
        st->qhead[threadIdx.x] = 0;
    }
}

__device__ __forceinline__ void note_succ(ListStatus* st, unsigned long long i, unsigned long long v,
                                          unsigned long long n) {
    if (v >= n) {
        atomicMin(&st->oor_first, i);
    } else if (v == i) {
        atomicAdd(&st->loop_count, 1ull);
        atomicMin(&st->loop_first, i);
    }
}

// ---------------------------------------------------------------------------
// Wyllie

template <class SuccT>
__global__ void __launch_bounds__(JUMP_THREADS) k_wy_init(const SuccT* __restrict__ succ,
                                                          unsigned long long* __restrict__ word,
                                                          unsigned long long n, ListStatus* st) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        unsigned long long v = as_index<SuccT>(succ[i]);
        note_succ(st, i, v, n);
        if (v >= n) v = i;  // neutralise: never gather out of range
        word[i] = ((unsigned long long)(v != i) << 32) | v;
    }
}

__device__ __forceinline__ uint32_t wy_tail(const ListStatus* st) {
    const unsigned long long lc = *(volatile const unsigned long long*)&st->loop_count;
    const unsigned long long lf = *(volatile const unsigned long long*)&st->loop_first;
    return lc == 1 ? (uint32_t)lf : NIL;
}

// one jump round, in place; `rank` != nullptr on the last round (extracts ranks)
template <class OutT>
__global__ void __launch_bounds__(JUMP_THREADS) k_wy_jump(unsigned long long* word, unsigned long long n,
                                                          const ListStatus* st, OutT* __restrict__ rank) {
    constexpr int U = 4;
    const uint32_t tail = wy_tail(st);
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long i0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i0 < n; i0 += stride * U) {
        unsigned long long w[U];
        bool live[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned long long i = i0 + (unsigned long long)u * stride;
            w[u] = i < n ? word[i] : 0ull;
            const uint32_t s = (uint32_t)w[u];
            live[u] = i < n && s != tail && (unsigned long long)s != i;
        }
        unsigned long long w2[U];
#pragma unroll
        for (int u = 0; u < U; ++u) w2[u] = live[u] ? __ldcg(word + (uint32_t)w[u]) : 0ull;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned long long i = i0 + (unsigned long long)u * stride;
            if (live[u]) {
                const unsigned long long rk = ((w[u] >> 32) + (w2[u] >> 32)) & 0xFFFFFFFFull;
                w[u] = (rk << 32) | (w2[u] & 0xFFFFFFFFull);
                word[i] = w[u];
            }
            if (rank != nullptr && i < n) rank[i] = (OutT)(w[u] >> 32);
        }
    }
}

__global__ void k_wy_check(const unsigned long long* word, unsigned long long n, ListStatus* st) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const uint32_t tail = wy_tail(st);
        const unsigned long long w0 = word[0];
        st->head_ok = ((uint32_t)w0 == tail) ? 1ull : 0ull;
        st->head_sum = (w0 >> 32) + 1;  // inclusive count of nodes from the head
    }
}

// single CTA: init, `rounds` in-place jump rounds separated by block
// barriers, rank extraction (listrank.py:120-150)
template <class SuccT, class OutT>
__global__ void __launch_bounds__(1024) k_wy_single(const SuccT* __restrict__ succ, unsigned long long* word,
                                                    unsigned long long n, ListStatus* st, OutT* __restrict__ rank,
                                                    int rounds) {
    for (unsigned long long i = threadIdx.x; i < n; i += blockDim.x) {
        unsigned long long v = as_index<SuccT>(succ[i]);
        note_succ(st, i, v, n);
        if (v >= n) v = i;
        word[i] = ((unsigned long long)(v != i) << 32) | v;
    }
    __threadfence();
    __syncthreads();
    const uint32_t tail = wy_tail(st);
    for (int r = 0; r < rounds; ++r) {
        for (unsigned long long i = threadIdx.x; i < n; i += blockDim.x) {
            unsigned long long w = __ldcg(word + i);
            const uint32_t s = (uint32_t)w;
            if (s != tail && (unsigned long long)s != i) {
                const unsigned long long w2 = __ldcg(word + s);
                const unsigned long long rk = ((w >> 32) + (w2 >> 32)) & 0xFFFFFFFFull;
                __stcg(word + i, (rk << 32) | (w2 & 0xFFFFFFFFull));
            }
        }
        __syncthreads();
    }
    for (unsigned long long i = threadIdx.x; i < n; i += blockDim.x) rank[i] = (OutT)(__ldcg(word + i) >> 32);
    if (threadIdx.x == 0) {
        const unsigned long long w0 = __ldcg(word);
        st->head_ok = ((uint32_t)w0 == tail) ? 1ull : 0ull;
        st->head_sum = (w0 >> 32) + 1;
    }
}

// ---------------------------------------------------------------------------
// ruling set: census (+ validation at level 0), scan, select

template <class SuccT, bool kValidate>
__global__ void __launch_bounds__(TILE_THREADS) k_rs_count(const SuccT* __restrict__ succ,
                                                           uint32_t* __restrict__ tile_cnt, ListStatus* st,
                                                           int level, uint32_t kbits, uint32_t salt, int census) {
    const unsigned long long N = st->R[level];
    const unsigned long long base = (unsigned long long)blockIdx.x * TILE;
    if (base >= N) {
        if (threadIdx.x == 0 && census) tile_cnt[blockIdx.x] = 0;
        return;
    }
    uint32_t cnt = 0;
    if (kValidate) {
        // all loads first (the atomics below would otherwise serialise them)
        SuccT v[TILE_ITEMS];
#pragma unroll
        for (int j = 0; j < TILE_ITEMS; ++j) {
            const unsigned long long i = base + (unsigned long long)j * TILE_THREADS + threadIdx.x;
            v[j] = i < N ? __ldcs(succ + i) : SuccT(0);
        }
#pragma unroll
        for (int j = 0; j < TILE_ITEMS; ++j) {
            const unsigned long long i = base + (unsigned long long)j * TILE_THREADS + threadIdx.x;
            if (i < N) {
                const unsigned long long x = as_index<SuccT>(v[j]);
                if (x >= N || x == i) note_succ(st, i, x, N);
            }
        }
    }
    if (census) {
#pragma unroll
        for (int j = 0; j < TILE_ITEMS; ++j) {
            const unsigned long long i = base + (unsigned long long)j * TILE_THREADS + threadIdx.x;
            if (i < N) cnt += is_ruler((uint32_t)i, kbits, salt) ? 1u : 0u;
        }
    }
    if (census) {
        typedef cub::BlockReduce<uint32_t, TILE_THREADS> BR;
        __shared__ typename BR::TempStorage tmp;
        const uint32_t tot = BR(tmp).Sum(cnt);
        if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
    }
}

// level 0: validate the successors (range, self-loops), count rulers per tile
// and in-tile chain ends per tile (nodes whose successor leaves the tile, or
// the tail): the segment count of the tile contraction below.  Full tiles
// are read with 16-B vector loads; node ids are 32-bit (n < 2^32 - 1).
// kNarrow: 32-bit range check (u32 ids, or int32 ids with n <= 2^31, where a
// negative id reads as >= 2^31 >= n)
template <class SuccT, bool kVec, bool kNarrow>
__global__ void __launch_bounds__(TILE_THREADS) k_rs_count0(const SuccT* __restrict__ succ,
                                                            uint32_t* __restrict__ tile_cnt,
                                                            uint32_t* __restrict__ tile_end, ListStatus* st,
                                                            uint32_t kbits, uint32_t salt,
                                                            uint32_t* __restrict__ tile_run) {
    // one warp per tile (persistent warps): no block barrier between tiles, so
    // a warp's next loads never wait on its neighbours' reductions
    constexpr int VEC = 16 / sizeof(SuccT);  // ids per 16-B load
    constexpr int SUB = 4;                   // 16-B loads per lane in flight
    constexpr int PER = 32 * SUB * VEC;      // ids per warp step
    typedef typename std::conditional<sizeof(SuccT) == 4, uint4, ulonglong2>::type V;
    const unsigned long long N = st->R[0];
    const unsigned long long ntiles = (N + TILE - 1) / TILE;
    const uint32_t lane = lane_id();
    const uint32_t rT = 1u << (32u - kbits);  // ruler iff (i * PHI + salt) < rT, or i == 0 (is_ruler)
    const unsigned long long gw = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    for (unsigned long long tile = gw; tile < ntiles; tile += nw) {
        const unsigned long long base = tile * TILE;
        const bool full = kVec && base + TILE <= N;
        uint32_t packed = 0;  // rulers << 16 | ends
        // full tiles of 32-bit ids: branch-free counts, the range and
        // self-loop checks folded into one flag per lane (half the
        // instructions of the exact path: the census was issue-bound at 4.5
        // TB/s); a tile that raises the flag is re-scanned below with the
        // exact per-node report (note_succ)
#ifdef SG_COUNT0_EXACT_ONLY
        constexpr bool kFast = false;
#else
        constexpr bool kFast = kNarrow;
#endif
        bool exact = !(kFast && full);
        if (kFast && full) {
            const uint32_t Nn = (uint32_t)N, b32 = (uint32_t)base;
            uint32_t rul = 0, ends = 0;
            bool err = false, brk = false;  // brk: some successor is not the next id
#pragma unroll 1
            for (uint32_t s0 = 0; s0 < (uint32_t)TILE; s0 += PER) {
                V v[SUB];
                const V* src = reinterpret_cast<const V*>(succ + base + s0);
#pragma unroll
                for (int j = 0; j < SUB; ++j) v[j] = __ldcs(src + j * 32 + lane);
#pragma unroll
                for (int j = 0; j < SUB; ++j) {
                    const uint32_t i0 = b32 + s0 + (uint32_t)(j * 32 + lane) * VEC;
                    uint32_t h = i0 * PHI + salt;
#pragma unroll
                    for (int c = 0; c < VEC; ++c, h += PHI) {
                        const uint32_t x = (uint32_t)reinterpret_cast<const SuccT*>(&v[j])[c];
                        err |= (x >= Nn) | (x == i0 + c);
                        brk |= x != i0 + c + 1;
                        rul += h < rT ? 1u : 0u;
                        ends += (x - b32) >= (uint32_t)TILE ? 1u : 0u;
                    }
                }
            }
            exact = __any_sync(0xffffffffu, err);
            packed = (rul << 16) + ends;
            // a full tile whose every successor is the next id (its last node
            // continues into the next tile): the contraction takes it without
            // reading it again
            const bool run = !exact && !__any_sync(0xffffffffu, brk);
            if (lane == 0) tile_run[tile] = run ? 1u : 0u;
        } else if (lane == 0) {
            tile_run[tile] = 0u;
        }
        if (exact) {
            packed = 0;
#pragma unroll 1
            for (uint32_t s0 = 0; s0 < (uint32_t)TILE; s0 += PER) {
                SuccT e[SUB * VEC];
                if (full) {
                    const V* src = reinterpret_cast<const V*>(succ + base + s0);
#pragma unroll
                    for (int j = 0; j < SUB; ++j) {
                        const V v = __ldcs(src + j * 32 + lane);
#pragma unroll
                        for (int c = 0; c < VEC; ++c) e[j * VEC + c] = reinterpret_cast<const SuccT*>(&v)[c];
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < SUB; ++j)
#pragma unroll
                        for (int c = 0; c < VEC; ++c) {
                            const unsigned long long i = base + s0 + (unsigned long long)(j * 32 + lane) * VEC + c;
                            e[j * VEC + c] = i < N ? __ldcs(succ + i) : SuccT(0);
                        }
                }
#pragma unroll
                for (int j = 0; j < SUB; ++j) {
                    // ruler hash along the lane's VEC consecutive ids: h advances by PHI per id
                    // (is_ruler's (h >> (32 - kbits)) == 0 is h < 2^(32 - kbits); node 0 is added below)
                    uint32_t h = ((uint32_t)base + s0 + (uint32_t)(j * 32 + lane) * VEC) * PHI + salt;
#pragma unroll
                    for (int c = 0; c < VEC; ++c, h += PHI) {
                        const uint32_t l = s0 + (j * 32 + lane) * VEC + c;
                        if (full || base + l < N) {
                            const unsigned long long x64 = as_index<SuccT>(e[j * VEC + c]);
                            const uint32_t i = (uint32_t)base + l, x = (uint32_t)x64;
                            const bool oor = kNarrow ? x >= (uint32_t)N : x64 >= N;
                            const bool self = !oor && x == i;
                            if (oor | self) note_succ(st, i, x64, N);
                            packed += (h < rT ? 0x10000u : 0u) + ((oor | self | ((x ^ i) >= TILE)) ? 1u : 0u);
                        }
                    }
                }
            }
        }
        if (tile == 0 && lane == 0 && !(salt < rT)) packed += 0x10000u;  // node 0 is always a ruler
        const uint32_t tot = __reduce_add_sync(0xffffffffu, packed);
        if (lane == 0) {
            tile_cnt[tile] = tot >> 16;
            tile_end[tile] = tot & 0xFFFFu;
        }
    }
}

// Lists whose chains mostly stay inside their 4096-node tile (ordered or
// locally shuffled layouts) are contracted tile by tile in shared memory
// (k_rs_contract); scattered lists take the ruling-set record walk.
__device__ __forceinline__ bool layout_local(const ListStatus* st) { return st->local != 0; }
// the top level has found the list invalid (set before any rank is written):
// the passes that write ranks skip, so an aliased successor array
// (reuse_succ) survives for the host's violation report
__device__ __forceinline__ bool ranks_invalid(const ListStatus* st) {
    return st->overflow || st->bad || !st->head_ok || st->head_sum != st->R[0];
}

// Single-CTA exclusive scan of per-tile counts, in place, chunk by chunk
// with coalesced (transposed) loads and stores.  Returns the total.
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_CHUNK = SCAN_THREADS * SCAN_ITEMS;

struct ScanSmem {
    typedef cub::BlockLoad<uint32_t, SCAN_THREADS, SCAN_ITEMS, cub::BLOCK_LOAD_TRANSPOSE> BL;
    typedef cub::BlockStore<uint32_t, SCAN_THREADS, SCAN_ITEMS, cub::BLOCK_STORE_TRANSPOSE> BSt;
    typedef cub::BlockScan<unsigned long long, SCAN_THREADS> BSc;
    typedef cub::BlockReduce<unsigned long long, SCAN_THREADS> BR;
    union {
        typename BL::TempStorage load;
        typename BSt::TempStorage store;
        typename BSc::TempStorage scan;
        typename BR::TempStorage red;
    };
};

__device__ unsigned long long cta_sum(const uint32_t* __restrict__ a, unsigned long long cnt, ScanSmem& sm) {
    unsigned long long acc = 0;
    for (unsigned long long c0 = 0; c0 < cnt; c0 += SCAN_CHUNK) {
        const int valid = (int)min((unsigned long long)SCAN_CHUNK, cnt - c0);
        uint32_t v[SCAN_ITEMS];
        ScanSmem::BL(sm.load).Load(a + c0, v, valid, 0u);
        __syncthreads();
        unsigned long long x = 0;
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; ++j) x += v[j];
        acc += ScanSmem::BR(sm.red).Sum(x);
        __syncthreads();
    }
    return acc;  // valid in thread 0
}

__device__ unsigned long long cta_exclusive_scan(const uint32_t* src, uint32_t* dst, unsigned long long cnt,
                                                 ScanSmem& sm) {
    unsigned long long carry = 0;
    for (unsigned long long c0 = 0; c0 < cnt; c0 += SCAN_CHUNK) {
        const int valid = (int)min((unsigned long long)SCAN_CHUNK, cnt - c0);
        uint32_t v[SCAN_ITEMS];
        ScanSmem::BL(sm.load).Load(src + c0, v, valid, 0u);
        __syncthreads();
        unsigned long long x = 0;
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; ++j) x += v[j];
        unsigned long long pre, tot;
        ScanSmem::BSc(sm.scan).ExclusiveSum(x, pre, tot);
        __syncthreads();
        pre += carry;
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; ++j) {
            const uint32_t c = v[j];
            v[j] = (uint32_t)pre;
            pre += c;
        }
        ScanSmem::BSt(sm.store).Store(dst + c0, v, valid);
        __syncthreads();
        carry += tot;
    }
    return carry;
}

// level 0: pick the path and scan its tile counts.  Contraction when the
// in-tile segments are few (>= 16 nodes per segment on average) and fit the
// level-1 buffers; otherwise the hashed ruling set.
__global__ void __launch_bounds__(SCAN_THREADS) k_rs_scan0(uint32_t* tile_cnt, const uint32_t* __restrict__ tile_end,
                                                           ListStatus* st, unsigned long long cap, int allow_contract) {
    __shared__ ScanSmem sm;
    __shared__ int s_contract;
    const unsigned long long N = st->R[0];
    const unsigned long long ntiles = (N + TILE - 1) / TILE;
    const unsigned long long segs = cta_sum(tile_end, ntiles, sm);
    if (threadIdx.x == 0) s_contract = allow_contract && segs <= cap && segs * 16 <= N;
    __syncthreads();
    const int contract = s_contract;
    unsigned long long total = cta_exclusive_scan(contract ? tile_end : tile_cnt, tile_cnt, ntiles, sm);
    if (threadIdx.x == 0) {
        if (total > cap) {
            st->overflow = 1;
            total = cap;
        }
        st->R[1] = total;
        st->local = contract ? 1ull : 0ull;
    }
}

// single CTA exclusive scan of the tile counts of `level`
__global__ void __launch_bounds__(SCAN_THREADS) k_rs_scan(uint32_t* tile_cnt, ListStatus* st, int level,
                                                          unsigned long long cap) {
    __shared__ ScanSmem sm;
    const unsigned long long N = st->R[level];
    const unsigned long long ntiles = (N + TILE - 1) / TILE;
    unsigned long long total = cta_exclusive_scan(tile_cnt, tile_cnt, ntiles, sm);
    if (threadIdx.x == 0) {
        if (total > cap) {
            st->overflow = 1;
            total = cap;
        }
        st->R[level + 1] = total;
    }
}

// install ruler ids in index order: spl[id] = node, word[node] = id << 32
// (level 0: the packed array keeps the successor in the low half)
// Level 0 keeps no per-node id array: rgrp[g] = {ruler mask of the 32 ids
// 32g..32g+31, id of the first ruler at or after 32g}, so a walk that hits
// ruler x reads one 8-B word (an L2-resident n/4-byte table) instead of a
// random 4-B id -- and this pass writes the table coalesced instead of
// scattering n/32 ids.
__device__ __forceinline__ uint32_t ruler_id(const uint2* __restrict__ rgrp, uint32_t x) {
    const uint2 g = __ldg(rgrp + (x >> 5));
    return g.y + __popc(g.x & ((1u << (x & 31u)) - 1u));
}

template <bool kPacked>
__global__ void __launch_bounds__(TILE_THREADS) k_rs_select(const uint32_t* __restrict__ tile_off,
                                                            uint32_t* __restrict__ spl,
                                                            unsigned long long* __restrict__ word,
                                                            const ListStatus* st, int level, uint32_t kbits,
                                                            uint32_t salt, unsigned long long cap,
                                                            uint2* __restrict__ rgrp) {
    if (level == 0 && layout_local(st)) return;  // k_rs_contract takes this list
    const unsigned long long N = st->R[level];
    const unsigned long long ntiles = (N + TILE - 1) / TILE;
    typedef cub::BlockScan<uint32_t, TILE_THREADS> BS;
    __shared__ typename BS::TempStorage tmp;
    static_assert(TILE_ITEMS == 16, "two threads per 32-id group");
    for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const unsigned long long base = tile * TILE;
        const unsigned long long i0 = base + (unsigned long long)threadIdx.x * TILE_ITEMS;
        // ruler test along the run: h = i * PHI + salt advances by PHI per id,
        // and (h >> (32 - kbits)) == 0 is h < 2^(32 - kbits) (is_ruler)
        uint32_t flags = 0;
        const uint32_t T = 1u << (32u - kbits);
        uint32_t h = (uint32_t)i0 * PHI + salt;
#pragma unroll
        for (int j = 0; j < TILE_ITEMS; ++j) {
            flags |= (h < T ? 1u : 0u) << j;
            h += PHI;
        }
        if (i0 == 0) flags |= 1u;  // node 0 is always a ruler
        if (i0 + TILE_ITEMS > N) flags &= i0 >= N ? 0u : (1u << (uint32_t)(N - i0)) - 1u;
        uint32_t pre;
        BS(tmp).ExclusiveSum((uint32_t)__popc(flags), pre);
        unsigned long long id = (unsigned long long)tile_off[tile] + pre;
        if (rgrp != nullptr) {
            const uint32_t hi = __shfl_down_sync(0xffffffffu, flags, 1);
            if ((threadIdx.x & 1) == 0 && i0 < N) rgrp[i0 >> 5] = make_uint2(flags | (hi << 16), (uint32_t)id);
        }
        for (uint32_t rem = flags; rem != 0; rem &= rem - 1, ++id) {
            const uint32_t j = __ffs(rem) - 1;
            if (id < cap) {
                spl[id] = (uint32_t)(i0 + j);
                if (rgrp == nullptr)
                    word[i0 + j] = kPacked ? ((id << 32) | (word[i0 + j] & 0xFFFFFFFFull)) : (id << 32);
            }
        }
        __syncthreads();
    }
}

// Level-0 ruler ids, one warp per 4096-node tile (no block barrier): lane l
// owns ids [l*128, (l+1)*128) of the tile as four 32-id groups, hashes them
// along the run, and a warp scan of the lanes' ruler counts gives every
// group its first id -> rgrp {mask, first id} (a warp writes 1 KiB
// contiguously) and spl[id] = node for the rulers.
__global__ void __launch_bounds__(256) k_rs_select0(const uint32_t* __restrict__ tile_off, uint32_t* __restrict__ spl,
                                                    const ListStatus* st, uint32_t kbits, uint32_t salt,
                                                    unsigned long long cap, uint2* __restrict__ rgrp) {
    if (layout_local(st)) return;  // k_rs_contract takes this list
    static_assert(TILE == 32 * 128, "a lane owns 128 ids of a tile");
    const unsigned long long N = st->R[0];
    const unsigned long long ntiles = (N + TILE - 1) / TILE;
    const uint32_t lane = lane_id();
    const uint32_t T = 1u << (32u - kbits);
    const unsigned long long gw = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    for (unsigned long long tile = gw; tile < ntiles; tile += nw) {
        const unsigned long long i0 = tile * TILE + (unsigned long long)lane * 128;
        uint32_t m[4], cnt = 0;
        uint32_t h = (uint32_t)i0 * PHI + salt;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            uint32_t f = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j, h += PHI) f |= (h < T ? 1u : 0u) << j;
            const unsigned long long gb = i0 + (unsigned long long)g * 32;
            if (gb == 0) f |= 1u;  // node 0 is always a ruler
            if (gb + 32 > N) f &= gb >= N ? 0u : (1u << (uint32_t)(N - gb)) - 1u;
            m[g] = f;
            cnt += __popc(f);
        }
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += y;
        }
        unsigned long long id = (unsigned long long)tile_off[tile] + (incl - cnt);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const unsigned long long gb = i0 + (unsigned long long)g * 32;
            if (gb < N) rgrp[gb >> 5] = make_uint2(m[g], (uint32_t)id);
            for (uint32_t rem = m[g]; rem != 0; rem &= rem - 1, ++id)
                if (id < cap) spl[id] = (uint32_t)(gb + (__ffs(rem) - 1));
        }
    }
}

// ---------------------------------------------------------------------------
// sublist walk (RS3 at level 0, weighted RS4 walk above)
//
// Lanes pull rulers from a global queue (warp-aggregated atomics), so a long
// sublist never holds a whole warp's share of work hostage.

// Warp-local pool of ruler ids: a warp claims QBATCH rulers from the level's
// global queue with one atomic and hands them to its lanes as their chains
// end.  (One atomic per refill from every warp serialised the walk on the
// queue head: half of all stall samples sat on that broadcast.)
constexpr uint32_t QBATCH = 64;  // >= 32: one refill must cover a whole warp's request

struct ChainPool {
    unsigned long long base = 0;   // next unclaimed id in the warp's batch (warp-uniform)
    uint32_t left = 0;             // ids left in the batch (warp-uniform)

    // lanes with `need` get an id < R (or none once the queue is dry);
    // returns the lane's id or ~0ull
    __device__ __forceinline__ unsigned long long take(bool need, unsigned long long* q, unsigned long long R,
                                                       uint32_t lane) {
        const unsigned m = __ballot_sync(0xffffffffu, need);
        if (m == 0) return ~0ull;
        const uint32_t cnt = __popc(m);
        const uint32_t r = __popc(m & ((1u << lane) - 1u));
        unsigned long long id;
        if (cnt <= left) {
            id = base + r;
            base += cnt;
            left -= cnt;
        } else {
            unsigned long long nb = 0;
            if (lane == 0) nb = atomicAdd(q, (unsigned long long)QBATCH);
            nb = __shfl_sync(0xffffffffu, nb, 0);
            id = r < left ? base + r : nb + (r - left);
            const uint32_t used_new = cnt - left;
            base = nb + used_new;
            left = QBATCH - used_new;
        }
        return (need && id < R) ? id : ~0ull;
    }
};

template <class View>
__global__ void __launch_bounds__(WALK_THREADS) k_rs_walk(View src, unsigned long long* __restrict__ word,
                                                          const uint32_t* __restrict__ spl,
                                                          uint2* __restrict__ up, ListStatus* st, int level,
                                                          uint32_t kbits, uint32_t salt, uint32_t cap_hops) {
    const unsigned long long N = st->R[level];
    const unsigned long long R = st->R[level + 1];
    unsigned long long* q = &st->qhead[level];
    const uint32_t lane = lane_id();
    uint32_t sid = NIL, cur = 0, pre = 0, hops = 0;
    bool done = false;
    ChainPool pool;
    for (;;) {
        const bool need = !done && sid == NIL;
        const unsigned long long s = pool.take(need, q, R, lane);
        if (need) {
            if (s != ~0ull) {
                sid = (uint32_t)s;
                cur = spl[s];
                pre = 0;
                hops = 0;
            } else {
                done = true;
            }
        }
        if (__all_sync(0xffffffffu, done)) break;
        if (done) continue;
        word[cur] = ((unsigned long long)sid << 32) | pre;
        unsigned long long nx;
        uint32_t w;
        src.load(cur, nx, w);
        pre += w;
        ++hops;
        if (nx == cur) {  // the tail: end of the whole list
            up[sid] = make_uint2(sid, pre);
            sid = NIL;
        } else if (nx >= N) {  // out-of-range successor (invalid input)
            st->bad = 1;
            up[sid] = make_uint2(sid, pre);
            sid = NIL;
        } else if (is_ruler((uint32_t)nx, kbits, salt)) {
            up[sid] = make_uint2((uint32_t)(word[nx] >> 32), pre);
            sid = NIL;
        } else if (hops >= cap_hops) {
            st->overflow = 1;
            up[sid] = make_uint2(sid, pre);
            sid = NIL;
        } else {
            cur = (uint32_t)nx;
        }
    }
}

// ---------------------------------------------------------------------------
// Level-0 record walk (scattered layouts).
//
// HBM serves ~40 G random 64-B atoms/s on this part (tools/ubench_random.cu)
// whether they are dependent or not, and a random partial store costs a
// read-modify-write on top.  So the walk only *reads* at random -- succ[cur],
// one atom per hop -- and appends {cur, sid, local} records contiguously per
// warp (all active lanes of a warp emit one record per step, compacted with a
// ballot), i.e. as full-line streaming writes.  Each warp owns 1024-record
// chunks.  The node-order materialisation of the ranks follows in the window
// passes (rs5_partition / rs5_refine / rs5_scatter).

constexpr int REC_CH = 1024;

// kPacked: one u64 record {cur : 64-sb | sid : sb-lb | local : lb} instead of
// cur u32 + {sid, local} u64 (the host picks the field widths from n)
template <class SuccT, bool kPacked>
__global__ void __launch_bounds__(WALK_THREADS, 2048 / WALK_THREADS) k_rs_walk_rec(const SuccT* __restrict__ succ,
                                                              const uint2* __restrict__ rgrp,
                                                              const uint32_t* __restrict__ spl,
                                                              uint2* __restrict__ up, uint32_t* __restrict__ rec_cur,
                                                              unsigned long long* __restrict__ rec_sl,
                                                              ListStatus* st, uint32_t kbits, uint32_t salt,
                                                              uint32_t cap_hops, unsigned long long maxchunks,
                                                              int load_mode, uint32_t sb, uint32_t lb) {
    if (layout_local(st)) return;  // k_rs_contract takes this list
    const unsigned long long N = st->R[0];
    const unsigned long long R = st->R[1];
    unsigned long long* q = &st->qhead[0];
    const uint32_t lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    unsigned long long chunk = ~0ull;  // warp-uniform
    uint32_t fill = REC_CH;            // warp-uniform: records used in the current chunk
    uint32_t sid = NIL, cur = 0, pre = 0;
    bool done = false;
    auto close_chunk = [&]() {  // pad the tail with NIL records
        if (chunk == ~0ull) return;
        for (uint32_t k = fill + lane; k < REC_CH; k += 32) {
            if (kPacked)
                rec_sl[chunk * REC_CH + k] = ~0ull;
            else
                rec_cur[chunk * REC_CH + k] = NIL;
        }
    };
    ChainPool pool;
    for (;;) {
        const bool need = !done && sid == NIL;
        const unsigned long long s = pool.take(need, q, R, lane);
        if (need) {
            if (s != ~0ull) {
                sid = (uint32_t)s;
                cur = spl[s];
                pre = 0;
            } else {
                done = true;
            }
        }
        const unsigned act = __ballot_sync(0xffffffffu, !done);
        if (act == 0) break;
        unsigned long long nxl = 0;
        if (!done) nxl = as_index<SuccT>(ld_mode(succ + cur, load_mode));
        // append this step's records, warp-contiguous
        const uint32_t cnt = __popc(act);
        if (fill + cnt > REC_CH) {
            close_chunk();
            unsigned long long c = 0;
            if (lane == 0) c = atomicAdd(&st->chunks, 1ull);
            chunk = __shfl_sync(0xffffffffu, c, 0);
            fill = 0;
            if (chunk >= maxchunks) {  // cannot happen for valid inputs; fall back to Wyllie
                if (lane == 0) st->overflow = 1;
                chunk = ~0ull;
                return;
            }
        }
        if (!done) {
            const unsigned long long r = chunk * REC_CH + fill + __popc(act & lt);
            if (kPacked) {
                rec_sl[r] = ((unsigned long long)cur << sb) | ((unsigned long long)sid << lb) | pre;
            } else {
                rec_cur[r] = cur;
                rec_sl[r] = ((unsigned long long)sid << 32) | pre;
            }
        }
        fill += cnt;
        if (!done) {
            ++pre;
            bool end = true;
            uint2 upv = make_uint2(sid, pre);
            if (nxl == cur) {  // the tail
            } else if (nxl >= N) {  // out-of-range successor (invalid input)
                st->bad = 1;
            } else if (is_ruler((uint32_t)nxl, kbits, salt)) {
                upv.x = ruler_id(rgrp, (uint32_t)nxl);
            } else if (pre >= cap_hops) {
                st->overflow = 1;
            } else {
                end = false;
                cur = (uint32_t)nxl;
            }
            if (end) {
                up[sid] = upv;
                sid = NIL;
            }
        }
    }
    close_chunk();
}

// Level-0 walk that bins its records by coarse output window on the fly
// (packed records only), so the rs5_partition pass disappears.  The walk is
// bound by the dependent random load; the binning runs in its shadow.  Each
// CTA keeps WB_SLOTS records per coarse window in shared memory:
//   reserve  res[b]++ (a lane that finds the buffer full retries next round),
//   store    the record into the reserved slot, then commit com[b]++;
//   flush    the lane whose commit completes the buffer hands it to its warp,
//            which claims WB_SLOTS slots of window b's region with one global
//            atomic and writes them as one 256-B run, then reopens the buffer
//            (com = 0 before res = 0: a reserver that sees res reopened also
//            sees com reset).
// A valid list puts exactly 2^cshift records into each full window, so the
// regions are known in advance; an invalid list can overfill one -- those
// records are dropped and the call is flagged (it reports the list invalid).
constexpr uint32_t WB_MAXBINS = 256;

template <class SuccT, int WB_THREADS, int WB_CTAS_PER_SM, uint32_t WB_SLOTS>
__global__ void __launch_bounds__(WB_THREADS, WB_CTAS_PER_SM) k_rs_walk_bin(
    const SuccT* __restrict__ succ, const uint2* __restrict__ rgrp, const uint32_t* __restrict__ spl,
    uint2* __restrict__ up, unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ out,
    ListStatus* st, uint32_t kbits, uint32_t salt, uint32_t cap_hops, int load_mode, uint32_t sb, uint32_t lb,
    uint32_t cshift, uint32_t cbins) {
    if (layout_local(st)) return;  // k_rs_contract takes this list
    extern __shared__ __align__(16) unsigned long long buf[];  // [cbins][WB_SLOTS]
    __shared__ uint32_t res[WB_MAXBINS], com[WB_MAXBINS];
    for (uint32_t i = threadIdx.x; i < cbins; i += blockDim.x) res[i] = com[i] = 0;
    __syncthreads();
    const unsigned long long N = st->R[0];
    const unsigned long long R = st->R[1];
    const unsigned long long wsize = 1ull << cshift;
    unsigned long long* q = &st->qhead[0];
    const uint32_t lane = lane_id();
    bool over = false;
    // warp-cooperative copy of `cnt` records of bin b into its window, claimed at `base`
    auto store_run = [&](uint32_t b, uint32_t cnt, unsigned long long base, uint32_t k) {
        if (k < cnt) {
            const unsigned long long v = buf[b * WB_SLOTS + k];
            if (base + k < wsize)
                __stcs(out + ((unsigned long long)b << cshift) + base + k, v);
            else
                over = true;
        }
    };
    uint32_t sid = NIL, cur = 0, pre = 0;
    bool done = false;
    ChainPool pool;
    for (;;) {
        const bool need = !done && sid == NIL;
        const unsigned long long s = pool.take(need, q, R, lane);
        if (need) {
            if (s != ~0ull) {
                sid = (uint32_t)s;
                cur = spl[s];
                pre = 0;
            } else {
                done = true;
            }
        }
        if (__all_sync(0xffffffffu, done)) break;
        unsigned long long nxl = 0;
        if (!done) nxl = as_index<SuccT>(ld_mode(succ + cur, load_mode));
        // place this step's record while the load is in flight
        bool pend = !done;
        const uint32_t b = cur >> cshift;
        const unsigned long long recv = ((unsigned long long)cur << sb) | ((unsigned long long)sid << lb) | pre;
        while (__any_sync(0xffffffffu, pend)) {
            bool last = false;
            if (pend) {
                const uint32_t pos = atomicAdd(&res[b], 1u);
                if (pos < WB_SLOTS) {
                    buf[b * WB_SLOTS + pos] = recv;
                    __threadfence_block();
                    last = atomicAdd(&com[b], 1u) == WB_SLOTS - 1;
                    pend = false;
                }
            }
            unsigned m = __ballot_sync(0xffffffffu, last);
            if (m == 0) continue;
            __threadfence_block();
            // all full buffers of this warp: claim their runs together, then copy one per pass
            unsigned long long base = 0;
            if (last) base = atomicAdd(&cursor[b], (unsigned long long)WB_SLOTS);
            while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t fb = __shfl_sync(0xffffffffu, b, src);
                const unsigned long long fbase = __shfl_sync(0xffffffffu, base, src);
                for (uint32_t k = lane; k < WB_SLOTS; k += 32) store_run(fb, WB_SLOTS, fbase, k);
                __syncwarp();
                if (lane == 0) {
                    atomicExch(&com[fb], 0u);
                    __threadfence_block();
                    atomicExch(&res[fb], 0u);
                }
                __syncwarp();
            }
        }
        if (!done) {
            ++pre;
            bool end = true;
            uint2 upv = make_uint2(sid, pre);
            if (nxl == cur) {  // the tail
            } else if (nxl >= N) {  // out-of-range successor (invalid input)
                st->bad = 1;
            } else if (is_ruler((uint32_t)nxl, kbits, salt)) {
                upv.x = ruler_id(rgrp, (uint32_t)nxl);
            } else if (pre >= cap_hops) {
                st->overflow = 1;
            } else {
                end = false;
                cur = (uint32_t)nxl;
            }
            if (end) {
                up[sid] = upv;
                sid = NIL;
            }
        }
    }
    // drain the partial buffers: one warp per bin
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5;
    for (uint32_t bb = warp; bb < cbins; bb += WB_THREADS / 32) {
        const uint32_t cnt = com[bb];
        if (cnt == 0) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&cursor[bb], (unsigned long long)cnt);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (uint32_t k = lane; k < cnt; k += 32) store_run(bb, cnt, base, k);
    }
    if (__any_sync(0xffffffffu, over) && lane == 0) st->bad = 1;
}

// Node-order materialisation of the ranks in three streaming passes.  For a
// valid list every node appears in exactly one record, so every output window
// receives exactly its own node count: window w of 2^shift nodes owns the
// slots [w << shift, (w + 1) << shift) of the next buffer.
//   rs5_partition: record -> {cur, rank} pair, by coarse window (<= MS_MAXB bins)
//   rs5_refine:    coarse window -> fine windows (2^fshift nodes)
//   rs5_scatter:   one CTA per fine window: shared memory -> coalesced ranks
// Both bucketing passes are ballot multisplits (sg_msplit.cuh).  Invalid
// inputs can overfill a window; such writes are dropped (the call reports
// the list invalid anyway).

// TMA-staged versions (persistent, 2 CTAs per SM): the next 4096-element
// tile streams into shared memory while the current one is split.

template <int IT, bool kPacked>
__global__ void __launch_bounds__(MS_THREADS, IT >= 16 ? 2 : 3) k_rs_rec_partition2(
    const uint32_t* __restrict__ rec_cur, const unsigned long long* __restrict__ rec_sl,
    const uint32_t* __restrict__ IS1, unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ pairs,
    ListStatus* st, uint32_t cshift, uint32_t cbins, uint32_t sb, uint32_t lb) {
    if (layout_local(st) || st->overflow) return;
    extern __shared__ __align__(128) unsigned char ms_raw[];
    uint32_t* s_cur = reinterpret_cast<uint32_t*>(ms_raw);
    unsigned long long* s_sl = reinterpret_cast<unsigned long long*>(ms_raw + (MS_THREADS * IT) * 4);
    MsSmem sm = MsSmem::carve(ms_raw + (MS_THREADS * IT) * 12, cbins, (MS_THREADS * IT));
    __shared__ unsigned long long bar;
    const unsigned long long total = st->chunks * REC_CH;  // a multiple of REC_CH
    const unsigned long long ntiles = (total + (MS_THREADS * IT) - 1) / (MS_THREADS * IT);
    const unsigned long long R1 = st->R[1];
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    auto issue = [&](unsigned long long tile) {
        if (threadIdx.x == 0 && tile < ntiles) {
            const unsigned long long e0 = tile * (MS_THREADS * IT);
            const uint32_t cnt = (uint32_t)min((unsigned long long)(MS_THREADS * IT), total - e0);
            if (kPacked) {
                mbar_expect_tx(&bar, cnt * 8u);
                bulk_g2s(s_sl, rec_sl + e0, cnt * 8u, &bar);
            } else {
                mbar_expect_tx(&bar, cnt * 12u);
                bulk_g2s(s_cur, rec_cur + e0, cnt * 4u, &bar);
                bulk_g2s(s_sl, rec_sl + e0, cnt * 8u, &bar);
            }
        }
    };
    auto bin_of = [&](unsigned long long pr) { return (uint32_t)((pr >> 32) >> cshift); };
    auto slot = [&](uint32_t b) { return make_ulonglong2((unsigned long long)b << cshift, 1ull << cshift); };
    bool over = false;
    uint32_t phase = 0;
    issue(blockIdx.x);
    for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t cnt = (uint32_t)min((unsigned long long)(MS_THREADS * IT), total - tile * (MS_THREADS * IT));
        mbar_wait(&bar, phase);
        phase ^= 1u;
        unsigned long long pr[IT];
        uint32_t bn[IT];
#pragma unroll
        for (int g = 0; g < IT / 4; ++g) {
            const uint32_t e = (g * MS_THREADS + threadIdx.x) * 4;  // 4 records per vector access
            if (kPacked) {
                const ulonglong2 r01 = e < cnt ? reinterpret_cast<const ulonglong2*>(s_sl)[e >> 1] : make_ulonglong2(~0ull, ~0ull);
                const ulonglong2 r23 = e < cnt ? reinterpret_cast<const ulonglong2*>(s_sl)[(e >> 1) + 1] : make_ulonglong2(~0ull, ~0ull);
                const unsigned long long rr[4] = {r01.x, r01.y, r23.x, r23.y};
                const unsigned long long smask = (1ull << (sb - lb)) - 1, lmask = (1ull << lb) - 1;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int j = g * 4 + q;
                    const bool nil = rr[q] == ~0ull;
                    const unsigned long long o = (rr[q] >> lb) & smask;
                    pr[j] = ((unsigned long long)(nil ? NIL : (uint32_t)(rr[q] >> sb)) << 32) | (uint32_t)(rr[q] & lmask);
                    bn[j] = __ldg(IS1 + (o < R1 ? o : 0));
                }
                continue;
            }
            const uint4 c4 = e < cnt ? reinterpret_cast<const uint4*>(s_cur)[e >> 2] : make_uint4(NIL, NIL, NIL, NIL);
            const ulonglong2 s01 = e < cnt ? reinterpret_cast<const ulonglong2*>(s_sl)[e >> 1] : make_ulonglong2(0, 0);
            const ulonglong2 s23 = e < cnt ? reinterpret_cast<const ulonglong2*>(s_sl)[(e >> 1) + 1] : make_ulonglong2(0, 0);
            const uint32_t cc[4] = {c4.x, c4.y, c4.z, c4.w};
            const unsigned long long sl[4] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = g * 4 + q;
                const unsigned long long o = sl[q] >> 32;
                pr[j] = ((unsigned long long)cc[q] << 32) | (uint32_t)sl[q];
                bn[j] = __ldg(IS1 + (o < R1 ? o : 0));  // gathers first, all in flight together
            }
        }
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t c = (uint32_t)(pr[j] >> 32);
            const uint32_t local = (uint32_t)pr[j];
            // rank = IS_1[sid] - local - 1 (listrank.py:375-379)
            pr[j] = ((unsigned long long)c << 32) | (bn[j] - local - 1u);
            const uint32_t b = c >> cshift;
            bn[j] = (c != NIL && b < cbins) ? b : (uint32_t)MS_MAXB;
        }
        __syncthreads();  // staging consumed: refill it behind the split
        issue(tile + gridDim.x);
        over |= ms_split<IT, 8>(pr, bn, bin_of, slot, cbins, cursor, pairs, sm);
    }
    if (over) st->bad = 1;
}

// kMode 0: {cur, rank} pairs in and out.  kMode 1: packed walk records
// binned by k_rs_walk_bin in, ranked here (rank = IS_1[sid] - local - 1,
// listrank.py:375-379), pairs out.  (Ranking them in rs5_scatter instead
// measured slower: the IS_1 gather costs the same ~0.8 ms at 2^28 wherever it
// runs -- it is bound by L2 sector reads -- and rs5_scatter has less to hide it behind.)
template <int IT, int kMode, int NB = 8>  // NB: bits of the fine bin (>= cshift - fshift)
__global__ void __launch_bounds__(MS_THREADS, IT >= 16 ? 2 : 3) k_rs_rec_refine2(
    const unsigned long long* __restrict__ in, unsigned long long* __restrict__ cursor,
    unsigned long long* __restrict__ out, ListStatus* st, unsigned long long n, uint32_t cshift, uint32_t fshift,
    const uint32_t* __restrict__ IS1, uint32_t sb, uint32_t lb) {
    if (layout_local(st) || st->overflow) return;
    const uint32_t fb = 1u << (cshift - fshift);
    extern __shared__ __align__(128) unsigned char ms_raw[];
    unsigned long long* s_in = reinterpret_cast<unsigned long long*>(ms_raw);
    MsSmem sm = MsSmem::carve(ms_raw + (MS_THREADS * IT) * 8, fb, (MS_THREADS * IT));
    __shared__ unsigned long long bar;
    // tiles never straddle a coarse window (2^cshift is a multiple of (MS_THREADS * IT))
    const unsigned long long ntiles = (n + (MS_THREADS * IT) - 1) / (MS_THREADS * IT);
    const unsigned long long R1 = st->R[1];
    const unsigned long long pol_last = l2_evict_last();
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    auto issue = [&](unsigned long long tile) {
        if (threadIdx.x == 0 && tile < ntiles) {
            const unsigned long long e0 = tile * (MS_THREADS * IT);
            const uint32_t cnt = (uint32_t)min((unsigned long long)(MS_THREADS * IT), n - e0);
            const uint32_t bytes = (cnt * 8u + 15u) & ~15u;  // the buffer is padded to whole windows
            mbar_expect_tx(&bar, bytes);
            bulk_g2s_hint(s_in, in + e0, bytes, &bar, l2_evict_first());
        }
    };
    bool over = false;
    uint32_t phase = 0;
    issue(blockIdx.x);
    for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const unsigned long long e0 = tile * (MS_THREADS * IT);
        const uint32_t cnt = (uint32_t)min((unsigned long long)(MS_THREADS * IT), n - e0);
        const unsigned long long c = e0 >> cshift;
        mbar_wait(&bar, phase);
        phase ^= 1u;
        unsigned long long pr[IT];
        uint32_t bn[IT], gv[IT];
#pragma unroll
        for (int g = 0; g < IT / 2; ++g) {
            const uint32_t e = (g * MS_THREADS + threadIdx.x) * 2;
            const ulonglong2 v = e < cnt ? reinterpret_cast<const ulonglong2*>(s_in)[e >> 1] : make_ulonglong2(0, 0);
            const unsigned long long vv[2] = {v.x, v.y};
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int j = g * 2 + q;
                pr[j] = vv[q];
                // kMode 1: the IS_1 gather is issued here and first used when
                // the tile is placed, so it flies while the ballots rank it
                const unsigned long long cur = kMode == 1 ? (vv[q] >> sb) : (vv[q] >> 32);
                if (kMode == 1) {
                    const unsigned long long o = (vv[q] >> lb) & ((1ull << (sb - lb)) - 1);
                    gv[j] = ld_hint(IS1 + (o < R1 ? o : 0), pol_last);
                }
                bn[j] = (e + q < cnt && (cur >> cshift) == c) ? (uint32_t)((cur >> fshift) & (fb - 1))
                                                             : (uint32_t)MS_MAXB;
            }
        }
        __syncthreads();
        issue(tile + gridDim.x);
        auto bin_of = [&](unsigned long long pr) { return (uint32_t)(((pr >> 32) >> fshift) & (fb - 1)); };
        auto slot = [&](uint32_t b) { return make_ulonglong2((c * fb + b) << fshift, 1ull << fshift); };
        auto pair = [&](int j) -> unsigned long long {
            if (kMode != 1) return pr[j];
            const unsigned long long cur = pr[j] >> sb;
            return (cur << 32) | (uint32_t)(gv[j] - (uint32_t)(pr[j] & ((1ull << lb) - 1)) - 1u);
        };
        over |= ms_split_fn<IT, NB>(pair, bn, bin_of, slot, fb, cursor + c * fb, out, sm);
    }
    if (over) st->bad = 1;
}

// rs5_refine, lean (default for <= 64 fine bins).  Same job as
// k_rs_rec_refine2<.., 1, ..> -- coarse-window records -> {cur, rank} pairs
// split by fine window (rank = IS_1[sid] - local - 1, listrank.py:375-379) --
// written for the issue slots and the L1TEX pipe, which the IS_1 gathers
// already load to ~1 wavefront per record (tools/ubench_l2.cu: ~288 G random
// L2 sectors/s per GPU, 0.93 ms for 2^28 gathers):
//   * 32-bit slot and node arithmetic (a tile holds RL_TILE records; node
//     ids and window slots are < 2^32),
//   * peer ranking by ballots over the NB bin bits (or match.any, kPeers),
//     warp counters in shared memory touched by the group leaders only,
//   * one small pass turns the (warp, bin) counts into absolute tile slots,
//     so placing a record is one shared load and one shared store,
//   * runs leave the SM warp by warp, bin by bin (no per-record bin lookup).
// Persistent, 2 CTAs of 512 threads per SM; the next tile streams in
// (cp.async.bulk, evict-first) while the current one is split.
constexpr int RL_THREADS = 512;
constexpr int RL_WARPS = RL_THREADS / 32;
constexpr int RL_IT = 8;
constexpr int RL_TILE = RL_THREADS * RL_IT;  // 4096 records (2^cshift is a multiple)
constexpr int RL_MAXB = 64;                  // fine bins per coarse window handled here
constexpr int RL_CTAS_PER_SM = 2;

static size_t rl_smem_bytes() { return (size_t)RL_TILE * 8 * 2; }

// kTiles: the tile keeps its own slot range [tile * RL_TILE, ...) of `out`,
// sorted by fine bin, and its fb + 1 bin offsets go to toff[tile]; the
// scatter then collects a fine window's runs from the coarse window's tiles
// (k_rs_rec_scatter_tiles).  No global atomics, one linear 16-B copy out.
template <int NB, int kPeers, bool kTiles = false>  // NB: bin bits (fb <= 2^NB <= 64); kPeers: 1 ballots, 0 match.any, 2 alternate, 3 shared atomics
__global__ void __launch_bounds__(RL_THREADS, RL_CTAS_PER_SM) k_rs_refine_lean(
    const unsigned long long* __restrict__ in, unsigned long long* __restrict__ cursor,
    unsigned long long* __restrict__ out, ListStatus* st, unsigned long long n, uint32_t cshift, uint32_t fshift,
    const uint32_t* __restrict__ IS1, uint32_t sb, uint32_t lb, uint32_t* __restrict__ toff = nullptr) {
    if (layout_local(st) || st->overflow) return;
    const uint32_t fb = 1u << (cshift - fshift);  // <= 2^NB
    extern __shared__ __align__(128) unsigned char rl_raw[];
    unsigned long long* s_in = reinterpret_cast<unsigned long long*>(rl_raw);
    unsigned long long* s_sort = s_in + RL_TILE;
    __shared__ unsigned long long bar;
    __shared__ uint32_t s_w[RL_WARPS][RL_MAXB];  // per-warp bin counts -> absolute tile slots
    __shared__ uint32_t s_bs[RL_MAXB + 1];         // bin starts in the sorted tile
    __shared__ uint32_t s_gb[RL_MAXB];             // window slot of the bin's first tile record
    __shared__ uint32_t s_ge[RL_MAXB];             // tile end of the bin's writable run
    __shared__ uint32_t s_half;
    const uint32_t t = threadIdx.x, lane = lane_id(), warp = t >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned long long ntiles = (n + RL_TILE - 1) / RL_TILE;
    const uint32_t R1 = (uint32_t)min(st->R[1], (unsigned long long)0xFFFFFFFFu);
    const unsigned long long pol_last = l2_evict_last();
    const uint32_t fmask = fb - 1;
    const uint32_t lmask = (1u << lb) - 1u;            // lb < 32 (host-checked)
    const uint32_t smask = (uint32_t)((1ull << (sb - lb)) - 1);
    if (t == 0) mbar_init(&bar, 1);
    __syncthreads();
    auto issue = [&](unsigned long long tile) {
        if (t == 0 && tile < ntiles) {
            const unsigned long long e0 = tile * RL_TILE;
            const uint32_t cnt = (uint32_t)min((unsigned long long)RL_TILE, n - e0);
            const uint32_t bytes = (cnt * 8u + 15u) & ~15u;  // the buffer is padded to whole windows
            mbar_expect_tx(&bar, bytes);
            bulk_g2s_hint(s_in, in + e0, bytes, &bar, l2_evict_first());
        }
    };
    bool over = false;
    uint32_t phase = 0;
    issue(blockIdx.x);
    for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const unsigned long long e0 = tile * RL_TILE;
        const uint32_t cnt = (uint32_t)min((unsigned long long)RL_TILE, n - e0);
        const uint32_t c = (uint32_t)(e0 >> cshift);  // tiles never straddle a coarse window
        if (lane < (uint32_t)RL_MAXB / 2) {         // this warp's counters
            s_w[warp][lane] = 0u;
            s_w[warp][lane + RL_MAXB / 2] = 0u;
        }
        mbar_wait(&bar, phase);
        phase ^= 1u;
        uint32_t cur[RL_IT], gv[RL_IT], loc[RL_IT], bn[RL_IT];
#pragma unroll
        for (int g = 0; g < RL_IT / 2; ++g) {
            const uint32_t e = (g * RL_THREADS + t) * 2;
            const ulonglong2 v = e < cnt ? reinterpret_cast<const ulonglong2*>(s_in)[e >> 1] : make_ulonglong2(0, 0);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const unsigned long long r = q ? v.y : v.x;
                const int j = 2 * g + q;
                cur[j] = (uint32_t)(r >> sb);
                const uint32_t sid = (uint32_t)(r >> lb) & smask;
                loc[j] = (uint32_t)r & lmask;
                // issued now, first used at the placement: the gathers fly while the tile is ranked
                gv[j] = ld_hint(IS1 + (sid < R1 ? sid : 0u), pol_last);
                bn[j] = (e + q < cnt && (cur[j] >> cshift) == c) ? (cur[j] >> fshift) & fmask : 0xFFu;
            }
        }
        __syncthreads();  // staging consumed, counters zeroed
        issue(tile + gridDim.x);
        // rank among the warp's records of the same bin: rk = warp counter before + peers below
#pragma unroll
        for (int j = 0; j < RL_IT; ++j) {
            if (kPeers == 3) {  // shared atomics on the warp's counters: one ATOMS per record, any order in a bin
                if (bn[j] != 0xFFu) loc[j] |= atomicAdd(&s_w[warp][bn[j]], 1u) << 20;
                continue;
            }
            unsigned peers;
            if (kPeers == 0 || (kPeers == 2 && (j & 1))) {
                peers = __match_any_sync(0xffffffffu, bn[j]);
            } else {
                const bool valid = bn[j] != 0xFFu;
                const unsigned vb = __ballot_sync(0xffffffffu, valid);
                peers = valid ? vb : ~vb;
#pragma unroll
                for (int k = 0; k < NB; ++k) {
                    const unsigned b = __ballot_sync(0xffffffffu, (bn[j] >> k) & 1u);
                    peers &= ((bn[j] >> k) & 1u) ? b : ~b;
                }
            }
            const int leader = __ffs(peers) - 1;
            uint32_t old = 0;
            if (bn[j] != 0xFFu && (int)lane == leader) {
                old = s_w[warp][bn[j]];
                s_w[warp][bn[j]] = old + __popc(peers);
            }
            loc[j] |= (__shfl_sync(0xffffffffu, old, leader) + __popc(peers & lt)) << 20;  // local < 2^12
        }
        __syncthreads();
        // (warp, bin) counts -> absolute slots of the bin-sorted tile; one
        // atomic per non-empty bin claims the bin's run in its fine window
        if (t < 64) {
            const uint32_t d = t;
            uint32_t tot = 0;
            if (d < fb) {
#pragma unroll
                for (int w = 0; w < RL_WARPS; ++w) {
                    const uint32_t x = s_w[w][d];
                    s_w[w][d] = tot;
                    tot += x;
                }
            }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += y;
            }
            if (t == 31) s_half = incl;
            asm volatile("bar.sync 1, 64;" ::: "memory");
            const uint32_t start = incl - tot + (t >= 32 ? s_half : 0u);
            if (d < fb) {
#pragma unroll
                for (int w = 0; w < RL_WARPS; ++w) s_w[w][d] += start;
                if (kTiles) {
                    uint32_t* to = toff + tile * (fb + 1);
                    to[d] = start;
                    if (d == fb - 1) to[fb] = start + tot;
                }
                uint32_t base = 0;
                if (!kTiles && tot)
                    base = (uint32_t)atomicAdd(cursor + (unsigned long long)c * fb + d, (unsigned long long)tot);
                const uint32_t cap = 1u << fshift;
                const uint32_t room = base < cap ? cap - base : 0u;
                s_bs[d] = start;
                s_gb[d] = base;
                s_ge[d] = start + (tot < room ? tot : room);
                if (d == fb - 1) s_bs[fb] = start + tot;
            }
        }
        __syncthreads();
        // place: slot = absolute (warp, bin) slot + rank within the warp
#pragma unroll
        for (int j = 0; j < RL_IT; ++j) {
            if (bn[j] != 0xFFu) {
                const uint32_t pos = s_w[warp][bn[j]] + (loc[j] >> 20);
                const uint32_t rank = gv[j] - (loc[j] & 0xFFFFFu) - 1u;
                s_sort[pos] = ((unsigned long long)cur[j] << 32) | rank;
            }
        }
        __syncthreads();
        if (kTiles) {  // the sorted tile, as is, to its own slots
            const uint32_t total = s_bs[fb];
            ulonglong2* dst = reinterpret_cast<ulonglong2*>(out + e0);
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(s_sort);
            for (uint32_t i = t; i < total / 2; i += RL_THREADS) __stcs(dst + i, src[i]);
            if ((total & 1u) && t == 0) __stcs(out + e0 + total - 1, s_sort[total - 1]);
            __syncthreads();
            continue;
        }
        // write out: warp w copies the runs of bins w, w + RL_WARPS, ...
        unsigned long long* wout = out + ((unsigned long long)c * fb << fshift);
        for (uint32_t d = warp; d < fb; d += RL_WARPS) {
            const uint32_t s0 = s_bs[d], s1 = s_bs[d + 1], se = s_ge[d];
            unsigned long long* dst = wout + ((unsigned long long)d << fshift) + s_gb[d];
            for (uint32_t i = s0 + lane; i < se; i += 32) __stcs(dst + (i - s0), s_sort[i]);
            if (se < s1) over = true;
        }
        __syncthreads();  // s_sort and the tables are reused by the next tile
    }
    if (over) st->bad = 1;
}

#ifndef RA_THREADS_CFG
#define RA_THREADS_CFG 256
#endif
// rs5_refine with shared-atomic ranking (default).  Same job and output as
// k_rs_refine_lean: a coarse window's records -> {cur, rank} pairs split by
// fine window (rank = IS_1[sid] - local - 1, listrank.py:375-379).
//  * A record's slot among its warp's records of the same fine bin comes from
//    one shared atomicAdd on the warp's bin counter (order inside a bin is
//    free: rs5_scatter places every pair by its node id), instead of NB + 1
//    ballots and a leader update per record (1.25 G -> 0.8 G warp
//    instructions at 2^28, rs5_refine 2.36 -> 1.85 ms).
//  * The global atomic that claims a bin's run in its fine window is issued
//    before the placement barrier and only consumed after the placement, so
//    its latency overlaps the tile's shared-memory sort.
//  * Tiles of 2048 records, 4 CTAs of 256 threads per SM.  (A variant that
//    deferred each tile's write-out by one iteration behind a double-buffered
//    sorted tile measured slower: 2.74 ms.)
constexpr int RA_THREADS = RA_THREADS_CFG;
constexpr int RA_WARPS = RA_THREADS / 32;
constexpr int RA_IT = 8;
constexpr int RA_TILE = RA_THREADS * RA_IT;  // 2048 records (2^cshift is a multiple)
constexpr int RA_MAXB = 64;
constexpr int RA_CTAS_PER_SM = 1024 / RA_THREADS;

static size_t ra_smem_bytes() { return (size_t)RA_TILE * 8 * 2; }

__global__ void __launch_bounds__(RA_THREADS, RA_CTAS_PER_SM) k_rs_refine_atom(
    const unsigned long long* __restrict__ in, unsigned long long* __restrict__ cursor,
    unsigned long long* __restrict__ out, ListStatus* st, unsigned long long n, uint32_t cshift, uint32_t fshift,
    const uint32_t* __restrict__ IS1, uint32_t sb, uint32_t lb) {
    if (layout_local(st) || st->overflow) return;
    const uint32_t fb = 1u << (cshift - fshift);  // <= RA_MAXB
    extern __shared__ __align__(128) unsigned char ra_raw[];
    unsigned long long* s_in = reinterpret_cast<unsigned long long*>(ra_raw);
    unsigned long long* s_sort = s_in + RA_TILE;
    __shared__ unsigned long long bar;
    // per-(bin, warp) counts -> absolute tile slots, bin-major with a stride of
    // RA_WARPS + 1 words so a warp's counter updates spread over the banks
    constexpr uint32_t kStride = RA_WARPS + 1;
    __shared__ uint32_t s_c[RA_MAXB * kStride];
    __shared__ uint32_t s_tot[RA_WARPS];
    __shared__ uint32_t s_bs[RA_MAXB + 1];        // bin starts in the sorted tile
    // per bin: {window slot of the bin's first tile record minus its tile slot, tile end of the writable run}
    __shared__ uint2 s_de[RA_MAXB];
    const uint32_t t = threadIdx.x, lane = lane_id(), warp = t >> 5;
    const unsigned long long ntiles = (n + RA_TILE - 1) / RA_TILE;
    const uint32_t R1 = (uint32_t)min(st->R[1], (unsigned long long)0xFFFFFFFFu);
    const unsigned long long pol_last = l2_evict_last();
    const uint32_t fmask = fb - 1;
    const uint32_t lmask = (1u << lb) - 1u;  // lb < 32 (host-checked)
    const uint32_t smask = (uint32_t)((1ull << (sb - lb)) - 1);
    const uint32_t cap = 1u << fshift;
    if (t == 0) mbar_init(&bar, 1);
    __syncthreads();
    auto issue = [&](unsigned long long tile) {
        if (t == 0 && tile < ntiles) {
            const unsigned long long e0 = tile * RA_TILE;
            const uint32_t cnt = (uint32_t)min((unsigned long long)RA_TILE, n - e0);
            const uint32_t bytes = (cnt * 8u + 15u) & ~15u;  // the buffer is padded to whole windows
            mbar_expect_tx(&bar, bytes);
            bulk_g2s_hint(s_in, in + e0, bytes, &bar, l2_evict_first());
        }
    };
    bool over = false;
    uint32_t phase = 0;
    issue(blockIdx.x);
    for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const unsigned long long e0 = tile * RA_TILE;
        const uint32_t cnt = (uint32_t)min((unsigned long long)RA_TILE, n - e0);
        const uint32_t c = (uint32_t)(e0 >> cshift);  // tiles never straddle a coarse window
        s_c[lane * kStride + warp] = 0u;  // this warp's counters
        s_c[(lane + 32) * kStride + warp] = 0u;
        mbar_wait(&bar, phase);
        phase ^= 1u;
        // loc: local (bits 0-19) | rank among the warp's records of the bin (bits 20-27) | valid (bit 31);
        // the fine bin is recomputed from cur (fewer live registers)
        constexpr uint32_t kValid = 0x80000000u;
        uint32_t cur[RA_IT], gv[RA_IT], loc[RA_IT];
#pragma unroll
        for (int j = 0; j < RA_IT; ++j) {
            const uint32_t e = j * RA_THREADS + t;
            const unsigned long long r = e < cnt ? s_in[e] : 0ull;
            cur[j] = (uint32_t)(r >> sb);
            const uint32_t sid = (uint32_t)(r >> lb) & smask;
            loc[j] = (uint32_t)r & lmask;
            // issued now, first used at the placement: the gathers fly while the tile is ranked
            gv[j] = ld_hint(IS1 + (sid < R1 ? sid : 0u), pol_last);
            if (e < cnt && (cur[j] >> cshift) == c) loc[j] |= kValid;
        }
        __syncwarp();  // this warp's counters are zeroed
        // branch-free: an invalid record adds 0 to bin 0, so the eight atomics issue back to back
        uint32_t slot[RA_IT];
#pragma unroll
        for (int j = 0; j < RA_IT; ++j) {
            const bool v = (loc[j] & kValid) != 0;
            slot[j] = atomicAdd(&s_c[(v ? (cur[j] >> fshift) & fmask : 0u) * kStride + warp], v ? 1u : 0u);
        }
#pragma unroll
        for (int j = 0; j < RA_IT; ++j) loc[j] |= slot[j] << 20;  // local < 2^20 (host-checked)
        __syncthreads();  // (1) staging consumed, every warp's counts in
        issue(tile + gridDim.x);
        // (bin, warp) counts -> absolute slots of the bin-sorted tile: a block
        // scan in bin-major order, thread t owning bin t / TPB, warps 2 (t % TPB)
        // and 2 (t % TPB) + 1; one global atomic per non-empty bin claims the
        // bin's run in its fine window (issued here, consumed after the placement)
        constexpr uint32_t TPB = RA_WARPS / 2;  // threads per bin (2 counters each)
        static_assert(RA_MAXB * TPB == RA_THREADS, "two counters per thread");
        const uint32_t bq = t / TPB, i0 = bq * kStride + 2 * (t % TPB);
        const uint32_t a0 = s_c[i0], a1 = s_c[i0 + 1], pair = a0 + a1;
        uint32_t incl = pair;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += y;
        }
        if (lane == 31) s_tot[warp] = incl;
        // the bin's total: the TPB threads of a bin are adjacent lanes
        uint32_t btot = pair;
#pragma unroll
        for (uint32_t o = 1; o < TPB; o <<= 1) btot += __shfl_xor_sync(0xffffffffu, btot, o);
        uint32_t base = 0;
        const bool head = (t % TPB) == 0 && bq < fb;
        if (head && btot) base = (uint32_t)atomicAdd(cursor + (unsigned long long)c * fb + bq, (unsigned long long)btot);
        __syncthreads();  // (1b) warp totals
        uint32_t woff = lane < (uint32_t)warp ? s_tot[lane] : 0u;  // lanes < 8 hold the earlier warps' totals
#pragma unroll
        for (int o = 1; o < RA_WARPS; o <<= 1) woff += __shfl_xor_sync(0xffffffffu, woff, o);
        woff = __shfl_sync(0xffffffffu, woff, 0);  // (the reduction ran in groups of RA_WARPS lanes)
        const uint32_t excl = incl - pair + woff;
        s_c[i0] = excl;
        s_c[i0 + 1] = excl + a0;
        if (head) s_bs[bq] = excl;
        if (t == RA_THREADS - 1) s_bs[fb] = incl + woff;  // every record of the tile (bins >= fb are empty)
        __syncthreads();  // (2) tile slots known
#pragma unroll
        for (int j = 0; j < RA_IT; ++j) {
            if (loc[j] & kValid) {
                const uint32_t pos = s_c[((cur[j] >> fshift) & fmask) * kStride + warp] + ((loc[j] >> 20) & 0xFFu);
                const uint32_t rank = gv[j] - (loc[j] & 0xFFFFFu) - 1u;
                s_sort[pos] = ((unsigned long long)cur[j] << 32) | rank;
            }
        }
        if (head) {  // the claims, now back
            const uint32_t room = base < cap ? cap - base : 0u;
            s_de[bq] = make_uint2(base - excl, excl + (btot < room ? btot : room));
        }
        __syncthreads();  // (3) tile sorted, runs claimed
        // write out, flat: slot i -> its bin's run in the fine window (consecutive
        // slots of a bin are consecutive in the window, so a warp's stores coalesce)
        unsigned long long* wout = out + ((unsigned long long)c * fb << fshift);
        const uint32_t total = s_bs[fb];
#pragma unroll 4
        for (uint32_t i = t; i < total; i += RA_THREADS) {
            const unsigned long long x = s_sort[i];
            const uint32_t d = ((uint32_t)(x >> 32) >> fshift) & fmask;
            const uint2 de = s_de[d];
            if (i < de.y)
                __stcs(wout + ((unsigned long long)d << fshift) + (uint32_t)(i + de.x), x);
            else
                over = true;
        }
        // no closing barrier: the next tile zeroes a warp's counters from that
        // warp, and rewrites s_bs / s_de / s_sort after barrier (1)
    }
    if (over) st->bad = 1;
}

// rs5_refine + rs5_scatter in one pass (SG_RS_REFINE=7, experiment): every
// record's rank (IS_1[sid] - local - 1, listrank.py:375-379) is stored
// straight to rank[cur].  The records arrive binned by coarse window and the
// blocks run roughly in index order, so the stores of the ~1-2 coarse windows
// in flight (4-8 MiB of output) land in L2 and their sectors are complete
// before eviction: no pairs buffer, no sort, no second pass -- at the price of
// one L2 sector write per node next to the IS_1 gather.
constexpr int RD_THREADS = 256;
constexpr int RD_IT = 8;  // records per thread (four 16-B loads)
template <class OutT>
__global__ void __launch_bounds__(RD_THREADS) k_rs_refine_direct(const unsigned long long* __restrict__ in,
                                                                 OutT* __restrict__ rank, const ListStatus* st,
                                                                 unsigned long long n, uint32_t cshift,
                                                                 const uint32_t* __restrict__ IS1, uint32_t sb,
                                                                 uint32_t lb) {
    if (layout_local(st) || ranks_invalid(st)) return;
    const uint32_t R1 = (uint32_t)min(st->R[1], (unsigned long long)0xFFFFFFFFu);
    const unsigned long long pol_last = l2_evict_last();
    const uint32_t lmask = (1u << lb) - 1u;
    const uint32_t smask = (uint32_t)((1ull << (sb - lb)) - 1);
    const unsigned long long e0 = (unsigned long long)blockIdx.x * (RD_THREADS * RD_IT);
    unsigned long long r[RD_IT];
    uint32_t g[RD_IT];
#pragma unroll
    for (int j = 0; j < RD_IT / 2; ++j) {
        const unsigned long long e = e0 + (unsigned long long)(j * RD_THREADS + threadIdx.x) * 2;
        if (e + 1 < n) {
            const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(in + e));
            r[2 * j] = v.x;
            r[2 * j + 1] = v.y;
        } else {
            r[2 * j] = e < n ? __ldcs(in + e) : ~0ull;
            r[2 * j + 1] = ~0ull;
        }
    }
#pragma unroll
    for (int j = 0; j < RD_IT; ++j) {
        const uint32_t sid = (uint32_t)(r[j] >> lb) & smask;
        g[j] = ld_hint(IS1 + (sid < R1 ? sid : 0u), pol_last);
    }
#pragma unroll
    for (int j = 0; j < RD_IT; ++j) {
        const unsigned long long e = e0 + (unsigned long long)((j >> 1) * RD_THREADS + threadIdx.x) * 2 + (j & 1);
        const unsigned long long cur = r[j] >> sb;
        // padding / dropped slots hold ids outside the record's own coarse window
        if (e < n && (cur >> cshift) == (e >> cshift)) rank[cur] = (OutT)(g[j] - ((uint32_t)r[j] & lmask) - 1u);
    }
}

// rs5_scatter over the tile layout of k_rs_refine_lean<.., true>: one CTA
// per fine window f (bin d of coarse window c) collects bin d's run from
// each of the coarse window's tiles -- lane l of a warp reads the run bounds
// of one tile, the warp then copies the runs four at a time -- scatters the
// pairs into shared memory and stores the window coalesced.
template <class OutT>
__global__ void __launch_bounds__(256) k_rs_rec_scatter_tiles(const unsigned long long* __restrict__ pairs,
                                                              const uint32_t* __restrict__ toff,
                                                              OutT* __restrict__ rank, unsigned long long n,
                                                              uint32_t cshift, uint32_t fshift, const ListStatus* st,
                                                              int vec) {
    if (layout_local(st) || ranks_invalid(st)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    OutT* win = reinterpret_cast<OutT*>(smem_raw);
    const unsigned long long w0 = (unsigned long long)blockIdx.x << fshift;
    if (w0 >= n) return;
    const uint32_t size = (uint32_t)min((unsigned long long)1 << fshift, n - w0);
    const uint32_t mask = (1u << fshift) - 1u;
    const uint32_t fb = 1u << (cshift - fshift);
    const uint32_t d = blockIdx.x & (fb - 1);
    const unsigned long long c = (unsigned long long)blockIdx.x >> (cshift - fshift);
    const unsigned long long t0 = (c << cshift) / RL_TILE;
    const unsigned long long t1 = min(((c + 1) << cshift), n + RL_TILE - 1) / RL_TILE;  // tiles of window c holding records
    const uint32_t ntile = (uint32_t)(t1 > t0 ? t1 - t0 : 0);
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    auto put = [&](unsigned long long pr) {
        const uint32_t cur = (uint32_t)(pr >> 32);
        if ((cur >> fshift) == (uint32_t)blockIdx.x) win[cur & mask] = (OutT)(uint32_t)pr;
    };
    for (uint32_t tb = warp * 32; tb < ntile; tb += 8 * 32) {
        const uint32_t tl = tb + lane;
        uint32_t lo = 0, hi = 0;
        if (tl < ntile) {
            const uint32_t* to = toff + (t0 + tl) * (fb + 1) + d;
            lo = __ldg(to);
            hi = __ldg(to + 1);
        }
        const uint32_t nr = min(32u, ntile - tb);
        for (uint32_t r = 0; r < nr; r += 4) {
            uint32_t a[4], e[4];
            const unsigned long long* src[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t rr = min(r + q, 31u);
                a[q] = __shfl_sync(0xffffffffu, lo, rr);
                e[q] = (r + q < nr) ? __shfl_sync(0xffffffffu, hi, rr) : a[q];
                src[q] = pairs + (t0 + tb + rr) * RL_TILE;
            }
            for (uint32_t k = lane;; k += 32) {
                bool any = false;
                unsigned long long v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool ok = a[q] + k < e[q];
                    v[q] = ok ? __ldcs(src[q] + a[q] + k) : ~0ull;
                    any |= a[q] + k - lane < e[q];
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (v[q] != ~0ull) put(v[q]);
                if (!__any_sync(0xffffffffu, any)) break;
            }
        }
    }
    __syncthreads();
    if (vec && size == (1u << fshift)) {
        constexpr uint32_t V = 16 / sizeof(OutT);
        const uint4* s4 = reinterpret_cast<const uint4*>(win);
        uint4* dst = reinterpret_cast<uint4*>(rank + w0);
        for (uint32_t i = threadIdx.x; i < size / V; i += blockDim.x) __stcs(dst + i, s4[i]);
        return;
    }
    for (uint32_t i = threadIdx.x; i < size; i += blockDim.x) rank[w0 + i] = win[i];
}

// one CTA per fine window: scatter its pairs into shared memory, then store
// the window coalesced
template <class OutT>
__global__ void __launch_bounds__(256) k_rs_rec_scatter(const unsigned long long* __restrict__ pairs,
                                                               OutT* __restrict__ rank, unsigned long long n,
                                                               uint32_t fshift, const ListStatus* st, int vec) {
    if (layout_local(st) || ranks_invalid(st)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    OutT* win = reinterpret_cast<OutT*>(smem_raw);
    const unsigned long long w0 = (unsigned long long)blockIdx.x << fshift;
    if (w0 >= n) return;
    const uint32_t size = (uint32_t)min((unsigned long long)1 << fshift, n - w0);
    const uint32_t mask = (1u << fshift) - 1u;
    const unsigned long long wid = w0 >> fshift;
    auto put = [&](unsigned long long pr) {
        const unsigned long long cur = pr >> 32;
        if ((cur >> fshift) == wid) win[cur & mask] = (OutT)(uint32_t)pr;
    };
    if (vec && size == (1u << fshift)) {  // full window, aligned output: 16-B loads and stores
        const ulonglong2* p2 = reinterpret_cast<const ulonglong2*>(pairs + w0);
        for (uint32_t i = threadIdx.x; i < size / 2; i += blockDim.x) {
            const ulonglong2 v = __ldcs(p2 + i);
            put(v.x);
            put(v.y);
        }
        __syncthreads();
        constexpr uint32_t V = 16 / sizeof(OutT);
        const uint4* src = reinterpret_cast<const uint4*>(win);
        uint4* dst = reinterpret_cast<uint4*>(rank + w0);
        for (uint32_t i = threadIdx.x; i < size / V; i += blockDim.x) __stcs(dst + i, src[i]);
        return;
    }
    for (uint32_t i = threadIdx.x; i < size; i += blockDim.x) put(__ldcs(pairs + w0 + i));
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < size; i += blockDim.x) rank[w0 + i] = win[i];
}

// ---------------------------------------------------------------------------
// top level: one CTA of weighted pointer jumping (RS4 single block,
// listrank.py:333-342) producing inclusive suffix sums IS[i].

template <class View>
__global__ void __launch_bounds__(1024) k_rs_final(View src, uint2* A, uint2* B, uint32_t* __restrict__ IS,
                                                   ListStatus* st, int level) {
    const uint32_t R = (uint32_t)st->R[level];
    for (uint32_t i = threadIdx.x; i < R; i += blockDim.x) {
        unsigned long long nx;
        uint32_t w;
        src.load(i, nx, w);
        uint32_t nxt = NIL;
        if (nx >= R) {
            st->bad = 1;
        } else if (nx != i) {
            nxt = (uint32_t)nx;
        }
        A[i] = make_uint2(w, nxt);
    }
    __syncthreads();
    int maxr = 2;
    for (uint32_t r = R; r > 1; r = (r + 1) >> 1) ++maxr;
    uint2* cur = A;
    uint2* nxt = B;
    for (int r = 0; r < maxr; ++r) {
        int active = 0;
        for (uint32_t i = threadIdx.x; i < R; i += blockDim.x) {
            uint2 a = __ldcg(cur + i);
            if (a.y != NIL) {
                const uint2 b = __ldcg(cur + a.y);
                a.x += b.x;
                a.y = b.y;
                active |= (b.y != NIL);
            }
            __stcg(nxt + i, a);
        }
        active = __syncthreads_or(active);
        uint2* t = cur;
        cur = nxt;
        nxt = t;
        if (!active) break;
    }
    for (uint32_t i = threadIdx.x; i < R; i += blockDim.x) IS[i] = __ldcg(cur + i).x;
    if (threadIdx.x == 0 && R > 0) {
        const uint2 h = __ldcg(cur);
        st->head_sum = h.x;
        st->head_ok = (h.y == NIL) ? 1ull : 0ull;
    }
}

// Multi-CTA weighted pointer jumping on a ruler list too big for one CTA
// (used right above level 0: a level's walk is bound by its longest sublist,
// ~2^kbits * ln(R) dependent hops, so three more walked levels cost more than
// ~log2(R) in-place jump rounds over an L2-resident list).  Entries are
// {inclusive weight up to `next`, next}; next = NIL once the sum reaches the
// tail.  Rounds update in place: every version of an entry a reader can see is
// a consistent (weight, next) pair of one 64-bit access, and each round at
// least doubles every live pointer's reach, so ceil(log2 R) + 1 rounds suffice.
template <class View>
__global__ void __launch_bounds__(256) k_rs_top_init(View src, uint2* __restrict__ A, ListStatus* st, int level) {
    const unsigned long long R = st->R[level];
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += stride) {
        unsigned long long nx;
        uint32_t w;
        src.load((uint32_t)i, nx, w);
        uint32_t nxt = NIL;
        if (nx >= R) {
            st->bad = 1;
        } else if (nx != i) {
            nxt = (uint32_t)nx;
        }
        A[i] = make_uint2(w, nxt);
    }
}

__global__ void __launch_bounds__(256) k_rs_top_jump(uint2* A, ListStatus* st, int level,
                                                     uint32_t* __restrict__ IS) {
    constexpr int U = 4;
    const unsigned long long R = st->R[level];
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < R;
         i0 += stride * U) {
        uint2 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned long long i = i0 + (unsigned long long)u * stride;
            a[u] = i < R ? __ldcg(A + i) : make_uint2(0u, NIL);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) b[u] = a[u].y != NIL ? __ldcg(A + a[u].y) : make_uint2(0u, NIL);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned long long i = i0 + (unsigned long long)u * stride;
            if (i >= R) continue;
            if (a[u].y != NIL) {
                a[u].x += b[u].x;
                a[u].y = b[u].y;
                __stcg(A + i, a[u]);
            }
            if (IS != nullptr) {  // last round: the inclusive suffix sums
                IS[i] = a[u].x;
                if (i == 0) {
                    st->head_sum = a[u].x;
                    st->head_ok = (a[u].y == NIL) ? 1ull : 0ull;
                }
            }
        }
    }
}

// The same as one cooperative launch: init, the jump rounds separated by
// grid barriers (a round costs ~3 us instead of a ~5 us launch), stopping
// once a round finds no live pointer, and the extraction.
template <class View>
__global__ void __launch_bounds__(512) k_rs_top_coop(View src, uint2* A, ListStatus* st, int level,
                                                     uint32_t* __restrict__ IS, int rounds) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const unsigned long long R = st->R[level];
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long t0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (unsigned long long i = t0; i < R; i += stride) {
        unsigned long long nx;
        uint32_t w;
        src.load((uint32_t)i, nx, w);
        uint32_t nxt = NIL;
        if (nx >= R) {
            st->bad = 1;
        } else if (nx != i) {
            nxt = (uint32_t)nx;
        }
        A[i] = make_uint2(w, nxt);
    }
    grid.sync();
    for (int r = 0; r < rounds; ++r) {
        if (t0 == 0) st->top_live[(r + 1) % 3] = 0;  // next round's flag (last read two barriers ago)
        int live = 0;
        for (unsigned long long i = t0; i < R; i += stride) {
            uint2 a = __ldcg(A + i);
            if (a.y != NIL) {
                const uint2 b = __ldcg(A + a.y);
                a.x += b.x;
                a.y = b.y;
                __stcg(A + i, a);
                live |= (b.y != NIL);
            }
        }
        live = __syncthreads_or(live);
        if (live && threadIdx.x == 0) atomicOr(&st->top_live[r % 3], 1ull);
        grid.sync();
        if (*(volatile unsigned long long*)&st->top_live[r % 3] == 0) break;  // every pointer reached the tail
    }
    for (unsigned long long i = t0; i < R; i += stride) {
        const uint2 a = __ldcg(A + i);
        IS[i] = a.x;
        if (i == 0) {
            st->head_sum = a.x;
            st->head_ok = (a.y == NIL) ? 1ull : 0ull;
        }
    }
}

// ---------------------------------------------------------------------------
// expand (RS5 at level 0, listrank.py:360-382)

__global__ void __launch_bounds__(256) k_rs_expand_k(const unsigned long long* __restrict__ word,
                                                     const uint32_t* __restrict__ IS_up, uint32_t* __restrict__ IS,
                                                     const ListStatus* st, int level) {
    const unsigned long long N = st->R[level];
    const unsigned long long Rup = st->R[level + 1];
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
        const unsigned long long w = word[i];
        const unsigned long long o = w >> 32;
        IS[i] = o < Rup ? __ldg(IS_up + o) - (uint32_t)w : 0u;
    }
}

template <class OutT>
__global__ void k_rs_expand_direct(const uint32_t* __restrict__ IS0, OutT* __restrict__ rank, unsigned long long n,
                                   const ListStatus* st) {
    if (ranks_invalid(st)) return;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        rank[i] = (OutT)(IS0[i] - 1u);
}

// ---------------------------------------------------------------------------
// Tile contraction (local layouts: ordered or locally shuffled lists).
//
// A tile is TILE consecutive node ids.  Inside a tile the successor links
// that stay in the tile form disjoint chains ("segments"); a segment starts
// at a node with no in-tile predecessor (its head) and ends at a node whose
// successor leaves the tile (or the tail).  One CTA per tile loads the tile's
// successors into shared memory (coalesced) and ranks every node inside its
// segment with a small ruling set of its own: segment heads plus every
// CT_STRIDE-th node walk to the next local ruler, then weighted pointer
// jumping over the local rulers gives each node its distance to the segment
// end.  The contracted list -- one node per segment, weight = segment length,
// numbered by head index so node 0's segment is 0 -- is ranked by the
// upper levels; the expand pass recomputes the same tile structure and writes
// rank = (IS1[segment] - length) + distance to the end, coalesced.  Per node
// this costs two streaming 4-B reads and one 4-B write; no walk touches HBM
// at random.  Validation: no in-tile node with two in-tile predecessors, no
// in-tile cycle, heads == ends per tile, every segment's successor is some
// segment's head; the top level then checks that the head's segment reaches
// the tail with weight n (listrank.py:297-298, core.py:148-167).
constexpr uint32_t CT_STRIDE = 16;
constexpr uint16_t CT_END = 0xFFFF;
constexpr int CT_CTAS_PER_SM = 3;

struct ContractSmem {
    uint32_t own[TILE];      // node -> (local ruler << 16) | offset from the ruler          [sw32]
    uint32_t link[TILE];     // ruler -> (next ruler << 16) | distance; next = CT_END: distance to the segment end
    uint16_t nx[TILE];       // node -> in-tile successor, CT_END if it leaves the tile / is the tail [sw16]
    uint16_t rid[TILE];      // node -> local ruler index (walk); end node -> tile-local segment     [sw16]
    uint16_t term[TILE];     // ruler -> end node of its segment
    uint8_t pred[TILE];      // node has an in-tile predecessor
    uint16_t brk[TILE / 16]; // per 16-id block: bit q = id q's successor is not id q + 1
    uint16_t rd[TILE];       // ruler -> distance to its segment end (after jumping)
};

// Bank swizzles for node-indexed arrays.  Walkers start 16 nodes apart (one
// local ruler per 16 ids), so an unswizzled u32 array puts a warp's 32 walk
// steps into 2 banks.  sw32 spreads them over all 32 banks; sw16 (2 ids per
// bank word) leaves at most 2-way conflicts.  Both keep aligned groups of 4
// ids together (sw16 also in order; sw32 permutes a group by XOR with
// sw32(group base) & 3), so 16-B / 8-B vector accesses stay legal.
__device__ __forceinline__ uint32_t sw32(uint32_t l) { return l ^ (((l >> 5) & 3u) << 2) ^ ((l >> 7) & 3u); }
__device__ __forceinline__ uint32_t sw16(uint32_t l) { return l ^ (((l >> 6) & 7u) << 2); }

template <class SuccT, bool kVec>
__global__ void __launch_bounds__(TILE_THREADS, CT_CTAS_PER_SM) k_rs_contract(
    const SuccT* __restrict__ succ, ListStatus* st, const uint32_t* __restrict__ tile_off,
    uint32_t* __restrict__ headsid, uint32_t* __restrict__ seg_head, uint32_t* __restrict__ seg_succ,
    uint2* __restrict__ lvl1, uint32_t* __restrict__ node_word, uint32_t* __restrict__ tile_run) {
    if (!layout_local(st)) return;
    constexpr int VEC = 4;  // ids per thread and vector access
    constexpr int NV = TILE_ITEMS / VEC;
    extern __shared__ __align__(16) unsigned char ct_raw[];
    ContractSmem& S = *reinterpret_cast<ContractSmem*>(ct_raw);
    typedef cub::BlockScan<unsigned long long, TILE_THREADS> BS;
    __shared__ typename BS::TempStorage scan_tmp;
    const unsigned long long N = st->R[0];
    const unsigned long long R1 = st->R[1];
    const unsigned long long ntiles = (N + TILE - 1) / TILE;
    const uint32_t t = threadIdx.x;
    const uint32_t lane = lane_id();
    static_assert(TILE == TILE_THREADS * 16, "one uint4 of predecessor flags per thread");
    bool bad = false;
    // the CTA's tiles in batches of TILE_THREADS: thread k settles batch tile k
    // if the census flagged it as a run (succ = id + 1 throughout, the last
    // node continuing into the next tile: one segment, written without
    // reading the tile again); the CTA then contracts the others together
    __shared__ uint32_t s_run[TILE_THREADS];
    const unsigned long long bstep = (unsigned long long)TILE_THREADS * gridDim.x;
    for (unsigned long long tb = blockIdx.x; tb < ntiles; tb += bstep) {
        {
            const unsigned long long mt = tb + (unsigned long long)t * gridDim.x;
            const uint32_t r = mt < ntiles ? __ldg(tile_run + mt) : 1u;
            if (mt < ntiles && r) {
                const unsigned long long sid = tile_off[mt];
                const uint32_t segs = mt + 1 < ntiles ? tile_off[mt + 1] - tile_off[mt] : (uint32_t)(R1 - tile_off[mt]);
                if (segs != 1u) {
                    bad = true;
                } else {
                    const unsigned long long mb = mt * TILE;
                    seg_head[sid] = (uint32_t)mb;
                    headsid[mb] = (uint32_t)sid;
                    lvl1[sid] = make_uint2(0u, (uint32_t)TILE);
                    seg_succ[sid] = (uint32_t)(mb + TILE);
                }
            }
            s_run[t] = r;
            __syncthreads();
        }
        for (uint32_t k = 0; k < (uint32_t)TILE_THREADS; ++k) {
            if (s_run[k]) continue;  // a run (settled above) or past the end
            const unsigned long long tile = tb + (unsigned long long)k * gridDim.x;
            const unsigned long long base = tile * TILE;
            const uint32_t tn = (uint32_t)min((unsigned long long)TILE, N - base);
            const bool full = kVec && tn == TILE;
            // 1. successors -> in-tile links, predecessor flags (plain byte
            //    stores: a node with two in-tile predecessors shows up as fewer
            //    flags than links), run-break masks.  Thread t holds ids
            //    4(j*256+t) .. +3.
            SuccT v[TILE_ITEMS];
            if (full) {
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    const SuccT* p = succ + base + (size_t)(j * TILE_THREADS + t) * VEC;
                    if (sizeof(SuccT) == 4) {
                        const uint4 w = __ldcs(reinterpret_cast<const uint4*>(p));
                        v[j * 4 + 0] = (SuccT)w.x, v[j * 4 + 1] = (SuccT)w.y, v[j * 4 + 2] = (SuccT)w.z, v[j * 4 + 3] = (SuccT)w.w;
                    } else {
                        const ulonglong2 w0 = __ldcs(reinterpret_cast<const ulonglong2*>(p));
                        const ulonglong2 w1 = __ldcs(reinterpret_cast<const ulonglong2*>(p) + 1);
                        v[j * 4 + 0] = (SuccT)w0.x, v[j * 4 + 1] = (SuccT)w0.y, v[j * 4 + 2] = (SuccT)w1.x, v[j * 4 + 3] = (SuccT)w1.y;
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < NV; ++j)
#pragma unroll
                    for (int c = 0; c < VEC; ++c) {
                        const uint32_t l = (j * TILE_THREADS + t) * VEC + c;
                        v[j * 4 + c] = l < tn ? succ[base + l] : SuccT(0);
                    }
            }
            // Single-run tile (every id's successor is the next id, the last one
            // leaves the tile or is the tail), decided from the registers: one
            // segment, distance to its end = tn - 1 - l, written in closed form
            // without the shared-memory ranking.
            {
                bool run = true;
                const uint32_t last = tn - 1;
#pragma unroll
                for (int j = 0; j < NV; ++j)
#pragma unroll
                    for (int c = 0; c < VEC; ++c) {
                        const uint32_t l = (j * TILE_THREADS + t) * VEC + c;
                        const unsigned long long x = as_index<SuccT>(v[j * 4 + c]);
                        if (l < last)
                            run &= x == base + l + 1;
                        else if (l == last)
                            run &= (x - base >= tn) || x == base + l;
                    }
                if (__syncthreads_and(run)) {
                    const uint32_t segs = tile + 1 < ntiles ? tile_off[tile + 1] - tile_off[tile]
                                                            : (uint32_t)(R1 - tile_off[tile]);
                    if (segs != 1u) bad = true;
                    if (t == 0 && segs == 1u) {
                        const unsigned long long sid = tile_off[tile];
                        seg_head[sid] = (uint32_t)base;
                        headsid[base] = (uint32_t)sid;
                        lvl1[sid] = make_uint2(0u, tn);
                        const unsigned long long x = as_index<SuccT>(succ[base + last]);
                        seg_succ[sid] = (x >= N || x == base + last) ? NIL : (uint32_t)x;
                    }
                    // the node words of a run are tn - 1 - l (segment 0): the
                    // expand recomputes them from this flag instead of a 4-B
                    // write and read per node
                    if (t == 0) tile_run[tile] = 1u;
                    continue;  // no shared memory was touched
                }
            }
            if (t == 0) tile_run[tile] = 0u;
            reinterpret_cast<uint4*>(S.pred)[t] = make_uint4(0u, 0u, 0u, 0u);  // 4096 flags
            __syncthreads();
            uint32_t links = 0;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const uint32_t l0 = (j * TILE_THREADS + t) * VEC;
                uint16_t nx[VEC];
                uint32_t nib = 0;  // run breaks: nx[l] != l + 1
#pragma unroll
                for (int c = 0; c < VEC; ++c) {
                    const uint32_t l = l0 + c;
                    nx[c] = CT_END;
                    if (l < tn) {
                        const unsigned long long dx = as_index<SuccT>(v[j * 4 + c]) - base;
                        if (dx < tn && dx != l) {
                            nx[c] = (uint16_t)dx;
                            S.pred[dx] = 1;
                            ++links;
                        }
                    }
                    if (nx[c] != l + 1) nib |= 1u << c;
                }
                *reinterpret_cast<ushort4*>(&S.nx[sw16(l0)]) = make_ushort4(nx[0], nx[1], nx[2], nx[3]);
                *reinterpret_cast<uint4*>(&S.own[sw32(l0) & ~3u]) = make_uint4(~0u, ~0u, ~0u, ~0u);
                // the 4 nibbles of a 16-id block sit in 4 consecutive lanes
                uint32_t m16 = nib << (4 * (lane & 3));
                m16 |= __shfl_xor_sync(0xffffffffu, m16, 1);
                m16 |= __shfl_xor_sync(0xffffffffu, m16, 2);
                if ((lane & 3) == 0) S.brk[l0 >> 4] = (uint16_t)m16;
            }
            __syncthreads();
            if (tile == 0 && S.pred[0]) bad = true;  // node 0 must start the list
            // 2. local rulers (blocked: thread t owns nodes 16t .. 16t+15): heads
            //    and every CT_STRIDE-th node; numbered in index order
            uint32_t rflags = 0, hflags = 0;
            const uint4 pf = reinterpret_cast<const uint4*>(S.pred)[t];
            const uint32_t pw[4] = {pf.x, pf.y, pf.z, pf.w};
#pragma unroll
            for (int q = 0; q < TILE_ITEMS; ++q) {
                const uint32_t l = t * TILE_ITEMS + q;
                if (l < tn) {
                    const bool head = ((pw[q >> 2] >> (8 * (q & 3))) & 0xFFu) == 0u;
                    if (head) hflags |= 1u << q;
                    if (head || (l % CT_STRIDE) == 0) rflags |= 1u << q;
                }
            }
            // one scan: rulers (bits 32..), heads (16..31), in-tile links (0..15)
            unsigned long long packed = ((unsigned long long)__popc(rflags) << 32) |
                                        ((unsigned long long)__popc(hflags) << 16) | links, pre, tot;
            BS(scan_tmp).ExclusiveSum(packed, pre, tot);
            const uint32_t rpre = (uint32_t)(pre >> 32), hpre = (uint32_t)(pre >> 16) & 0xFFFFu;
            const uint32_t K = (uint32_t)(tot >> 32), H = (uint32_t)(tot >> 16) & 0xFFFFu;
            if (H + (uint32_t)(tot & 0xFFFFu) != tn) bad = true;  // two in-tile predecessors
#pragma unroll
            for (int g = 0; g < TILE_ITEMS / 4; ++g) {
                uint16_t r[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int q = g * 4 + c;
                    r[c] = (rflags & (1u << q)) ? (uint16_t)(rpre + __popc(rflags & ((1u << q) - 1u))) : CT_END;
                }
                *reinterpret_cast<ushort4*>(&S.rid[sw16(t * TILE_ITEMS + g * 4)]) = make_ushort4(r[0], r[1], r[2], r[3]);
            }
            __syncthreads();
            // 3. each thread walks from its own local rulers to the next local
            //    ruler / the segment end.  A run of +1 successors inside a 16-id
            //    block is crossed in one step (no ruler can sit inside it: its
            //    nodes have in-tile predecessors and are not 16-aligned); the
            //    block start after a full run is a ruler.
            for (uint32_t rem = rflags; rem != 0; rem &= rem - 1) {
                const uint32_t q = __ffs(rem) - 1;
                const uint32_t k = rpre + __popc(rflags & ((1u << q) - 1u));
                uint32_t l = t * TILE_ITEMS + q, off = 0;
                for (;;) {
                    const uint32_t m = (uint32_t)S.brk[l >> 4] >> (l & 15u);
                    const uint32_t r = m ? (uint32_t)(__ffs(m) - 1) : 16u - (l & 15u);
                    if (r) {
                        if (r == 16) {  // a whole block: four 16-B stores (sw32 permutes each group by XOR)
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                const uint32_t gp = sw32(l + 4 * g), xr = gp & 3u;
                                const uint32_t b0 = (k << 16) | (off + 4 * g);
                                *reinterpret_cast<uint4*>(&S.own[gp & ~3u]) =
                                    make_uint4(b0 + (0u ^ xr), b0 + (1u ^ xr), b0 + (2u ^ xr), b0 + (3u ^ xr));
                            }
                        } else {
                            for (uint32_t j = 0; j < r; ++j) S.own[sw32(l + j)] = (k << 16) | (off + j);
                        }
                        l += r;
                        off += r;
                        if (m == 0) {  // l: the next block's first id, a ruler
                            S.link[k] = ((uint32_t)S.rid[sw16(l)] << 16) | off;
                            S.term[k] = CT_END;
                            break;
                        }
                    }
                    S.own[sw32(l)] = (k << 16) | off;
                    const uint16_t nx = S.nx[sw16(l)];
                    if (nx == CT_END) {
                        S.link[k] = ((uint32_t)CT_END << 16) | off;
                        S.term[k] = (uint16_t)l;
                        break;
                    }
                    const uint16_t r2 = S.rid[sw16(nx)];
                    if (r2 != CT_END || off + 1 >= TILE) {  // the cap only trips on invalid lists
                        if (r2 == CT_END) bad = true;
                        S.link[k] = ((uint32_t)(r2 == CT_END ? k : r2) << 16) | ((off + 1) & 0xFFFFu);
                        S.term[k] = CT_END;
                        break;
                    }
                    l = nx;
                    ++off;
                }
            }
            __syncthreads();
            // 4. weighted pointer jumping over the local rulers, in place (one
            //    32-bit {next, distance} word per ruler keeps every read
            //    consistent), until each ruler points at the last ruler of its
            //    segment -- whose word holds the distance to the end
            for (int round = 0; round < 16; ++round) {
                int active = 0;
                for (uint32_t k = t; k < K; k += TILE_THREADS) {
                    const uint32_t a = S.link[k];
                    const uint32_t p = a >> 16;
                    if (p != CT_END) {
                        const uint32_t b = S.link[p];
                        if ((b >> 16) != CT_END) {
                            S.link[k] = (b & 0xFFFF0000u) | ((a + b) & 0xFFFFu);
                            active = 1;
                        }
                    }
                }
                if (!__syncthreads_or(active)) break;
            }
            // distance from ruler k to its segment end, and the end node
            auto seg_end = [&](uint32_t k, uint32_t& d, uint16_t& e) {
                const uint32_t a = S.link[k];
                const uint32_t p = a >> 16;
                if (p == CT_END) {
                    d = a & 0xFFFFu;
                    e = S.term[k];
                } else {
                    const uint32_t b = S.link[p];
                    d = (a + b) & 0xFFFFu;
                    e = (b >> 16) == CT_END ? S.term[p] : CT_END;
                }
            };
            for (uint32_t k = t; k < K; k += TILE_THREADS) {
                uint32_t d;
                uint16_t e;
                seg_end(k, d, e);
                if (e == CT_END) bad = true;  // a cycle through local rulers
            }
            // 5. segments: numbered by head index; end node -> tile-local segment
            const uint32_t segs = tile + 1 < ntiles ? tile_off[tile + 1] - tile_off[tile]
                                                    : (uint32_t)(R1 - tile_off[tile]);
            if (segs != H) bad = true;
            __syncthreads();  // rid[] is rewritten below
            for (uint32_t rem = hflags; rem != 0; rem &= rem - 1) {
                const uint32_t q = __ffs(rem) - 1;
                const uint32_t k = rpre + __popc(rflags & ((1u << q) - 1u));
                const uint32_t h = hpre + __popc(hflags & ((1u << q) - 1u));
                uint32_t d;
                uint16_t e;
                seg_end(k, d, e);
                if (e != CT_END) S.rid[sw16(e)] = (uint16_t)h;
                if (h < segs && e != CT_END) {
                    const unsigned long long sid = (unsigned long long)tile_off[tile] + h;
                    const uint32_t l = t * TILE_ITEMS + q;
                    seg_head[sid] = (uint32_t)(base + l);
                    headsid[base + l] = (uint32_t)sid;
                    lvl1[sid] = make_uint2(0u, d + 1u);
                    const unsigned long long x = as_index<SuccT>(succ[base + e]);
                    seg_succ[sid] = (x >= N || x == base + e) ? NIL : (uint32_t)x;
                }
            }
            __syncthreads();
            // per ruler: its segment (tile-local) and distance to the segment end;
            // nx[] is dead after the walk and holds the segment from here on
            for (uint32_t k = t; k < K; k += TILE_THREADS) {
                uint32_t d;
                uint16_t e;
                seg_end(k, d, e);
                S.nx[k] = e != CT_END ? S.rid[sw16(e)] : CT_END;
                S.rd[k] = (uint16_t)d;
            }
            __syncthreads();
            // 6. per node: {tile-local segment : 16 | distance to the segment end : 16}
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const uint32_t l0 = (j * TILE_THREADS + t) * VEC;
                const uint32_t g = sw32(l0);
                const uint4 ow4 = *reinterpret_cast<const uint4*>(&S.own[g & ~3u]);
                const uint32_t ow[4] = {ow4.x, ow4.y, ow4.z, ow4.w};
                uint32_t wd[VEC];
#pragma unroll
                for (int c = 0; c < VEC; ++c) {
                    const uint32_t o = ow[c ^ (g & 3u)];
                    wd[c] = 0xFFFFFFFFu;
                    if (l0 + c < tn) {
                        if (o == 0xFFFFFFFFu) {
                            bad = true;  // a cycle without local rulers
                        } else {
                            const uint32_t k = o >> 16;
                            wd[c] = ((uint32_t)S.nx[k] << 16) | (((uint32_t)S.rd[k] - (o & 0xFFFFu)) & 0xFFFFu);
                        }
                    }
                }
                if (full) {
                    *reinterpret_cast<uint4*>(node_word + base + l0) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
                } else {
#pragma unroll
                    for (int c = 0; c < VEC; ++c)
                        if (l0 + c < tn) node_word[base + l0 + c] = wd[c];
                }
            }
            __syncthreads();  // shared memory is reused by the next tile
        }
        __syncthreads();  // s_run is rewritten by the next batch
    }
    if (bad) st->bad = 1;
}

// expand the contraction: rank = (IS1[segment] - length) + distance to the
// segment end.  One warp per tile: the tile's flag and first segment are
// loaded once, then the lanes stream the tile -- a run tile (k_rs_count0 /
// k_rs_contract flag) is one segment whose words are tn - 1 - l, so its ranks
// are written without reading anything per node; other tiles read their node
// words and gather their segments' bases (L1-resident).
template <class OutT, bool kVec>
__global__ void __launch_bounds__(256) k_rs_contract_expand(const uint32_t* __restrict__ node_word,
                                                            const uint32_t* __restrict__ tile_off,
                                                            const uint2* __restrict__ lvl1,
                                                            const uint32_t* __restrict__ IS1, OutT* __restrict__ rank,
                                                            const ListStatus* st, const uint32_t* __restrict__ tile_run) {
    if (!layout_local(st) || ranks_invalid(st)) return;
    const unsigned long long N = st->R[0];
    const unsigned long long R1 = st->R[1];
    const unsigned long long ntiles = (N + TILE - 1) / TILE;
    const uint32_t lane = lane_id();
    const unsigned long long gw = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    auto put4 = [&](unsigned long long i, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
        if (sizeof(OutT) == 4) {
            __stcs(reinterpret_cast<uint4*>(rank + i), make_uint4(r0, r1, r2, r3));
        } else {
            ulonglong2* q = reinterpret_cast<ulonglong2*>(rank + i);
            __stcs(q, make_ulonglong2(r0, r1));
            __stcs(q + 1, make_ulonglong2(r2, r3));
        }
    };
    for (unsigned long long tile = gw; tile < ntiles; tile += nw) {
        const unsigned long long base = tile * TILE;
        const uint32_t tn = (uint32_t)min((unsigned long long)TILE, N - base);
        const unsigned long long off = __ldg(tile_off + tile);
        if (__ldg(tile_run + tile)) {
            // rank of id base + l = r - l (0 throughout for an out-of-range segment, as rank_of)
            const uint32_t r = off < R1 ? __ldg(IS1 + off) - __ldg(&lvl1[off].y) + (tn - 1) : 0u;
            const uint32_t dl = off < R1 ? 1u : 0u;
            const uint32_t nq = kVec ? tn / 4 : 0;
            for (uint32_t q = lane; q < nq; q += 32) {
                const uint32_t x = r - 4 * q * dl;
                put4(base + 4 * q, x, x - dl, x - 2 * dl, x - 3 * dl);
            }
            for (uint32_t l = nq * 4 + lane; l < tn; l += 32) rank[base + l] = (OutT)(r - l * dl);
        } else {
            auto rank_of = [&](uint32_t w) -> uint32_t {
                const unsigned long long sid = off + (w >> 16);
                return sid < R1 ? __ldg(IS1 + sid) - __ldg(&lvl1[sid].y) + (w & 0xFFFFu) : 0u;
            };
            const uint32_t nq = kVec ? tn / 4 : 0;
            for (uint32_t q = lane; q < nq; q += 32) {
                const uint4 w = __ldcs(reinterpret_cast<const uint4*>(node_word + base) + q);
                put4(base + 4 * q, rank_of(w.x), rank_of(w.y), rank_of(w.z), rank_of(w.w));
            }
            for (uint32_t l = nq * 4 + lane; l < tn; l += 32) rank[base + l] = (OutT)rank_of(node_word[base + l]);
        }
    }
}

// contracted list links: segment s -> the segment whose head is succ(end(s))
__global__ void k_rs_contract_link(const uint32_t* __restrict__ headsid, const uint32_t* __restrict__ seg_head,
                                   const uint32_t* __restrict__ seg_succ, uint2* __restrict__ lvl1, ListStatus* st) {
    if (!layout_local(st)) return;
    const unsigned long long S = st->R[1];
    const unsigned long long N = st->R[0];
    bool bad = false;
    for (unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; s < S;
         s += (unsigned long long)gridDim.x * blockDim.x) {
        const uint32_t x = seg_succ[s];
        uint32_t nxt = (uint32_t)s;  // the tail's segment points at itself
        if (x != NIL) {
            const uint32_t y = x < N ? headsid[x] : NIL;
            if (y < S && seg_head[y] == x) {
                nxt = y;
            } else {
                bad = true;  // succ(end) is not a segment head: a node with two predecessors
            }
        }
        lvl1[s].x = nxt;
    }
    if (bad) st->bad = 1;
}

// ---------------------------------------------------------------------------
// host side

struct RsPlan {
    int levels = 0;                              // walked levels (final level = levels)
    uint32_t walk_cap = WALK_CAP_HOPS;
    int load_mode = 0;
    uint32_t fshift = 13;                        // record path: fine window = 2^fshift nodes (32 KiB)
    uint32_t cshift = 20;                        // coarse window = 2^cshift nodes
    uint32_t cbins = 1;                          // number of coarse windows
    unsigned long long nwin = 1;                 // number of fine windows
    uint32_t walk_grid = sm_count() * (2048 / WALK_THREADS);
    bool rec_ok = true;                          // fine windows fit shared memory
    int contract = 1;                            // allow the tile contraction for local layouts
    bool packed = false;                         // level-0 records packed into one u64
    bool fused = false;                          // packed records binned by the walk (no rs5_partition)
    bool coop_top = true;                        // top-level jumping as one cooperative launch
    uint32_t rec_sb = 0, rec_lb = 0;             // packed record: cur << sb | sid << lb | local
    unsigned long long maxchunks = 0;            // record chunks (REC_CH records each)
    uint32_t kbits[SG_MAX_LEVELS] = {};
    uint32_t salt[SG_MAX_LEVELS] = {};
    unsigned long long cap[SG_MAX_LEVELS + 1] = {};  // node capacity per level
};

static uint32_t mix32(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return (uint32_t)x;
}

static RsPlan plan_rs(uint64_t n, uint64_t seed, int out_bytes) {
    RsPlan p;
    // a fine window fills win_kb (64) KiB of shared memory in rs5_scatter;
    // coarse windows: few enough bins for one multisplit
    const Tuning tu = tuning();
    const uint32_t win_kb = tu.rs_win_kb;
    p.fshift = 10;
    while (((size_t)out_bytes << (p.fshift + 1)) <= ((size_t)win_kb << 10)) ++p.fshift;
    uint32_t cs = p.fshift + 1;
    if (cs < 13) cs = 13;  // 2^cshift must be a multiple of MS_TILE
    while (cs < 40 && ((n + (1ull << cs) - 1) >> cs) > 256ull) ++cs;
    while (cs - p.fshift > 8) ++p.fshift;  // <= 256 fine windows per coarse window
    p.rec_ok = ((size_t)out_bytes << p.fshift) <= (200u << 10);  // false only for n > ~2^31
    p.cshift = cs;
    p.cbins = (uint32_t)((n + (1ull << cs) - 1) >> cs);
    p.nwin = (unsigned long long)p.cbins << (cs - p.fshift);
    // one lane per ruler is plenty; every warp that walks may leave one partial chunk
    unsigned long long wg = ((n >> 5) + 2 * WALK_THREADS - 1) / (2 * WALK_THREADS);
    if (wg < (unsigned long long)sm_count()) wg = sm_count();
    if (wg > (unsigned long long)sm_count() * (2048 / WALK_THREADS)) wg = sm_count() * (2048 / WALK_THREADS);
    p.walk_grid = (uint32_t)wg;
    const unsigned long long warps = wg * (WALK_THREADS / 32);
    p.maxchunks = n / (REC_CH - 32) + warps + 2;
    const uint32_t kb0 = tu.rs_kb0;
    const uint32_t kb1 = tu.rs_kb1;
    const uint32_t fin = tu.rs_fin;
    p.walk_cap = tu.rs_walk_cap;
    p.load_mode = (int)tu.rs_load_mode;
    p.contract = (int)tu.rs_contract;
    p.coop_top = tu.rs_coop != 0;

    p.cap[0] = n;
    // a ruler list of at most SG_RS_TOPN (> FINAL_CAP) nodes above level 0 is
    // ranked by multi-CTA pointer jumping (k_rs_top_jump) instead of more walks
    const unsigned long long topn = tu.rs_topn;
    unsigned long long N = n;
    while (N > fin && p.levels < SG_MAX_LEVELS - 1 && !(p.levels >= 1 && N <= topn)) {
        const uint32_t kb = p.levels == 0 ? kb0 : kb1;
        const unsigned long long exp = (N >> kb) + 1;
        unsigned long long cap = exp + exp / 4 + 4096;
        if (cap > N) cap = N;
        p.kbits[p.levels] = kb;
        p.salt[p.levels] = mix32(seed * 0x9E3779B97F4A7C15ull + (uint64_t)p.levels + 1);
        ++p.levels;
        p.cap[p.levels] = cap;
        N = exp;
    }
    if (p.levels > 0 && tu.rs_packed) {
        // field widths: cur needs ceil(log2 n) bits; sid needs room for cap[1]
        // ids plus an all-ones pad value that is never an id
        uint32_t cb = 1, sbits = 1;
        while (cb < 40 && (1ull << cb) < n) ++cb;
        while (sbits < 40 && (1ull << sbits) <= p.cap[1]) ++sbits;
        if (cb <= 32 && cb + sbits + 10 <= 64) {
            p.packed = true;
            p.rec_lb = 64 - cb - sbits;
            p.rec_sb = 64 - cb;
            const unsigned long long lmax = p.rec_lb >= 32 ? 0xFFFFFFFFull : ((1ull << p.rec_lb) - 1);
            if (p.walk_cap > lmax) p.walk_cap = (uint32_t)lmax;  // longer chains: Wyllie fallback
            p.fused = p.cbins <= WB_MAXBINS && tu.rs_fused != 0;
        }
    }
    return p;
}

struct RsBufs {
    ListStatus* st = nullptr;
    unsigned long long* word0 = nullptr;
    uint32_t* rid = nullptr;        // contraction: segment id at each head
    uint2* rgrp = nullptr;          // ruling set: {ruler mask, first id} per 32 nodes
    uint32_t* rec_cur = nullptr;
    unsigned long long* rec_sl = nullptr;
    unsigned long long* pairs = nullptr;
    unsigned long long* cursor = nullptr;  // coarse cursors, then fine cursors
    uint32_t* toff = nullptr;              // rs5_refine tile layout: fine-bin offsets per refine tile
    uint32_t* tiles = nullptr;
    uint32_t* tiles_end = nullptr;
    uint32_t* tiles_run = nullptr;  // per tile: 1 = a run of consecutive ids (census, contraction -> expand)
    uint32_t* tiles_up = nullptr;   // levels >= 1 (level 0's offsets stay for the contraction expand)
    uint32_t* spl[SG_MAX_LEVELS] = {};
    uint2* lvl[SG_MAX_LEVELS + 1] = {};
    unsigned long long* word[SG_MAX_LEVELS + 1] = {};
    uint32_t* IS[SG_MAX_LEVELS + 1] = {};
    uint2* fa = nullptr;
    uint2* fb = nullptr;
};

static bool carve_rs(Carver& c, uint64_t n, const RsPlan& p, RsBufs& b) {
    b.st = c.take<ListStatus>(1);
    b.word0 = c.take<unsigned long long>(n);
    if (p.levels > 0) {
        const unsigned long long nrec = p.fused ? 0 : p.maxchunks * REC_CH;
        b.rid = c.take<uint32_t>(n);
        b.rgrp = c.take<uint2>(n / 32 + 2);
        b.rec_cur = c.take<uint32_t>(p.packed ? 0 : nrec);
        const unsigned long long npad = (unsigned long long)p.cbins << p.cshift;
        b.rec_sl = c.take<unsigned long long>(nrec > npad ? nrec : npad);  // reused by rs5_refine
        b.pairs = c.take<unsigned long long>((unsigned long long)p.cbins << p.cshift);
        b.cursor = c.take<unsigned long long>(p.cbins + p.nwin);
        b.toff = c.take<uint32_t>(p.fused ? (npad / RL_TILE + 1) * (RL_MAXB + 1) : 0);
    }
    const uint64_t ntiles = (n + TILE - 1) / TILE;
    b.tiles = c.take<uint32_t>(ntiles + 1);
    b.tiles_end = c.take<uint32_t>(ntiles + 1);
    b.tiles_run = c.take<uint32_t>(ntiles + 1);
    b.tiles_up = c.take<uint32_t>((p.levels > 0 ? (p.cap[1] + TILE - 1) / TILE : 0) + 1);
    for (int k = 0; k < p.levels; ++k) {
        const unsigned long long cap = p.cap[k + 1];
        b.spl[k] = c.take<uint32_t>(cap);
        b.lvl[k + 1] = c.take<uint2>(cap);
        b.word[k + 1] = c.take<unsigned long long>(cap);
        b.IS[k + 1] = c.take<uint32_t>(cap);
    }
    const unsigned long long fcap = p.levels == 0 ? n : p.cap[p.levels];
    b.fa = c.take<uint2>(fcap);
    b.fb = c.take<uint2>(fcap);
    if (p.levels == 0) b.IS[0] = c.take<uint32_t>(n);
    return c.ok;
}

// ---- Wyllie host driver --------------------------------------------------------

static int jump_rounds(uint64_t n) {
    int r = 0;
    if (n > 1) {
        uint64_t m = n - 1;
        while (m) {
            ++r;
            m >>= 1;
        }
    }
    return r;
}

template <class SuccT, class OutT>
static int wyllie_run(const SuccT* succ, OutT* rank, uint64_t n, int variant, ListStatus* st,
                      unsigned long long* word, cudaStream_t s, Recorder& rec, sg_stats* stats) {
    const int rounds = jump_rounds(n);
    if (stats) stats->rounds = (uint32_t)rounds;
    rec.begin(K_STATUS_INIT, 0, 1, 32, 0);
    k_status_init<<<1, 32, 0, s>>>(st, n);
    rec.end();
    SG_LAUNCH_CHECK();
    if (variant == SG_WY_SINGLE_BLOCK) {
        rec.begin(K_WY_SINGLE, 0, 1, 1024, n * (uint64_t)(rounds + 2));
        k_wy_single<SuccT, OutT><<<1, 1024, 0, s>>>(succ, word, n, st, rank, rounds);
        rec.end();
        SG_LAUNCH_CHECK();
        return SG_OK;
    }
    const uint32_t grid = grid_for(n, JUMP_THREADS, 1, sm_count() * 8);
    rec.begin(K_WY_INIT, 0, grid, JUMP_THREADS, n);
    k_wy_init<SuccT><<<grid, JUMP_THREADS, 0, s>>>(succ, word, n, st);
    rec.end();
    SG_LAUNCH_CHECK();
    const int launches = rounds > 0 ? rounds : 1;  // n == 1: one extraction pass
    for (int r = 1; r <= launches; ++r) {
        rec.begin(K_WY_JUMP, r, grid, JUMP_THREADS, n);
        k_wy_jump<OutT><<<grid, JUMP_THREADS, 0, s>>>(word, n, st, r == launches ? rank : (OutT*)nullptr);
        rec.end();
        SG_LAUNCH_CHECK();
    }
    rec.begin(K_WY_CHECK, 0, 1, 32, 1);
    k_wy_check<<<1, 32, 0, s>>>(word, n, st);
    rec.end();
    SG_LAUNCH_CHECK();
    return SG_OK;
}

template <class SuccT>
static int launch_contract(uint32_t grid, cudaStream_t s, const SuccT* succ, ListStatus* st, const uint32_t* tile_off,
                           uint32_t* headsid, uint32_t* seg_head, uint32_t* seg_succ, uint2* lvl1,
                           uint32_t* node_word, uint32_t* tile_run) {
    const bool vec = ((uintptr_t)succ & 15) == 0;
    auto k = vec ? k_rs_contract<SuccT, true> : k_rs_contract<SuccT, false>;
    SG_CUDA(set_smem_max(k, sizeof(ContractSmem)));
    k<<<grid, TILE_THREADS, sizeof(ContractSmem), s>>>(succ, st, tile_off, headsid, seg_head, seg_succ, lvl1,
                                                       node_word, tile_run);
    return SG_OK;
}

// ---- ruling-set host driver ----------------------------------------------------

template <class SuccT, class OutT>
static int rs_run(const SuccT* succ, OutT* rank, uint64_t n, const RsPlan& p, RsBufs& b, cudaStream_t s,
                  Recorder& rec, sg_stats* stats) {
    rec.begin(K_STATUS_INIT, 0, 1, 32, 0);
    k_status_init<<<1, 32, 0, s>>>(b.st, n);
    rec.end();
    SG_LAUNCH_CHECK();
    const uint32_t walk_grid = p.walk_grid;
    if (p.levels == 0) {
        const uint32_t nt = (uint32_t)((n + TILE - 1) / TILE);
        rec.begin(K_RS_COUNT, 0, nt, TILE_THREADS, n);
        k_rs_count<SuccT, true><<<nt, TILE_THREADS, 0, s>>>(succ, b.tiles, b.st, 0, 1, 0, 0);
        rec.end();
        SG_LAUNCH_CHECK();
        rec.begin(K_RS4_RANK, 0, 1, 1024, n);
        k_rs_final<Level0<SuccT>><<<1, 1024, 0, s>>>(Level0<SuccT>{succ, p.load_mode}, b.fa, b.fb, b.IS[0], b.st, 0);
        rec.end();
        SG_LAUNCH_CHECK();
        const uint32_t g = grid_for(n, 256, 1, sm_count() * 8);
        rec.begin(K_RS5_EXPAND, 0, g, 256, n);
        k_rs_expand_direct<OutT><<<g, 256, 0, s>>>(b.IS[0], rank, n, b.st);
        rec.end();
        SG_LAUNCH_CHECK();
        return SG_OK;
    }
    // downward: census, select, walk per level
    for (int k = 0; k < p.levels; ++k) {
        const unsigned long long capN = p.cap[k];
        const uint32_t nt = (uint32_t)((capN + TILE - 1) / TILE);
        const unsigned long long capR = p.cap[k + 1];
        unsigned long long* wk = k == 0 ? b.word0 : b.word[k];
        uint32_t* tk = k == 0 ? b.tiles : b.tiles_up;
        if (k == 0) {
            const bool narrow = sizeof(SuccT) == 4 && n <= 0x80000000ull;
            const bool vec = ((uintptr_t)succ & 15) == 0;
            auto kc = vec ? (narrow ? k_rs_count0<SuccT, true, true> : k_rs_count0<SuccT, true, false>)
                          : (narrow ? k_rs_count0<SuccT, false, true> : k_rs_count0<SuccT, false, false>);
            // persistent warps stride over the tiles by the grid's warp count, so
            // the grid is what stays resident (48 registers: 5 CTAs per SM, not 8)
            const uint32_t cw = (nt + TILE_THREADS / 32 - 1) / (TILE_THREADS / 32);  // one warp per tile
            const uint32_t cmax = sm_count() * resident_ctas(kc, TILE_THREADS);
            const uint32_t cg = cw < cmax ? cw : cmax;
            rec.begin(K_RS_COUNT, 0, cg, TILE_THREADS, capN);
            kc<<<cg, TILE_THREADS, 0, s>>>(succ, b.tiles, b.tiles_end, b.st, p.kbits[0], p.salt[0], b.tiles_run);
        } else {
            rec.begin(K_RS4_COUNT, k, nt, TILE_THREADS, capN);
            k_rs_count<uint32_t, false><<<nt, TILE_THREADS, 0, s>>>(nullptr, tk, b.st, k, p.kbits[k], p.salt[k], 1);
        }
        rec.end();
        SG_LAUNCH_CHECK();
        rec.begin(k == 0 ? K_RS_SCAN : K_RS4_SCAN, k, 1, SCAN_THREADS, nt);
        if (k == 0)
            k_rs_scan0<<<1, SCAN_THREADS, 0, s>>>(b.tiles, b.tiles_end, b.st, capR, p.contract);
        else
            k_rs_scan<<<1, SCAN_THREADS, 0, s>>>(tk, b.st, k, capR);
        rec.end();
        SG_LAUNCH_CHECK();
        rec.begin(k == 0 ? K_RS_SELECT : K_RS4_SELECT, k, nt, TILE_THREADS, capN);
        if (k == 0) {  // warp per tile, no block barrier
            const unsigned long long ctas = (nt + 7) / 8;
            const uint32_t g0 = (uint32_t)(ctas < (unsigned long long)sm_count() * 8 ? ctas : sm_count() * 8);
            k_rs_select0<<<g0 ? g0 : 1, 256, 0, s>>>(tk, b.spl[0], b.st, p.kbits[0], p.salt[0], capR, b.rgrp);
        } else {
            k_rs_select<false><<<nt < sm_count() * 8 ? nt : sm_count() * 8, TILE_THREADS, 0, s>>>(
                tk, b.spl[k], wk, b.st, k, p.kbits[k], p.salt[k], capR, nullptr);
        }
        rec.end();
        SG_LAUNCH_CHECK();
        if (k == 0) {
            // scattered layouts: record walk; local layouts: tile contraction
            if (p.fused) {
                SG_CUDA(cudaMemsetAsync(b.cursor, 0, sizeof(unsigned long long) * (size_t)(p.cbins + p.nwin), s));
                // 2 x 1024 threads per SM (the walk needs every resident lane:
                // 1536 per SM was 60 % slower), 32-record buffers per window
                constexpr int WB_T = 1024, WB_C = 2;
                constexpr uint32_t WB_S = 32;
                auto kern = k_rs_walk_bin<SuccT, WB_T, WB_C, WB_S>;
                const size_t smem = (size_t)p.cbins * WB_S * sizeof(unsigned long long);
                SG_CUDA(set_smem_max(kern, smem));
                rec.begin(K_RS3_WALK, 0, sm_count() * WB_C, WB_T, capN);
                kern<<<sm_count() * WB_C, WB_T, smem, s>>>(succ, b.rgrp, b.spl[0], b.lvl[1], b.cursor, b.pairs, b.st,
                                                     p.kbits[0], p.salt[0], p.walk_cap, p.load_mode, p.rec_sb, p.rec_lb,
                                                     p.cshift, p.cbins);
            } else {
            rec.begin(K_RS3_WALK, 0, walk_grid, WALK_THREADS, capN);
            if (p.packed)
                k_rs_walk_rec<SuccT, true><<<walk_grid, WALK_THREADS, 0, s>>>(
                    succ, b.rgrp, b.spl[0], b.lvl[1], b.rec_cur, b.rec_sl, b.st, p.kbits[0], p.salt[0], p.walk_cap,
                    p.maxchunks, p.load_mode, p.rec_sb, p.rec_lb);
            else
                k_rs_walk_rec<SuccT, false><<<walk_grid, WALK_THREADS, 0, s>>>(
                    succ, b.rgrp, b.spl[0], b.lvl[1], b.rec_cur, b.rec_sl, b.st, p.kbits[0], p.salt[0], p.walk_cap,
                    p.maxchunks, p.load_mode, 0, 0);
            }
            rec.end();
            SG_LAUNCH_CHECK();
            const uint32_t cg = nt < sm_count() * CT_CTAS_PER_SM ? nt : sm_count() * CT_CTAS_PER_SM;
            rec.begin(K_RS_CONTRACT, 0, cg, TILE_THREADS, capN);
            const int rc = launch_contract<SuccT>(cg, s, succ, b.st, b.tiles, b.rid, b.spl[0], b.IS[1], b.lvl[1],
                                                  reinterpret_cast<uint32_t*>(b.word0), b.tiles_run);
            if (rc != SG_OK) return rc;
            rec.end();
            SG_LAUNCH_CHECK();
            const uint32_t lg = grid_for(capR, 256, 1, sm_count() * 8);
            rec.begin(K_RS_CONTRACT_LINK, 0, lg, 256, capR);
            k_rs_contract_link<<<lg, 256, 0, s>>>(b.rid, b.spl[0], b.IS[1], b.lvl[1], b.st);
        } else {
            // about one sublist per lane: a bigger grid only queues its warps
            // on the work-queue atomic (~30 us at the small levels)
            unsigned long long wgk = (capR + WALK_THREADS - 1) / WALK_THREADS;
            if (wgk > walk_grid) wgk = walk_grid;
            if (wgk < 1) wgk = 1;
            rec.begin(K_RS4_WALK, k, (uint32_t)wgk, WALK_THREADS, capN);
            k_rs_walk<LevelK><<<(uint32_t)wgk, WALK_THREADS, 0, s>>>(LevelK{b.lvl[k]}, wk, b.spl[k], b.lvl[k + 1], b.st,
                                                                 k, p.kbits[k], p.salt[k], p.walk_cap);
        }
        rec.end();
        SG_LAUNCH_CHECK();
    }
    // top: single CTA on the last ruler list, or multi-CTA jumping if it is big
    const int L = p.levels;
    bool coop_done = false;
    if (p.cap[L] > FINAL_CAP && p.coop_top) {
        // resident 512-thread CTAs per SM for the cooperative launch, per device
        static std::atomic<int> coop_cache[64];  // 0: unknown, else blocks + 1
        int cdev = 0;
        cudaGetDevice(&cdev);
        std::atomic<int>& slot = coop_cache[cdev >= 0 && cdev < 64 ? cdev : 0];
        int coop_blocks = slot.load(std::memory_order_relaxed) - 1;
        if (coop_blocks < 0) {
            int nb = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_rs_top_coop<LevelK>, 512, 0) != cudaSuccess) {
                cudaGetLastError();
                nb = 0;
            }
            coop_blocks = nb;
            slot.store(nb + 1, std::memory_order_relaxed);
        }
        if (coop_blocks > 0) {
            LevelK view{b.lvl[L]};
            uint2* A = b.fa;
            ListStatus* stp = b.st;
            int lv = L;
            uint32_t* isp = b.IS[L];
            int rounds = jump_rounds(p.cap[L]) + 1;
            void* args[] = {&view, &A, &stp, &lv, &isp, &rounds};
            const uint32_t g = (uint32_t)(sm_count() * (coop_blocks < 2 ? coop_blocks : 2));
            rec.begin(K_RS4_RANK, L, g, 512, p.cap[L]);
            const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_rs_top_coop<LevelK>, g, 512, args, 0, s);
            rec.end();
            if (e == cudaSuccess) {
                coop_done = true;
            } else {
                (void)cudaGetLastError();  // not co-resident here: the multi-launch rounds below
            }
        }
    }
    if (coop_done) {
    } else if (p.cap[L] > FINAL_CAP) {
        const uint32_t g = grid_for(p.cap[L], 256, 4, sm_count() * 8);
        rec.begin(K_RS4_RANK, L, g, 256, p.cap[L]);
        k_rs_top_init<LevelK><<<g, 256, 0, s>>>(LevelK{b.lvl[L]}, b.fa, b.st, L);
        rec.end();
        SG_LAUNCH_CHECK();
        const int rounds = jump_rounds(p.cap[L]) + 1;
        for (int r = 1; r <= rounds; ++r) {
            rec.begin(K_RS4_RANK, L, g, 256, p.cap[L]);
            k_rs_top_jump<<<g, 256, 0, s>>>(b.fa, b.st, L, r == rounds ? b.IS[L] : nullptr);
            rec.end();
            SG_LAUNCH_CHECK();
        }
    } else {
        rec.begin(K_RS4_RANK, L, 1, 1024, p.cap[L]);
        k_rs_final<LevelK><<<1, 1024, 0, s>>>(LevelK{b.lvl[L]}, b.fa, b.fb, b.IS[L], b.st, L);
        rec.end();
        SG_LAUNCH_CHECK();
    }
    // upward: expand
    for (int k = L - 1; k >= 1; --k) {
        const uint32_t g = grid_for(p.cap[k], 256, 1, sm_count() * 8);
        rec.begin(K_RS4_EXPAND, k, g, 256, p.cap[k]);
        k_rs_expand_k<<<g, 256, 0, s>>>(b.word[k], b.IS[k + 1], b.IS[k], b.st, k);
        rec.end();
        SG_LAUNCH_CHECK();
    }
    {  // local layouts: expand the contraction
        const uint32_t eg = grid_for(n / 4 + 1, 256, 1, sm_count() * 8);
        rec.begin(K_RS5_EXPAND, 0, eg, 256, n);
        if (((uintptr_t)rank & 15) == 0)
            k_rs_contract_expand<OutT, true><<<eg, 256, 0, s>>>(reinterpret_cast<const uint32_t*>(b.word0), b.tiles,
                                                                b.lvl[1], b.IS[1], rank, b.st, b.tiles_run);
        else
            k_rs_contract_expand<OutT, false><<<eg, 256, 0, s>>>(reinterpret_cast<const uint32_t*>(b.word0), b.tiles,
                                                                 b.lvl[1], b.IS[1], rank, b.st, b.tiles_run);
        rec.end();
        SG_LAUNCH_CHECK();
    }
    // scattered layouts: rank the records, bucket them by window, scatter
    constexpr uint32_t tile2 = MS_THREADS * MS2_ITEMS;
    const uint32_t persist2 = sm_count() * 2;
    const size_t sm_ref2 = (size_t)tile2 * 8 + MsSmem::bytes(1u << (p.cshift - p.fshift), tile2);
    if (!p.fused) {
        SG_CUDA(cudaMemsetAsync(b.cursor, 0, sizeof(unsigned long long) * (size_t)(p.cbins + p.nwin), s));
        const size_t sm_part2 = (size_t)tile2 * 12 + MsSmem::bytes(p.cbins, tile2);
        auto kp = p.packed ? k_rs_rec_partition2<MS2_ITEMS, true> : k_rs_rec_partition2<MS2_ITEMS, false>;
        SG_CUDA(set_smem_max(kp, sm_part2));
        rec.begin(K_RS5_PARTITION, 0, persist2, MS_THREADS, n);
        kp<<<persist2, MS_THREADS, sm_part2, s>>>(b.rec_cur, b.rec_sl, b.IS[1], b.cursor, b.pairs, b.st, p.cshift,
                                                  p.cbins, p.rec_sb, p.rec_lb);
        rec.end();
        SG_LAUNCH_CHECK();
    }
    const uint32_t fbits_r = p.cshift - p.fshift;
    const Tuning tu_r = tuning();
    // the lean refine keeps local (< walk cap) in 20 bits next to the 8-bit warp rank
    const bool lean_ok = p.fused && fbits_r <= 6 && p.rec_lb < 32 && p.walk_cap < (1u << 20);
    bool tiled = false;
    if (p.fused && tu_r.rs_refine == 7) {  // one pass: ranks stored straight from the records
        const unsigned long long per = (unsigned long long)RD_THREADS * RD_IT;
        const uint32_t g = (uint32_t)((n + per - 1) / per);
        rec.begin(K_RS5_REFINE, 0, g, RD_THREADS, n);
        k_rs_refine_direct<OutT><<<g, RD_THREADS, 0, s>>>(b.pairs, rank, b.st, n, p.cshift, b.IS[1], p.rec_sb,
                                                           p.rec_lb);
        rec.end();
        SG_LAUNCH_CHECK();
        if (stats) stats->levels = (uint32_t)L;
        return SG_OK;
    }
    if (lean_ok && tu_r.rs_refine == 0 && ((1ull << p.cshift) % RA_TILE) == 0) {
        const size_t sma = ra_smem_bytes();  // (k_rs_refine_atom: staging + one sorted tile)
        SG_CUDA(set_smem_max(k_rs_refine_atom, sma));
        const uint32_t g = sm_count() * RA_CTAS_PER_SM;
        rec.begin(K_RS5_REFINE, 0, g, RA_THREADS, n);
        k_rs_refine_atom<<<g, RA_THREADS, sma, s>>>(b.pairs, b.cursor + p.cbins, b.rec_sl, b.st, n, p.cshift, p.fshift,
                                                   b.IS[1], p.rec_sb, p.rec_lb);
    } else if (lean_ok && tu_r.rs_refine != 1) {
        // SG_RS_REFINE: 0 k_rs_refine_atom above (default), 6 lean + ballots, 2 lean + match.any, 3 lean + alternate,
        // 4 lean + ballots in the tile layout (k_rs_rec_scatter_tiles); 5 lean + shared atomics;
        // 1 the ms_split_fn refine below
        tiled = tu_r.rs_refine == 4;
        const int pm = tu_r.rs_refine == 2 ? 0 : (tu_r.rs_refine == 3 ? 2 : (tu_r.rs_refine == 5 ? 3 : 1));  // 6: ballots
        using KL = void (*)(const unsigned long long*, unsigned long long*, unsigned long long*, ListStatus*,
                            unsigned long long, uint32_t, uint32_t, const uint32_t*, uint32_t, uint32_t, uint32_t*);
        KL kl;
        if (tiled)
            kl = fbits_r <= 2 ? k_rs_refine_lean<2, 1, true>
                              : (fbits_r <= 4 ? k_rs_refine_lean<4, 1, true> : k_rs_refine_lean<6, 1, true>);
        else if (pm == 0)
            kl = k_rs_refine_lean<6, 0>;
        else if (pm == 3)
            kl = k_rs_refine_lean<6, 3>;
        else if (pm == 2)
            kl = fbits_r <= 4 ? k_rs_refine_lean<4, 2> : k_rs_refine_lean<6, 2>;
        else
            kl = fbits_r <= 2 ? k_rs_refine_lean<2, 1>
                              : (fbits_r <= 4 ? k_rs_refine_lean<4, 1> : k_rs_refine_lean<6, 1>);
        const size_t smr = rl_smem_bytes();
        SG_CUDA(set_smem_max(kl, smr));
        const uint32_t g = sm_count() * RL_CTAS_PER_SM;
        rec.begin(K_RS5_REFINE, 0, g, RL_THREADS, n);
        kl<<<g, RL_THREADS, smr, s>>>(b.pairs, b.cursor + p.cbins, b.rec_sl, b.st, n, p.cshift, p.fshift, b.IS[1],
                                      p.rec_sb, p.rec_lb, b.toff);
    } else if (p.fused) {  // 8 records per thread, 3 CTAs per SM: more warps to hide the IS_1 gathers
        constexpr uint32_t t8 = MS_THREADS * 8;
        const size_t sm8 = (size_t)t8 * 8 + MsSmem::bytes(1u << (p.cshift - p.fshift), t8);
        const uint32_t fbits = p.cshift - p.fshift;  // ballots per element in the split
        auto kr = fbits <= 4 ? k_rs_rec_refine2<8, 1, 4>
                             : (fbits <= 6 ? k_rs_rec_refine2<8, 1, 6> : k_rs_rec_refine2<8, 1, 8>);
        SG_CUDA(set_smem_max(kr, sm8));
        rec.begin(K_RS5_REFINE, 0, sm_count() * 3, MS_THREADS, n);
        kr<<<sm_count() * 3, MS_THREADS, sm8, s>>>(b.pairs, b.cursor + p.cbins, b.rec_sl, b.st, n, p.cshift, p.fshift,
                                             b.IS[1], p.rec_sb, p.rec_lb);
    } else {
        auto kr = k_rs_rec_refine2<MS2_ITEMS, 0>;
        SG_CUDA(set_smem_max(kr, sm_ref2));
        rec.begin(K_RS5_REFINE, 0, persist2, MS_THREADS, n);
        kr<<<persist2, MS_THREADS, sm_ref2, s>>>(b.pairs, b.cursor + p.cbins, b.rec_sl, b.st, n, p.cshift, p.fshift,
                                                 b.IS[1], p.rec_sb, p.rec_lb);
    }
    rec.end();
    SG_LAUNCH_CHECK();
    if (tiled) {
        SG_CUDA(set_smem_max(k_rs_rec_scatter_tiles<OutT>, sizeof(OutT) << p.fshift));
        rec.begin(K_RS5_SCATTER, 0, (uint32_t)p.nwin, 256, n);
        k_rs_rec_scatter_tiles<OutT><<<(uint32_t)p.nwin, 256, sizeof(OutT) << p.fshift, s>>>(
            b.rec_sl, b.toff, rank, n, p.cshift, p.fshift, b.st, ((uintptr_t)rank & 15) == 0 ? 1 : 0);
    } else {
        SG_CUDA(set_smem_max(k_rs_rec_scatter<OutT>, sizeof(OutT) << p.fshift));
        rec.begin(K_RS5_SCATTER, 0, (uint32_t)p.nwin, 256, n);
        k_rs_rec_scatter<OutT><<<(uint32_t)p.nwin, 256, sizeof(OutT) << p.fshift, s>>>(
            b.rec_sl, rank, n, p.fshift, b.st, ((uintptr_t)rank & 15) == 0 ? 1 : 0);
    }
    rec.end();
    SG_LAUNCH_CHECK();
    if (stats) {
        stats->levels = (uint32_t)L;
    }
    return SG_OK;
}

static int read_status(const ListStatus* st_dev, ListStatus& h, cudaStream_t s) {
    SG_CUDA(cudaMemcpyAsync(&h, st_dev, sizeof(ListStatus), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    return SG_OK;
}

// pinned host copy of the status block, enqueued behind the pipeline so the
// call synchronises once
static ListStatus* pinned_status() {
    static thread_local ListStatus* p = nullptr;
    if (!p && cudaMallocHost(&p, sizeof(ListStatus)) != cudaSuccess) p = nullptr;
    return p;
}

// meta["splitter_set"] request, served on the same stream before the sync
struct MetaReq {
    const int64_t* spl;
    uint32_t r;
    int64_t* dev_out;   // 3 x r
    int64_t* host_out;  // 3 x r (pinned for an async copy)
    void* ws;
    size_t ws_bytes;
};

template <class OutT>
static int enqueue_meta(const MetaReq* mr, const void* rank, uint64_t n, cudaStream_t s) {
    if (!mr || mr->r == 0) return SG_OK;
    const int odt = sizeof(OutT) == 8 ? SG_I64 : (std::is_signed<OutT>::value ? SG_I32 : SG_U32);
    const int rc = sg_splitter_meta(rank, odt, n, mr->spl, mr->r, mr->dev_out, mr->ws, mr->ws_bytes, s);
    if (rc != SG_OK) return rc;
    if (mr->host_out)
        SG_CUDA(cudaMemcpyAsync(mr->host_out, mr->dev_out, sizeof(int64_t) * 3 * (size_t)mr->r, cudaMemcpyDeviceToHost,
                                s));
    return SG_OK;
}

// classify a finished pipeline: SG_OK, SG_ERR_INVALID_LIST (viol filled)
static int classify(const ListStatus& h, uint64_t n, sg_violation* v) {
    sg_violation tmp;
    if (!v) v = &tmp;
    v->kind = SG_LIST_OK;
    v->index = -1;
    v->pad = 0;
    if (h.oor_first != NONE64) {
        v->kind = SG_LIST_OUT_OF_RANGE;
        v->index = (int64_t)h.oor_first;
        return SG_ERR_INVALID_LIST;
    }
    if (h.loop_count == 0) {
        v->kind = SG_LIST_NO_TAIL;
        return SG_ERR_INVALID_LIST;
    }
    if (h.loop_count > 1) {
        v->kind = SG_LIST_MULTIPLE_SELF_LOOPS;  // index: host recomputes loops[1]
        return SG_ERR_INVALID_LIST;
    }
    if (h.bad || !h.head_ok || h.head_sum != n) {
        v->kind = SG_LIST_UNREACHABLE;  // index: host recomputes the first unreached node
        return SG_ERR_INVALID_LIST;
    }
    return SG_OK;
}

template <class SuccT, class OutT>
static int wyllie_entry(const void* succ_v, void* rank_v, uint64_t n, int variant, void* ws, size_t ws_bytes,
                        cudaStream_t s, sg_stats* stats, sg_violation* viol) {
    Carver c(ws, ws_bytes);
    ListStatus* st = c.take<ListStatus>(1);
    unsigned long long* word = c.take<unsigned long long>(n);
    if (!c.ok) return SG_ERR_WORKSPACE;
    Recorder rec(stats, s);
    int rc = wyllie_run<SuccT, OutT>((const SuccT*)succ_v, (OutT*)rank_v, n, variant, st, word, s, rec, stats);
    if (rc != SG_OK) return rc;
    SG_CUDA(rec.finish());
    ListStatus h;
    rc = read_status(st, h, s);
    if (rc != SG_OK) return rc;
    return classify(h, n, viol);
}

template <class SuccT, class OutT>
static int rs_entry(const void* succ_v, void* rank_v, uint64_t n, uint64_t seed, void* ws, size_t ws_bytes,
                    cudaStream_t s, sg_stats* stats, sg_violation* viol, const MetaReq* mr) {
    HostClock hc("rs_entry");
    const RsPlan p = plan_rs(n, seed, (int)sizeof(OutT));
    ms_configure();
    Carver c(ws, ws_bytes);
    RsBufs b;
    if (!carve_rs(c, n, p, b)) return SG_ERR_WORKSPACE;
    if (stats) {
        stats->levels = (uint32_t)p.levels;
        stats->fallback = 0;
        stats->list_path = 0;
        for (int k = 0; k < SG_MAX_LEVELS; ++k) stats->level_size[k] = 0;
    }
    Recorder rec(stats, s);
    auto wyllie_instead = [&](Recorder& r, sg_stats* st) -> int {
        if (stats) stats->fallback = 1;
        return wyllie_run<SuccT, OutT>((const SuccT*)succ_v, (OutT*)rank_v, n, SG_WY_MULTI_KERNEL, b.st, b.word0, s, r,
                                       st);
    };
    ListStatus* hs = pinned_status();
    ListStatus hloc;
    ListStatus& h = hs ? *hs : hloc;
    if (p.levels > 0 && !p.rec_ok) {
        // output windows would not fit shared memory (n > ~2^31): pointer jumping
        int rc = wyllie_instead(rec, stats);
        if (rc != SG_OK) return rc;
        rc = enqueue_meta<OutT>(mr, rank_v, n, s);
        if (rc != SG_OK) return rc;
        SG_CUDA(rec.finish());
        rc = read_status(b.st, h, s);
        if (rc != SG_OK) return rc;
        return classify(h, n, viol);
    }
    hc.mark("setup");
    int rc = rs_run<SuccT, OutT>((const SuccT*)succ_v, (OutT*)rank_v, n, p, b, s, rec, stats);
    if (rc != SG_OK) return rc;
    hc.mark("pipeline enqueued");
    rc = enqueue_meta<OutT>(mr, rank_v, n, s);
    if (rc != SG_OK) return rc;
    if (hs) SG_CUDA(cudaMemcpyAsync(hs, b.st, sizeof(ListStatus), cudaMemcpyDeviceToHost, s));
    hc.mark("meta enqueued");
    SG_CUDA(cudaStreamSynchronize(s));
    hc.mark("synchronised");
    SG_CUDA(rec.finish());  // the one synchronisation of a normal call
    hc.mark("events read");
    if (!hs) {
        rc = read_status(b.st, h, s);
        if (rc != SG_OK) return rc;
    }
    if (stats) {
        for (int k = 0; k <= p.levels && k < SG_MAX_LEVELS; ++k) stats->level_size[k] = h.R[k];
        stats->list_path = h.local ? 1u : 0u;
    }
    if (h.oor_first == NONE64 && h.loop_count == 1 && h.overflow) {
        // a walk hit the hop cap or a level overflowed its capacity: rank the
        // list by pointer jumping instead (terminates on every input)
        Recorder rec2(nullptr, s);
        rc = wyllie_instead(rec2, nullptr);
        if (rc != SG_OK) return rc;
        rc = enqueue_meta<OutT>(mr, rank_v, n, s);
        if (rc != SG_OK) return rc;
        SG_CUDA(rec2.finish());
        rc = read_status(b.st, h, s);
        if (rc != SG_OK) return rc;
    }
    return classify(h, n, viol);
}

}  // namespace sg

using namespace sg;

#define SG_DISPATCH_LIST(FN, SDT, ODT, ...)                                                   \
    do {                                                                                      \
        if ((SDT) == SG_U32 && (ODT) == SG_U32) return FN<uint32_t, uint32_t>(__VA_ARGS__);  \
        if ((SDT) == SG_U32 && (ODT) == SG_I32) return FN<uint32_t, int32_t>(__VA_ARGS__);   \
        if ((SDT) == SG_U32 && (ODT) == SG_I64) return FN<uint32_t, int64_t>(__VA_ARGS__);   \
        if ((SDT) == SG_I32 && (ODT) == SG_U32) return FN<int32_t, uint32_t>(__VA_ARGS__);   \
        if ((SDT) == SG_I32 && (ODT) == SG_I32) return FN<int32_t, int32_t>(__VA_ARGS__);    \
        if ((SDT) == SG_I32 && (ODT) == SG_I64) return FN<int32_t, int64_t>(__VA_ARGS__);    \
        if ((SDT) == SG_I64 && (ODT) == SG_U32) return FN<int64_t, uint32_t>(__VA_ARGS__);   \
        if ((SDT) == SG_I64 && (ODT) == SG_I32) return FN<int64_t, int32_t>(__VA_ARGS__);    \
        if ((SDT) == SG_I64 && (ODT) == SG_I64) return FN<int64_t, int64_t>(__VA_ARGS__);    \
        return SG_ERR_VALUE;                                                                  \
    } while (0)

extern "C" {

size_t sg_wyllie_workspace_bytes(uint64_t n) {
    Carver c(nullptr, 0);
    c.take<ListStatus>(1);
    c.take<unsigned long long>(n);
    return c.off + 256;
}

size_t sg_rs_workspace_bytes(uint64_t n) {
    size_t best = 0;
    for (int ob : {4, 8}) {  // window geometry depends on the output width
        const RsPlan p = plan_rs(n, 0, ob);
        Carver c(nullptr, 0);
        RsBufs b;
        carve_rs(c, n, p, b);
        if (c.off + 256 > best) best = c.off + 256;
    }
    return best;
}

int sg_wyllie_rank(const void* succ, int succ_dtype, void* rank, int rank_dtype, uint64_t n, int variant, void* ws,
                   size_t ws_bytes, void* stream, sg_stats* st, sg_violation* viol) {
    if (n == 0 || n >= 0xFFFFFFFFull) return SG_ERR_CAPABILITY;
    if (variant != SG_WY_MULTI_KERNEL && variant != SG_WY_SINGLE_BLOCK) return SG_ERR_VALUE;
    ::sg::apply_tuning();
    if (st) memset(st, 0, sizeof(sg_stats));
    SG_DISPATCH_LIST(wyllie_entry, succ_dtype, rank_dtype, succ, rank, n, variant, ws, ws_bytes, (cudaStream_t)stream,
                     st, viol);
}

int sg_rs_rank(const void* succ, int succ_dtype, void* rank, int rank_dtype, uint64_t n, uint64_t seed, void* ws,
               size_t ws_bytes, void* stream, sg_stats* st, sg_violation* viol) {
    if (n == 0 || n >= 0xFFFFFFFFull) return SG_ERR_CAPABILITY;
    ::sg::apply_tuning();
    if (st) memset(st, 0, sizeof(sg_stats));
    SG_DISPATCH_LIST(rs_entry, succ_dtype, rank_dtype, succ, rank, n, seed, ws, ws_bytes, (cudaStream_t)stream, st,
                     viol, (const MetaReq*)nullptr);
}

int sg_rs_rank_meta(const void* succ, int succ_dtype, void* rank, int rank_dtype, uint64_t n, uint64_t seed, void* ws,
                    size_t ws_bytes, const int64_t* spl, uint32_t r, int64_t* meta_dev, int64_t* meta_host,
                    void* meta_ws, size_t meta_ws_bytes, void* stream, sg_stats* st, sg_violation* viol) {
    if (n == 0 || n >= 0xFFFFFFFFull) return SG_ERR_CAPABILITY;
    ::sg::apply_tuning();
    if (st) memset(st, 0, sizeof(sg_stats));
    const MetaReq mr{spl, r, meta_dev, meta_host, meta_ws, meta_ws_bytes};
    SG_DISPATCH_LIST(rs_entry, succ_dtype, rank_dtype, succ, rank, n, seed, ws, ws_bytes, (cudaStream_t)stream, st,
                     viol, &mr);
}

}  // extern "C"
