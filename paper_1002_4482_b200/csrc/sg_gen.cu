// sg_gen.cu -- device input generation bit-exact with the reference
// generators (gen.py), plus small helpers.
//
// KISS64 (gen.py:30-64) is a sum of three recurrences; the caller computes
// the jump-ahead state of every chunk on the host (paper_1002_4482_b200/gen.py)
// and each thread then runs the exact scalar recurrence over its chunk, so
// draw j of the device stream equals draw j of kiss_batch().
#include <cub/device/device_radix_sort.cuh>

#include "sg_internal.cuh"

namespace sg {

// ---- splitter meta (listrank.py:252-357 outputs, derived from the ranks) ----
// key = n-1-rank (ascending = list order), value = splitter index
template <class RankT>
__global__ void k_spl_keys(const RankT* __restrict__ rank, const long long* __restrict__ spl, uint32_t r,
                           unsigned long long n, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= r) return;
    const unsigned long long rk = (unsigned long long)rank[spl[i]];
    keys[i] = (uint32_t)(n - 1 - rk);
    vals[i] = i;
}

// out[0][i] = splitter rank, out[1][i] = sublist length (to the next
// splitter in list order, the last one to the tail), out[2][i] = reduced
// successor (the last splitter points at itself)
__global__ void k_spl_meta(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ order, uint32_t r,
                           unsigned long long n, long long* __restrict__ out) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= r) return;
    const uint32_t i = order[j];
    const long long sr = (long long)(n - 1 - keys[j]);
    const bool last = j + 1 == r;
    out[i] = sr;
    out[(size_t)r + i] = last ? sr + 1 : sr - (long long)(n - 1 - keys[j + 1]);
    out[2 * (size_t)r + i] = last ? (long long)i : (long long)order[j + 1];
}

// Up to SPL_BLOCK_MAX splitters: keys, sort and meta in one CTA (one launch
// instead of cub's five; the meta sits on the tail of every rs_rank call).
// Random splitters have near-uniform ranks, so a counting sort by the top
// log2(SPL_BLOCK_MAX) key bits leaves ~1 key per bucket; each bucket is then
// finished by insertion sort (keys are distinct ranks).
constexpr int SPL_THREADS = 1024;
constexpr uint32_t SPL_BLOCK_MAX = 16384;
constexpr int SPL_PER = SPL_BLOCK_MAX / SPL_THREADS;

// keys come from k_spl_keys (many CTAs: one SM alone cannot keep enough
// random rank gathers in flight -- they cost ~30 us here)
__global__ void __launch_bounds__(SPL_THREADS) k_spl_meta_block(const uint32_t* __restrict__ keys, uint32_t r,
                                                                unsigned long long n, int shift,
                                                                long long* __restrict__ out) {
    extern __shared__ __align__(16) uint32_t spl_sm[];
    uint32_t* start = spl_sm;                    // [SPL_BLOCK_MAX + 1] bucket counts, then starts
    uint32_t* skey = start + SPL_BLOCK_MAX + 1;  // [r] keys in list order
    uint32_t* sval = skey + SPL_BLOCK_MAX;       // [r] splitter indices in list order
    __shared__ uint32_t warp_tot[SPL_THREADS / 32];
    const uint32_t t = threadIdx.x, lane = t & 31u, w = t >> 5;
    // (ranks of an invalid list are garbage: keep every key inside the table)
    auto bucket = [&](uint32_t k) { return min(k >> shift, SPL_BLOCK_MAX - 1); };
    for (uint32_t b = t; b <= SPL_BLOCK_MAX; b += SPL_THREADS) start[b] = 0;
    __syncthreads();
    uint32_t key[SPL_PER], slot[SPL_PER];
#pragma unroll
    for (int j = 0; j < SPL_PER; ++j) {
        const uint32_t i = j * SPL_THREADS + t;
        key[j] = i < r ? __ldg(keys + i) : 0u;
    }
#pragma unroll
    for (int j = 0; j < SPL_PER; ++j) {
        const uint32_t i = j * SPL_THREADS + t;
        slot[j] = i < r ? atomicAdd(&start[bucket(key[j])], 1u) : 0u;
    }
    __syncthreads();
    // exclusive scan of the counts: thread t owns buckets [t*SPL_PER, (t+1)*SPL_PER)
    uint32_t c[SPL_PER], tot = 0;
#pragma unroll
    for (int j = 0; j < SPL_PER; ++j) {
        c[j] = start[t * SPL_PER + j];
        tot += c[j];
    }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += v;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    uint32_t pre = 0;
    for (uint32_t k = 0; k < w; ++k) pre += warp_tot[k];
    uint32_t run = pre + incl - tot;
#pragma unroll
    for (int j = 0; j < SPL_PER; ++j) {
        start[t * SPL_PER + j] = run;
        run += c[j];
    }
    if (t == SPL_THREADS - 1) start[SPL_BLOCK_MAX] = run;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < SPL_PER; ++j) {
        const uint32_t i = j * SPL_THREADS + t;
        if (i < r) {
            const uint32_t pos = start[bucket(key[j])] + slot[j];
            skey[pos] = key[j];
            sval[pos] = i;
        }
    }
    __syncthreads();
    // finish each bucket (a handful of keys at most for random splitters)
    for (uint32_t b = t; b < SPL_BLOCK_MAX; b += SPL_THREADS) {
        const uint32_t lo = start[b], hi = start[b + 1];
        for (uint32_t x = lo + 1; x < hi; ++x) {
            const uint32_t kx = skey[x], vx = sval[x];
            uint32_t y = x;
            while (y > lo && skey[y - 1] > kx) {
                skey[y] = skey[y - 1];
                sval[y] = sval[y - 1];
                --y;
            }
            skey[y] = kx;
            sval[y] = vx;
        }
    }
    __syncthreads();
    // the three output rows are indexed by splitter: permute each through
    // shared memory (the bucket table is free now) and store it coalesced
    uint32_t* stage = start;
    for (int row = 0; row < 3; ++row) {
        for (uint32_t q = t; q < r; q += SPL_THREADS) {
            const uint32_t i = sval[q];
            const uint32_t k = skey[q];
            const bool last = q + 1 == r;
            uint32_t v;
            if (row == 0)
                v = (uint32_t)(n - 1 - k);                       // splitter rank
            else if (row == 1)
                v = last ? (uint32_t)(n - k) : skey[q + 1] - k;  // sublist length
            else
                v = last ? i : sval[q + 1];                      // reduced successor
            stage[i] = v;
        }
        __syncthreads();
        for (uint32_t i = t; i < r; i += SPL_THREADS) out[(size_t)row * r + i] = (long long)stage[i];
        __syncthreads();
    }
}

static int launch_spl_block(const uint32_t* keys, uint32_t r, uint64_t n, int bits, int64_t* out, cudaStream_t s) {
    int lb = 0;
    while ((1u << (lb + 1)) <= SPL_BLOCK_MAX) ++lb;
    const int shift = bits > lb ? bits - lb : 0;
    const size_t smem = sizeof(uint32_t) * (3 * (size_t)SPL_BLOCK_MAX + 1);
    auto k = k_spl_meta_block;
    SG_CUDA(set_smem_max(k, smem));
    k<<<1, SPL_THREADS, smem, s>>>(keys, r, n, shift, (long long*)out);
    SG_LAUNCH_CHECK();
    return SG_OK;
}

__global__ void __launch_bounds__(128) k_kiss(const unsigned long long* __restrict__ states, unsigned long long chunks,
                                              unsigned long long chunk_len, unsigned long long n,
                                              unsigned long long* __restrict__ out) {
    const unsigned long long k = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= chunks) return;
    unsigned long long x = states[4 * k + 0], y = states[4 * k + 1], z = states[4 * k + 2], c = states[4 * k + 3];
    const unsigned long long a = k * chunk_len;
    unsigned long long b = a + chunk_len;
    if (b > n) b = n;
    for (unsigned long long j = a; j < b; ++j) {
        // multiply-with-carry
        const unsigned long long t = (x << 58) + c;
        c = x >> 6;
        x += t;
        c += (x < t) ? 1ull : 0ull;
        // xorshift
        y ^= y << 13;
        y ^= y >> 17;
        y ^= y << 43;
        // congruential
        z = 6906969069ull * z + 1234567ull;
        out[j] = x + y + z;
    }
}

template <class T>
__global__ void k_list_from_order(const long long* __restrict__ perm, unsigned long long n, T* __restrict__ succ) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long j = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const unsigned long long a = j == 0 ? 0ull : 1ull + (unsigned long long)perm[j - 1];
        const unsigned long long b = (j + 1 < n) ? 1ull + (unsigned long long)perm[j] : a;
        succ[a] = (T)b;
    }
}

__global__ void k_edge_keys(const unsigned long long* __restrict__ draws, unsigned long long pairs,
                            unsigned long long n, long long* __restrict__ keys) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += stride) {
        const unsigned long long u = draws[2 * i] % n;
        const unsigned long long v = draws[2 * i + 1] % n;
        keys[i] = u == v ? -1ll : (long long)((u < v ? u : v) * n + (u < v ? v : u));
    }
}

__global__ void k_edges_from_keys(const long long* __restrict__ keys, unsigned long long m, unsigned long long n,
                                  long long* __restrict__ edges) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        const unsigned long long k = (unsigned long long)keys[i];
        edges[2 * i] = (long long)(k / n);
        edges[2 * i + 1] = (long long)(k % n);
    }
}

__global__ void k_gather_i64(const long long* __restrict__ src, const long long* __restrict__ idx,
                             unsigned long long k, long long* __restrict__ out) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride)
        out[i] = src[idx[i]];
}

}  // namespace sg

using namespace sg;

// rs_rank_even's splitters (listrank.py:431-436): the node at chain position
// k * step for k < p, i.e. the node whose rank is n - 1 - k * step.  One
// streaming pass over the ranks, p scattered 8-B writes.
template <class R>
__global__ void k_even_nodes(const R* __restrict__ rank, unsigned long long n, unsigned long long step,
                             unsigned long long p, long long* __restrict__ out) {
    const unsigned long long st = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
        const unsigned long long pos = (n - 1) - (unsigned long long)(long long)rank[i];
        if (pos % step == 0 && pos / step < p) out[pos / step] = (long long)i;
    }
}

extern "C" {

int sg_kiss_device(const uint64_t* states, uint64_t chunks, uint64_t chunk_len, uint64_t n, uint64_t* out,
                   void* stream) {
    if (chunks == 0 || n == 0) return SG_OK;
    if (chunk_len == 0 || (chunks - 1) * chunk_len >= n + chunk_len) return SG_ERR_VALUE;
    const uint32_t g = (uint32_t)((chunks + 127) / 128);
    k_kiss<<<g, 128, 0, (cudaStream_t)stream>>>((const unsigned long long*)states, chunks, chunk_len, n,
                                                (unsigned long long*)out);
    SG_LAUNCH_CHECK();
    return SG_OK;
}

int sg_list_from_order(const int64_t* perm, uint64_t n, void* succ, int succ_dtype, void* stream) {
    if (n == 0) return SG_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t g = grid_for(n, 256, 1, sm_count() * 8);
    const long long* p = (const long long*)perm;
    switch (succ_dtype) {
        case SG_U32: k_list_from_order<uint32_t><<<g, 256, 0, s>>>(p, n, (uint32_t*)succ); break;
        case SG_I32: k_list_from_order<int32_t><<<g, 256, 0, s>>>(p, n, (int32_t*)succ); break;
        case SG_I64: k_list_from_order<long long><<<g, 256, 0, s>>>(p, n, (long long*)succ); break;
        default: return SG_ERR_VALUE;
    }
    SG_LAUNCH_CHECK();
    return SG_OK;
}

int sg_edge_keys(const uint64_t* draws, uint64_t pairs, uint64_t n, int64_t* keys, void* stream) {
    if (pairs == 0) return SG_OK;
    if (n == 0) return SG_ERR_VALUE;
    k_edge_keys<<<grid_for(pairs, 256, 1, sm_count() * 8), 256, 0, (cudaStream_t)stream>>>(
        (const unsigned long long*)draws, pairs, n, (long long*)keys);
    SG_LAUNCH_CHECK();
    return SG_OK;
}

int sg_edges_from_keys(const int64_t* keys, uint64_t m, uint64_t n, int64_t* edges, void* stream) {
    if (m == 0) return SG_OK;
    if (n == 0) return SG_ERR_VALUE;
    k_edges_from_keys<<<grid_for(m, 256, 1, sm_count() * 8), 256, 0, (cudaStream_t)stream>>>(
        (const long long*)keys, m, n, (long long*)edges);
    SG_LAUNCH_CHECK();
    return SG_OK;
}

size_t sg_splitter_meta_workspace_bytes(uint32_t r) {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)r);
    return tmp + 4 * ((size_t)r * 4 + 256) + 256;
}

int sg_splitter_meta(const void* rank, int rank_dtype, uint64_t n, const int64_t* spl, uint32_t r, int64_t* out,
                     void* ws, size_t ws_bytes, void* stream) {
    if (r == 0) return SG_OK;
    if (n == 0 || n > 0xFFFFFFFFull) return SG_ERR_VALUE;
    cudaStream_t s = (cudaStream_t)stream;
    int bits = 1;
    while (bits < 32 && (1ull << bits) < n) ++bits;
    const bool block = r <= SPL_BLOCK_MAX && getenv("SG_SPL_DEVICE_SORT") == nullptr;
    Carver c(ws, ws_bytes);
    uint32_t* k0 = c.take<uint32_t>(r);
    uint32_t* k1 = c.take<uint32_t>(r);
    uint32_t* v0 = c.take<uint32_t>(r);
    uint32_t* v1 = c.take<uint32_t>(r);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, (int)r);
    void* t = c.take<unsigned char>(tmp);
    if (!c.ok) return SG_ERR_WORKSPACE;
    const uint32_t g = (r + 255) / 256;
    switch (rank_dtype) {
        case SG_U32: k_spl_keys<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)rank, (const long long*)spl, r, n, k0, v0); break;
        case SG_I32: k_spl_keys<int32_t><<<g, 256, 0, s>>>((const int32_t*)rank, (const long long*)spl, r, n, k0, v0); break;
        case SG_I64: k_spl_keys<int64_t><<<g, 256, 0, s>>>((const int64_t*)rank, (const long long*)spl, r, n, k0, v0); break;
        default: return SG_ERR_VALUE;
    }
    SG_LAUNCH_CHECK();
    if (block) return launch_spl_block(k0, r, n, bits, out, s);
    SG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, v0, v1, (int)r, 0, bits, s));
    k_spl_meta<<<g, 256, 0, s>>>(k1, v1, r, n, (long long*)out);
    SG_LAUNCH_CHECK();
    return SG_OK;
}

int sg_even_splitters(const void* rank, int rank_dtype, uint64_t n, uint64_t p, int64_t* out, void* stream) {
    if (p == 0) return SG_OK;
    if (n == 0 || n % p != 0) return SG_ERR_VALUE;
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t g = grid_for(n, 256, 4, sm_count() * 8);
    const unsigned long long step = n / p;
    switch (rank_dtype) {
        case SG_U32: k_even_nodes<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)rank, n, step, p, (long long*)out); break;
        case SG_I32: k_even_nodes<int32_t><<<g, 256, 0, s>>>((const int32_t*)rank, n, step, p, (long long*)out); break;
        case SG_I64: k_even_nodes<int64_t><<<g, 256, 0, s>>>((const int64_t*)rank, n, step, p, (long long*)out); break;
        default: return SG_ERR_VALUE;
    }
    SG_LAUNCH_CHECK();
    return SG_OK;
}

int sg_gather_i64(const int64_t* src, const int64_t* idx, uint64_t k, int64_t* out, void* stream) {
    if (k == 0) return SG_OK;
    k_gather_i64<<<grid_for(k, 256, 1, sm_count() * 8), 256, 0, (cudaStream_t)stream>>>(
        (const long long*)src, (const long long*)idx, k, (long long*)out);
    SG_LAUNCH_CHECK();
    return SG_OK;
}

}  // extern "C"
