// sg_scan.cuh -- multi-block exclusive scan of u32 counts into u64 offsets
// (reduce / top / down), shared by the edge partition (sg_cc.cu) and the
// ranking record partition (sg_list.cu).
#pragma once

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "sg_internal.cuh"

namespace sg {

// multi-block exclusive scan of u32 counts into u64 offsets (3 launches)
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_BLOCK = SCAN_THREADS * SCAN_ITEMS;

static __global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const uint32_t* __restrict__ in, unsigned long long len,
                                                             unsigned long long* __restrict__ block_sum) {
    const unsigned long long base = (unsigned long long)blockIdx.x * SCAN_BLOCK;
    unsigned long long t = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const unsigned long long i = base + (unsigned long long)j * SCAN_THREADS + threadIdx.x;
        if (i < len) t += in[i];
    }
    typedef cub::BlockReduce<unsigned long long, SCAN_THREADS> BR;
    __shared__ typename BR::TempStorage tmp;
    const unsigned long long tot = BR(tmp).Sum(t);
    if (threadIdx.x == 0) block_sum[blockIdx.x] = tot;
}

static __global__ void __launch_bounds__(SCAN_THREADS) k_scan_top(unsigned long long* block_sum, unsigned long long nblocks,
                                                          unsigned long long* total) {
    const unsigned long long per = (nblocks + SCAN_THREADS - 1) / SCAN_THREADS;
    const unsigned long long a = threadIdx.x * per, b = min(a + per, nblocks);
    unsigned long long sum = 0;
    for (unsigned long long t = a; t < b; ++t) sum += block_sum[t];
    typedef cub::BlockScan<unsigned long long, SCAN_THREADS> BS;
    __shared__ typename BS::TempStorage tmp;
    unsigned long long pre, tot;
    BS(tmp).ExclusiveSum(sum, pre, tot);
    for (unsigned long long t = a; t < b; ++t) {
        const unsigned long long c = block_sum[t];
        block_sum[t] = pre;
        pre += c;
    }
    if (threadIdx.x == 0 && total) *total = tot;
}

// out[i] = exclusive prefix; also off_part[i / stride_part] for i % stride_part == 0
static __global__ void __launch_bounds__(SCAN_THREADS) k_scan_down(const uint32_t* __restrict__ in, unsigned long long len,
                                                           const unsigned long long* __restrict__ block_pre,
                                                           unsigned long long* __restrict__ out,
                                                           unsigned long long stride_part,
                                                           unsigned long long* __restrict__ off_part) {
    const unsigned long long base = (unsigned long long)blockIdx.x * SCAN_BLOCK;
    // blocked arrangement: thread t owns SCAN_ITEMS consecutive entries
    uint32_t v[SCAN_ITEMS];
    unsigned long long t = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const unsigned long long i = base + (unsigned long long)threadIdx.x * SCAN_ITEMS + j;
        v[j] = i < len ? in[i] : 0u;
        t += v[j];
    }
    typedef cub::BlockScan<unsigned long long, SCAN_THREADS> BS;
    __shared__ typename BS::TempStorage tmp;
    unsigned long long pre;
    BS(tmp).ExclusiveSum(t, pre);
    pre += block_pre[blockIdx.x];
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const unsigned long long i = base + (unsigned long long)threadIdx.x * SCAN_ITEMS + j;
        if (i < len) {
            out[i] = pre;
            if (off_part && i % stride_part == 0) off_part[i / stride_part] = pre;
        }
        pre += v[j];
    }
}


// launch the three scan kernels over in[0, len); bsum needs len / SCAN_BLOCK + 2
// entries; off_part[i / stride_part] receives the offset of every stride_part-th
// entry and off_part[parts] the total.
static inline void launch_scan(const uint32_t* in, unsigned long long len, unsigned long long* bsum,
                               unsigned long long* out, unsigned long long stride_part,
                               unsigned long long* off_part, int parts, cudaStream_t s) {
    const unsigned long long nb = (len + SCAN_BLOCK - 1) / SCAN_BLOCK;
    k_scan_reduce<<<(uint32_t)(nb ? nb : 1), SCAN_THREADS, 0, s>>>(in, len, bsum);
    k_scan_top<<<1, SCAN_THREADS, 0, s>>>(bsum, nb ? nb : 1, off_part + parts);
    k_scan_down<<<(uint32_t)(nb ? nb : 1), SCAN_THREADS, 0, s>>>(in, len, bsum, out, stride_part, off_part);
}

}  // namespace sg
