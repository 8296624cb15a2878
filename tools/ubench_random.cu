#include <stdlib.h>
// Random-access ceilings of this B200 (development aid, not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_random tools/ubench_random.cu
// Each test touches a 2 GiB array at hashed addresses; prints accesses/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// independent random 8-B reads, U in flight per thread
template <int U>
__global__ void rd(const unsigned long long* a, uint32_t mask, int iters, unsigned long long* sink) {
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long acc = 0;
    for (int k = 0; k < iters; ++k) {
        unsigned long long v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = a[mix(t * 7919u + k * 104729u + u * 15485863u) & mask];
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 42) *sink = acc;
}

// dependent chase: next = a[cur] (a holds a random permutation-like map)
__global__ void chase(const unsigned long long* a, uint32_t mask, int iters, unsigned long long* sink) {
    uint32_t cur = mix(blockIdx.x * blockDim.x + threadIdx.x) & mask;
    for (int k = 0; k < iters; ++k) cur = (uint32_t)a[cur] & mask;
    if (cur == 0xFFFFFFFF) *sink = cur;
}

// dependent chase through L2 only (ld.global.cg) / without L1 allocation
__global__ void chase_cg(const unsigned long long* a, uint32_t mask, int iters, unsigned long long* sink) {
    uint32_t cur = mix(blockIdx.x * blockDim.x + threadIdx.x) & mask;
    for (int k = 0; k < iters; ++k) cur = (uint32_t)__ldcg(a + cur) & mask;
    if (cur == 0xFFFFFFFF) *sink = cur;
}
__global__ void chase_na(const unsigned long long* a, uint32_t mask, int iters, unsigned long long* sink) {
    uint32_t cur = mix(blockIdx.x * blockDim.x + threadIdx.x) & mask;
    for (int k = 0; k < iters; ++k) {
        unsigned long long v;
        asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(a + cur));
        cur = (uint32_t)v & mask;
    }
    if (cur == 0xFFFFFFFF) *sink = cur;
}
__global__ void chase32_cg(const uint32_t* a, uint32_t mask, int iters, unsigned long long* sink) {
    uint32_t cur = mix(blockIdx.x * blockDim.x + threadIdx.x) & mask;
    for (int k = 0; k < iters; ++k) cur = __ldcg(a + cur) & mask;
    if (cur == 0xFFFFFFFF) *sink = cur;
}
__global__ void chase32(const uint32_t* a, uint32_t mask, int iters, unsigned long long* sink) {
    uint32_t cur = mix(blockIdx.x * blockDim.x + threadIdx.x) & mask;
    for (int k = 0; k < iters; ++k) cur = a[cur] & mask;
    if (cur == 0xFFFFFFFF) *sink = cur;
}

// chase + write previous node's word (the in-place walk pattern)
__global__ void chase_wr(unsigned long long* a, uint32_t mask, int iters, unsigned long long* sink) {
    uint32_t cur = mix(blockIdx.x * blockDim.x + threadIdx.x) & mask, prev = cur;
    for (int k = 0; k < iters; ++k) {
        uint32_t nx = (uint32_t)a[cur] & mask;
        if (k) a[prev] = ((unsigned long long)k << 32) | (a[prev] & 0xFFFFFFFFull) ;
        prev = cur;
        cur = nx;
    }
    if (cur == 0xFFFFFFFF) *sink = cur;
}

// chase + write to a separate array (the two-array walk pattern)
__global__ void chase_wr2(const unsigned long long* a, unsigned long long* w, uint32_t mask, int iters,
                          unsigned long long* sink) {
    uint32_t cur = mix(blockIdx.x * blockDim.x + threadIdx.x) & mask;
    for (int k = 0; k < iters; ++k) {
        w[cur] = k;
        cur = (uint32_t)a[cur] & mask;
    }
    if (cur == 0xFFFFFFFF) *sink = cur;
}

__global__ void wr(unsigned long long* a, uint32_t mask, int iters) {
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int k = 0; k < iters; ++k) a[mix(t * 7919u + k * 104729u) & mask] = k;
}

__global__ void init32(uint32_t* a, uint32_t mask) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= mask; i += gridDim.x * blockDim.x)
        a[i] = mix(i * 2654435761u + 7) & mask;
}

__global__ void init(unsigned long long* a, uint32_t mask) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= mask; i += gridDim.x * blockDim.x)
        a[i] = mix(i * 2654435761u + 1) & mask;
}

int main() {
    if (const char* f = getenv("UB_FETCH")) {  // cudaLimitMaxL2FetchGranularity experiment
        size_t before = 0, after = 0;
        cudaDeviceGetLimit(&before, cudaLimitMaxL2FetchGranularity);
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(f));
        cudaDeviceGetLimit(&after, cudaLimitMaxL2FetchGranularity);
        printf("L2 fetch granularity %zu -> %zu\n", before, after);
    }
    const uint32_t n = 1u << 28;  // 2 GiB of u64
    const uint32_t mask = n - 1;
    unsigned long long *a, *w, *sink;
    cudaMalloc(&a, (size_t)n * 8);
    cudaMalloc(&w, (size_t)n * 8);
    cudaMalloc(&sink, 8);
    init<<<148 * 8, 256>>>(a, mask);
    init32<<<148 * 8, 256>>>((uint32_t*)w, mask);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch, double accesses) {
        launch();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-28s %8.3f ms  %7.2f G acc/s  (%6.0f GB/s at 32 B, %6.0f GB/s at 64 B)\n", name, ms,
               accesses / ms / 1e6, accesses * 32 / ms / 1e6, accesses * 64 / ms / 1e6);
    };
    const int grid = 148 * 8, blk = 256, T = grid * blk;
    const int it = 64;
    run("read  MLP1", [&] { rd<1><<<grid, blk>>>(a, mask, it * 4, sink); }, (double)T * it * 4);
    run("read  MLP4", [&] { rd<4><<<grid, blk>>>(a, mask, it, sink); }, (double)T * it * 4);
    run("read  MLP8", [&] { rd<8><<<grid, blk>>>(a, mask, it / 2, sink); }, (double)T * it * 4);
    run("chase (dependent)", [&] { chase<<<grid, blk>>>(a, mask, it * 2, sink); }, (double)T * it * 2);
    run("chase ld.cg", [&] { chase_cg<<<grid, blk>>>(a, mask, it * 2, sink); }, (double)T * it * 2);
    run("chase ld.L1::no_allocate", [&] { chase_na<<<grid, blk>>>(a, mask, it * 2, sink); }, (double)T * it * 2);
    run("chase u32 (1 GiB)", [&] { chase32<<<grid, blk>>>((const uint32_t*)w, mask, it * 2, sink); }, (double)T * it * 2);
    run("chase u32 ld.cg (1 GiB)", [&] { chase32_cg<<<grid, blk>>>((const uint32_t*)w, mask, it * 2, sink); }, (double)T * it * 2);
    run("chase + write same word", [&] { chase_wr<<<grid, blk>>>(a, mask, it * 2, sink); }, (double)T * it * 2);
    run("chase + write other array", [&] { chase_wr2<<<grid, blk>>>(a, w, mask, it * 2, sink); }, (double)T * it * 2);
    run("write random 8B", [&] { wr<<<grid, blk>>>(w, mask, it * 4); }, (double)T * it * 4);
    cudaDeviceSynchronize();
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
