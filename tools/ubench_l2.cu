// L2-resident random-access ceilings of this B200 (development aid, not
// product code): the IS_1 gathers of rs5_refine (random 4-B loads over a
// 32 MiB table) and the parent gathers / atomics of cc_hook (random 4-B
// loads and atomicMin over a 32 MiB window of D).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_ubench_l2 tools/ubench_l2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// U independent random 4-B loads per thread per iteration (default caching)
template <int U>
__global__ void gather(const uint32_t* a, uint32_t mask, int iters, unsigned long long* sink) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int k = 0; k < iters; ++k) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldg(a + (mix(t * 7919u + k * 104729u + u * 15485863u) & mask));
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 42) *sink = acc;
}

// the same through ld.global.cg (L2 only, no L1 allocation)
template <int U>
__global__ void gather_cg(const uint32_t* a, uint32_t mask, int iters, unsigned long long* sink) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int k = 0; k < iters; ++k) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcg(a + (mix(t * 7919u + k * 104729u + u * 15485863u) & mask));
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 42) *sink = acc;
}

// half-warp locality: lanes l and l^1 read the same 32-B sector
template <int U>
__global__ void gather_pair(const uint32_t* a, uint32_t mask, int iters, unsigned long long* sink) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int k = 0; k < iters; ++k) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            v[u] = __ldg(a + ((mix((t >> 1) * 7919u + k * 104729u + u * 15485863u) & mask & ~7u) | (t & 1u)));
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 42) *sink = acc;
}

// random atomicMin (returning) / red.min (no return)
template <int U>
__global__ void amin(uint32_t* a, uint32_t mask, int iters, unsigned long long* sink) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < U; ++u) acc += atomicMin(a + (mix(t * 7919u + k * 104729u + u * 15485863u) & mask), t);
    }
    if (acc == 42) *sink = acc;
}
template <int U>
__global__ void rmin(uint32_t* a, uint32_t mask, int iters) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < U; ++u) atomicMin(a + (mix(t * 7919u + k * 104729u + u * 15485863u) & mask), t);
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t maxbytes = 256ull << 20;
    uint32_t* a;
    unsigned long long* sink;
    cudaMalloc(&a, maxbytes);
    cudaMalloc(&sink, 8);
    cudaMemset(a, 0x7f, maxbytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 256, blocks = sms * 8, iters = 64;
    auto run = [&](const char* name, size_t bytes, int per, auto launch) {
        const uint32_t mask = (uint32_t)(bytes / 4 - 1);
        launch(mask);  // warm: fills L2
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch(mask);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 5;
        const double acc = (double)threads * blocks * iters * per;
        printf("%-28s table %4zu MiB  %8.3f ms  %7.1f G acc/s\n", name, bytes >> 20, ms, acc / ms / 1e6);
    };
    for (size_t mb : {8, 32, 64, 256}) {
        const size_t bytes = mb << 20;
        run("gather U8", bytes, 8, [&](uint32_t m) { gather<8><<<blocks, threads>>>(a, m, iters, sink); });
        run("gather U16", bytes, 16, [&](uint32_t m) { gather<16><<<blocks, threads>>>(a, m, iters, sink); });
        run("gather cg U8", bytes, 8, [&](uint32_t m) { gather_cg<8><<<blocks, threads>>>(a, m, iters, sink); });
        run("gather pairs U8", bytes, 8, [&](uint32_t m) { gather_pair<8><<<blocks, threads>>>(a, m, iters, sink); });
        run("atomicMin U4", bytes, 4, [&](uint32_t m) { amin<4><<<blocks, threads>>>(a, m, iters, sink); });
        run("red.min U4", bytes, 4, [&](uint32_t m) { rmin<4><<<blocks, threads>>>(a, m, iters); });
    }
    const cudaError_t e = cudaGetLastError();
    printf("err: %s\n", cudaGetErrorString(e));
    return 0;
}
