// Random 4-B stores into distributed shared memory (thread-block clusters):
// could a cluster hold a whole output window of ranks and scatter into it?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_dsmem tools/ubench_dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

template <int CS>
__global__ void dsmem_scatter(int iters, uint32_t words_per_cta, unsigned long long* sink) {
    extern __shared__ uint32_t win[];
    cg::cluster_group cl = cg::this_cluster();
    for (uint32_t i = threadIdx.x; i < words_per_cta; i += blockDim.x) win[i] = 0;
    cl.sync();
    uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
    for (int k = 0; k < iters; ++k) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        const uint32_t tgt = x % CS;
        const uint32_t off = (x >> 8) % words_per_cta;
        uint32_t* remote = cl.map_shared_rank(win, tgt);
        remote[off] = x;
    }
    cl.sync();
    unsigned long long acc = 0;
    for (uint32_t i = threadIdx.x; i < words_per_cta; i += blockDim.x) acc += win[i];
    if (acc == 42) *sink = acc;
}

__global__ void smem_scatter(int iters, uint32_t words_per_cta, unsigned long long* sink) {
    extern __shared__ uint32_t win[];
    for (uint32_t i = threadIdx.x; i < words_per_cta; i += blockDim.x) win[i] = 0;
    __syncthreads();
    uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
    for (int k = 0; k < iters; ++k) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        win[(x >> 8) % words_per_cta] = x;
    }
    __syncthreads();
    unsigned long long acc = 0;
    for (uint32_t i = threadIdx.x; i < words_per_cta; i += blockDim.x) acc += win[i];
    if (acc == 42) *sink = acc;
}

template <int CS>
void run(int blocks, int threads, int iters, uint32_t bytes, unsigned long long* sink) {
    auto k = dsmem_scatter<CS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (CS > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = bytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, k, iters, bytes / 4, sink);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, iters, bytes / 4, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double stores = (double)blocks * threads * iters;
    printf("cluster %2d  smem %6u B/CTA  active clusters %3d  %8.3f ms  %7.1f G stores/s  err %s\n", CS, bytes, ncl, ms,
           stores / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int iters = 512;
    run<16>(16 * 64, 1024, iters, 128 * 1024, sink);
    run<8>(8 * 128, 1024, iters, 128 * 1024, sink);
    run<8>(8 * 128, 1024, iters, 200 * 1024, sink);
    run<4>(4 * 256, 1024, iters, 128 * 1024, sink);
    run<2>(2 * 512, 1024, iters, 128 * 1024, sink);
    {
        cudaFuncSetAttribute(smem_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        smem_scatter<<<148 * 8, 1024, 128 * 1024>>>(iters, 32768, sink);
        cudaEventRecord(e0);
        smem_scatter<<<148 * 8, 1024, 128 * 1024>>>(iters, 32768, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("local smem scatter: %7.1f G stores/s  err %s\n", 148.0 * 8 * 1024 * iters / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
