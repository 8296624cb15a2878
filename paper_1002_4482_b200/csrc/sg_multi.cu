// sg_multi.cu -- edge-sharded connected components over G GPUs driven by one
// host thread (the C ABI SURVEY §8(b) asks for: sg_cc_multi).
//
// Same rounds as the one-process-per-GPU path (dist.py, reference
// concomp.py:225-240): every device hooks its shard of the stored edge list
// into its replica of the parent array D (split by vertex window in round 1,
// rows validated against their global row, re-hooked from the split copy
// afterwards), the replicas merge with an NCCL min all-reduce (hooks only
// lower parents, so the element-wise minimum is a valid forest), the word at
// index n carries "nothing changed" so convergence rides the same
// collective, and a sharded shortcut (device g chases roots for its slice) +
// an in-place all-gather restores the replicas.  Labels land on every device.
//
// NCCL is the process's own (torch loads libnccl.so.2; the symbols are
// resolved with dlopen at first use, so libsg does not link a second copy).
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "sg_internal.cuh"

namespace sg {
namespace {

struct Nccl {
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*group_start)();
    ncclResult_t (*group_end)();
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*);
    ncclResult_t (*comm_destroy)(ncclComm_t);
    bool ok = false;
};

const Nccl* nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch already loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        if (!h) return;
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
        n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
        n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(h, "ncclGroupStart"));
        n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(h, "ncclGroupEnd"));
        n.comm_init_all = reinterpret_cast<decltype(n.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        n.ok = n.all_reduce && n.all_gather && n.group_start && n.group_end && n.comm_init_all && n.comm_destroy;
    });
    return n.ok ? &n : nullptr;
}

#define SG_NCCL(x)                               \
    do {                                         \
        if ((x) != ncclSuccess) return SG_ERR_CUDA; \
    } while (0)

constexpr unsigned long long kNoRow = 1ull << 62;

// round 1: this device's first bad rows (flags hold ~row, 0 = none) -> min-reducible rows
__global__ void k_multi_bad_rows(const unsigned long long* flags, long long* bad) {
    if (threadIdx.x < 2) {
        const unsigned long long f = flags[1 + threadIdx.x];
        bad[threadIdx.x] = f ? (long long)~f : (long long)kNoRow;
    }
}

// the convergence word: D[n] = 1 if this device's sweep changed nothing
__global__ void k_multi_flag(const unsigned long long* flags, uint32_t* D, unsigned long long n, int force_quiet) {
    if (threadIdx.x == 0) D[n] = (force_quiet || flags[0] == 0) ? 1u : 0u;
}

struct Dev {
    uint32_t* D = nullptr;
    unsigned long long* flags = nullptr;  // [0] changed, [1] ~first out-of-range row, [2] ~first self-loop row
    long long* bad = nullptr;             // [2] first bad rows, min-reduced
    unsigned long long* roots = nullptr;  // [1]
    void* part = nullptr;
    size_t part_bytes = 0;
};

bool carve_multi(Carver& c, uint64_t n, uint64_t m, int G, Dev& d) {
    const unsigned long long S = (n + 1 + G - 1) / G;
    d.D = c.take<uint32_t>(S * G);
    d.flags = c.take<unsigned long long>(8);
    d.bad = c.take<long long>(2);
    d.roots = c.take<unsigned long long>(1);
    d.part_bytes = sg_cc_hook_workspace_bytes(n, m);
    d.part = c.take<unsigned char>(d.part_bytes);
    return c.ok;
}

}  // namespace
}  // namespace sg

using namespace sg;

extern "C" {

size_t sg_cc_multi_workspace_bytes(uint64_t n, uint64_t m_shard, int G) {
    if (G < 1) return 0;
    Carver c(nullptr, 0);
    Dev d;
    carve_multi(c, n, m_shard, G, d);
    return c.off + 256;
}

int sg_nccl_comms_init(int G, const int* devs, void** comms) {
    const Nccl* nc = nccl();
    if (!nc) return SG_ERR_CAPABILITY;
    if (G < 1 || !devs || !comms) return SG_ERR_VALUE;
    std::vector<ncclComm_t> c(G);
    SG_NCCL(nc->comm_init_all(c.data(), G, devs));
    for (int g = 0; g < G; ++g) comms[g] = c[g];
    return SG_OK;
}

int sg_nccl_comms_destroy(int G, void** comms) {
    const Nccl* nc = nccl();
    if (!nc) return SG_ERR_CAPABILITY;
    for (int g = 0; g < G; ++g)
        if (comms[g]) SG_NCCL(nc->comm_destroy((ncclComm_t)comms[g]));
    return SG_OK;
}

int sg_cc_multi(int G, const int* devs, const void* const* edges, int edge_dtype, const uint64_t* m_shard, uint64_t n,
                void* const* labels, int label_dtype, int variant, int round_bound, void* const* ws,
                const size_t* ws_bytes, void* const* comms, void* const* streams, sg_stats* st, sg_violation* viol) {
    if (G < 1 || !devs || !edges || !m_shard || !labels || !ws || !ws_bytes || !comms || !streams)
        return SG_ERR_VALUE;
    if (n == 0) return SG_ERR_INVALID_GRAPH;
    if (n >= 0x7FFFFFFFull) return SG_ERR_CAPABILITY;
    if (variant != SG_CC_UF && variant != SG_CC_SV) return SG_ERR_VALUE;
    if (label_dtype != SG_U32 && label_dtype != SG_I32 && label_dtype != SG_I64) return SG_ERR_VALUE;
    const Nccl* nc = nccl();
    if (!nc) return SG_ERR_CAPABILITY;
    ::sg::apply_tuning();
    if (st) memset(st, 0, sizeof(sg_stats));
    if (viol) {
        viol->kind = SG_GRAPH_OK;
        viol->index = -1;
        viol->pad = 0;
    }
    int prev = 0;
    SG_CUDA(cudaGetDevice(&prev));
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    const unsigned long long S = (n + 1 + G - 1) / G;
    std::vector<Dev> dv(G);
    std::vector<uint64_t> row0(G, 0);
    for (int g = 0; g < G; ++g) {
        if (g) row0[g] = row0[g - 1] + m_shard[g - 1];
        Carver c(ws[g], ws_bytes[g]);
        if (!carve_multi(c, n, m_shard[g], G, dv[g])) return SG_ERR_WORKSPACE;
    }
    auto strm = [&](int g) { return (cudaStream_t)streams[g]; };
    auto comm = [&](int g) { return (ncclComm_t)comms[g]; };
    for (int g = 0; g < G; ++g) {
        SG_CUDA(cudaSetDevice(devs[g]));
        int rc = sg_cc_init(dv[g].D, S * G, strm(g));
        if (rc != SG_OK) return rc;
    }
    if (st) {
        st->roots_per_round[0] = n;
        st->n_roots = 1;
    }
    int r = 0;
    for (;;) {
        ++r;
        if (r > round_bound) return SG_ERR_RUNTIME;
        for (int g = 0; g < G; ++g) {  // local hook sweeps
            SG_CUDA(cudaSetDevice(devs[g]));
            SG_CUDA(cudaMemsetAsync(dv[g].flags, 0, 8 * sizeof(unsigned long long), strm(g)));
            const int rc = sg_cc_hook_part(edges[g], edge_dtype, m_shard[g], row0[g], n, dv[g].D, variant, r == 1,
                                           reinterpret_cast<uint64_t*>(dv[g].flags), dv[g].part, dv[g].part_bytes,
                                           r > 1, strm(g));
            if (rc != SG_OK) return rc;
        }
        if (st) st->edge_sweeps += 1;
        if (r == 1) {  // the first bad global row of any shard (core.py:196-206 order)
            SG_NCCL(nc->group_start());
            for (int g = 0; g < G; ++g) {
                SG_CUDA(cudaSetDevice(devs[g]));
                k_multi_bad_rows<<<1, 32, 0, strm(g)>>>(dv[g].flags, dv[g].bad);
                SG_NCCL(nc->all_reduce(dv[g].bad, dv[g].bad, 2, ncclInt64, ncclMin, comm(g), strm(g)));
            }
            SG_NCCL(nc->group_end());
            long long bad[2];
            SG_CUDA(cudaSetDevice(devs[0]));
            SG_CUDA(cudaMemcpyAsync(bad, dv[0].bad, sizeof(bad), cudaMemcpyDeviceToHost, strm(0)));
            SG_CUDA(cudaStreamSynchronize(strm(0)));
            if (bad[0] != (long long)kNoRow || bad[1] != (long long)kNoRow) {
                if (viol) {
                    viol->kind = bad[0] != (long long)kNoRow ? SG_GRAPH_OUT_OF_RANGE : SG_GRAPH_SELF_LOOP;
                    viol->index = bad[0] != (long long)kNoRow ? bad[0] : bad[1];
                }
                return SG_ERR_INVALID_GRAPH;
            }
        }
        // merge: element-wise min of the replicas; word n = all quiet
        // (one UF sweep unites every edge of a shard, so one device is done after round 1)
        SG_NCCL(nc->group_start());
        for (int g = 0; g < G; ++g) {
            SG_CUDA(cudaSetDevice(devs[g]));
            k_multi_flag<<<1, 32, 0, strm(g)>>>(dv[g].flags, dv[g].D, n, variant == SG_CC_UF && G == 1);
            SG_NCCL(nc->all_reduce(dv[g].D, dv[g].D, S * G, ncclUint32, ncclMin, comm(g), strm(g)));
        }
        SG_NCCL(nc->group_end());
        uint32_t quiet = 0;
        SG_CUDA(cudaSetDevice(devs[0]));
        SG_CUDA(cudaMemcpyAsync(&quiet, dv[0].D + n, sizeof(quiet), cudaMemcpyDeviceToHost, strm(0)));
        SG_CUDA(cudaStreamSynchronize(strm(0)));
        const bool converged = quiet == 1;
        if (variant == SG_CC_SV || converged) {  // sharded shortcut + all-gather
            for (int g = 0; g < G; ++g) {
                SG_CUDA(cudaSetDevice(devs[g]));
                SG_CUDA(cudaMemsetAsync(dv[g].roots, 0, sizeof(unsigned long long), strm(g)));
                const unsigned long long lo = (unsigned long long)g * S;
                const unsigned long long hi = lo + S < n ? lo + S : n;
                const int rc = sg_cc_compress(dv[g].D, lo, hi > lo ? hi : lo, reinterpret_cast<uint64_t*>(dv[g].roots),
                                              strm(g));
                if (rc != SG_OK) return rc;
            }
            SG_NCCL(nc->group_start());
            for (int g = 0; g < G; ++g) {
                SG_CUDA(cudaSetDevice(devs[g]));
                SG_NCCL(nc->all_gather(dv[g].D + (size_t)g * S, dv[g].D, S, ncclUint32, comm(g), strm(g)));
                SG_NCCL(nc->all_reduce(dv[g].roots, dv[g].roots, 1, ncclUint64, ncclSum, comm(g), strm(g)));
            }
            SG_NCCL(nc->group_end());
            if (st) {
                unsigned long long roots = 0;
                SG_CUDA(cudaSetDevice(devs[0]));
                SG_CUDA(cudaMemcpyAsync(&roots, dv[0].roots, sizeof(roots), cudaMemcpyDeviceToHost, strm(0)));
                SG_CUDA(cudaStreamSynchronize(strm(0)));
                st->vertex_sweeps += 1;
                if (st->n_roots < SG_MAX_ROUNDS) st->roots_per_round[st->n_roots++] = roots;
            }
        }
        if (st) st->rounds = (uint32_t)r;
        if (converged) break;
    }
    for (int g = 0; g < G; ++g) {  // labels on every device
        SG_CUDA(cudaSetDevice(devs[g]));
        const int rc = sg_cc_labels(dv[g].D, n, labels[g], label_dtype, strm(g));
        if (rc != SG_OK) return rc;
    }
    for (int g = 0; g < G; ++g) {
        SG_CUDA(cudaSetDevice(devs[g]));
        SG_CUDA(cudaStreamSynchronize(strm(g)));
    }
    return SG_OK;
}

}  // extern "C"
