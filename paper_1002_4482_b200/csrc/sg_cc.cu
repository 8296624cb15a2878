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
#include <string.h>

#include "sg_internal.cuh"

namespace sg {

constexpr int HOOK_THREADS = 256;
constexpr int COMP_THREADS = 256;

// ---------------------------------------------------------------------------
// edge views: pair i -> (u, v) widened so that negative / >= n endpoints fail
// the range check

struct EdgesU32 {
    const uint2* e;
    __device__ __forceinline__ void load(unsigned long long i, unsigned long long& u, unsigned long long& v) const {
        const uint2 x = __ldcs(e + i);
        u = x.x;
        v = x.y;
    }
};
struct EdgesI32 {
    const int2* e;
    __device__ __forceinline__ void load(unsigned long long i, unsigned long long& u, unsigned long long& v) const {
        const int2 x = __ldcs(e + i);
        u = (unsigned long long)(long long)x.x;
        v = (unsigned long long)(long long)x.y;
    }
};
struct EdgesI64 {
    const longlong2* e;
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
__device__ __forceinline__ uint32_t find_from(uint32_t* D, uint32_t x, uint32_t p) {
    while (p != x) {
        const uint32_t gp = __ldcg(D + p);
        if (gp == p) return p;
        __stcg(D + x, gp);
        x = gp;
        p = __ldcg(D + x);
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
        ru = find_from(D, old, __ldcg(D + old));
        rv = lo;
    }
    return false;
}

template <class E, bool kValidate>
__global__ void __launch_bounds__(HOOK_THREADS) k_cc_hook_uf(E edges, unsigned long long m, unsigned long long row0,
                                                             unsigned long long n, uint32_t* D,
                                                             unsigned long long* flags) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    bool any = false;
    unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    // two edges per iteration: four independent parent loads in flight
    for (; i + stride < m; i += 2 * stride) {
        unsigned long long u0, v0, u1, v1;
        edges.load(i, u0, v0);
        edges.load(i + stride, u1, v1);
        bool ok0 = true, ok1 = true;
        if (kValidate) {
            ok0 = edge_ok(u0, v0, n, row0 + i, flags);
            ok1 = edge_ok(u1, v1, n, row0 + i + stride, flags);
        }
        const uint32_t pu0 = ok0 ? __ldcg(D + u0) : 0, pv0 = ok0 ? __ldcg(D + v0) : 0;
        const uint32_t pu1 = ok1 ? __ldcg(D + u1) : 0, pv1 = ok1 ? __ldcg(D + v1) : 0;
        if (ok0 && pu0 != pv0) any |= unite(D, (uint32_t)u0, pu0, (uint32_t)v0, pv0);
        if (ok1 && pu1 != pv1) any |= unite(D, (uint32_t)u1, pu1, (uint32_t)v1, pv1);
    }
    if (i < m) {
        unsigned long long u, v;
        edges.load(i, u, v);
        if (!kValidate || edge_ok(u, v, n, row0 + i, flags)) {
            const uint32_t pu = __ldcg(D + u), pv = __ldcg(D + v);
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
                                                             unsigned long long* flags) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    bool any = false;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        unsigned long long u, v;
        edges.load(i, u, v);
        if (kValidate && !edge_ok(u, v, n, row0 + i, flags)) continue;
        const uint32_t du = __ldcg(D + u), dv = __ldcg(D + v);
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
        uint32_t r = __ldcg(D + i);
        if (r == (uint32_t)i) {
            ++nroots;
        } else {
            for (;;) {
                const uint32_t p = __ldcg(D + r);
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

template <class OutT>
__global__ void __launch_bounds__(COMP_THREADS) k_cc_labels(const uint32_t* __restrict__ D, unsigned long long n,
                                                            OutT* __restrict__ out) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (OutT)D[i];
}

// ---------------------------------------------------------------------------
// host side

static uint32_t hook_grid(unsigned long long m) { return grid_for(m, HOOK_THREADS, 2, kSMs * 8); }
static uint32_t vtx_grid(unsigned long long n) { return grid_for(n, COMP_THREADS, 1, kSMs * 8); }

template <class E>
static int launch_hook(E view, unsigned long long m, unsigned long long row0, unsigned long long n, uint32_t* D,
                       int variant, bool validate, unsigned long long* flags, cudaStream_t s) {
    if (m == 0) return SG_OK;
    const uint32_t g = hook_grid(m);
    if (variant == SG_CC_UF) {
        if (validate)
            k_cc_hook_uf<E, true><<<g, HOOK_THREADS, 0, s>>>(view, m, row0, n, D, flags);
        else
            k_cc_hook_uf<E, false><<<g, HOOK_THREADS, 0, s>>>(view, m, row0, n, D, flags);
    } else {
        if (validate)
            k_cc_hook_sv<E, true><<<g, HOOK_THREADS, 0, s>>>(view, m, row0, n, D, flags);
        else
            k_cc_hook_sv<E, false><<<g, HOOK_THREADS, 0, s>>>(view, m, row0, n, D, flags);
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

static int compress_dispatch(uint32_t* D, unsigned long long lo, unsigned long long hi, unsigned long long* roots,
                             void* out, int odt, cudaStream_t s) {
    if (hi <= lo) return SG_OK;
    const uint32_t g = vtx_grid(hi - lo);
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

size_t sg_cc_workspace_bytes(uint64_t n, uint64_t m) {
    (void)m;
    Carver c(nullptr, 0);
    c.take<unsigned long long>(8);
    c.take<uint32_t>(n);
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
    Carver c(ws, ws_bytes);
    unsigned long long* flags = c.take<unsigned long long>(8);  // [0..3] flags, [4] roots
    uint32_t* Dws = c.take<uint32_t>(n);
    if (!c.ok) return SG_ERR_WORKSPACE;
    // u32/i32 labels: run in place in the output buffer
    uint32_t* D = (label_dtype == SG_I64) ? Dws : (uint32_t*)labels;
    unsigned long long* roots = flags + 4;

    Recorder rec(st, s);
    SG_CUDA(cudaMemsetAsync(flags, 0, 8 * sizeof(unsigned long long), s));
    const uint32_t gv = vtx_grid(n);
    rec.begin(K_CC_INIT, 0, gv, COMP_THREADS, n);
    k_cc_init<<<gv, COMP_THREADS, 0, s>>>(D, n);
    rec.end();
    SG_LAUNCH_CHECK();
    if (st) {
        st->roots_per_round[0] = n;
        st->n_roots = 1;
        st->vertex_sweeps = 1;
    }
    int rc;
    if (variant == SG_CC_UF) {
        rec.begin(K_CC_HOOK_UF, 1, hook_grid(m), HOOK_THREADS, m);
        rc = hook_dispatch(edges, edge_dtype, m, 0, n, D, SG_CC_UF, true, flags, s);
        rec.end();
        if (rc != SG_OK) return rc;
        rec.begin(K_CC_COMPRESS, 1, gv, COMP_THREADS, n);
        rc = compress_dispatch(D, 0, n, roots, labels, label_dtype, s);
        rec.end();
        if (rc != SG_OK) return rc;
        SG_CUDA(rec.finish());
        CcHostFlags h;
        rc = read_flags(flags, h, s);
        if (rc != SG_OK) return rc;
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
        rc = hook_dispatch(edges, edge_dtype, m, 0, n, D, SG_CC_SV, r == 1, flags, s);
        rec.end();
        if (rc != SG_OK) return rc;
        rec.begin(K_CC_COMPRESS, r, gv, COMP_THREADS, n);
        rc = compress_dispatch(D, 0, n, roots, nullptr, SG_U32, s);
        rec.end();
        if (rc != SG_OK) return rc;
        CcHostFlags h;
        rc = read_flags(flags, h, s);
        if (rc != SG_OK) return rc;
        if (r == 1) {
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
