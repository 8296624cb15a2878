/*
 * sg.h -- C ABI of the B200-native list-ranking / connected-components
 * library (libsg.so, built from paper_1002_4482_b200/csrc).
 *
 * The reference (simtgraph, a pure-Python package) has no native FFI: its
 * drop-in boundary is the Python API (wyllie_rank / rs_rank / rs_rank_even /
 * sv_components, /root/reference/pkg/src/simtgraph/__init__.py:42-43).  The
 * functions below are the native layer that Python API binds through ctypes
 * (paper_1002_4482_b200/_native.py); each cites the reference interface it
 * replaces.  INTEGRATION.md shows the binding a maintainer of the reference
 * would add.
 *
 * Conventions
 *   - plain C: device pointers are `void*`/typed pointers, sizes are uint64_t,
 *     a CUDA stream is passed as `void*` (cudaStream_t), NULL = legacy stream;
 *   - every entry returns an sg_status; sg_strerror() names it;
 *   - the caller owns every buffer.  Scratch comes from a caller-provided
 *     workspace whose size is given by the matching *_workspace_bytes();
 *     nothing allocated by the library outlives a call;
 *   - compute entry points are synchronous with respect to the host: they
 *     enqueue on `stream`, then wait for it so the status (validity of the
 *     input, capability overflow) can be returned.
 *   - node / vertex ids are 32-bit on the device: n must be < 2^32 - 1.
 */
#ifndef SG_H
#define SG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The Python layer maps them onto the reference's exception
 * types (core.py:16-29): INVALID_LIST -> InvalidListError, INVALID_GRAPH ->
 * InvalidGraphError, CAPABILITY -> CapabilityError, VALUE -> ValueError,
 * RUNTIME -> RuntimeError (concomp.py:227-229, listrank.py:297-298). */
enum sg_status {
    SG_OK = 0,
    SG_ERR_INVALID_LIST = 1,
    SG_ERR_INVALID_GRAPH = 2,
    SG_ERR_CAPABILITY = 3,
    SG_ERR_VALUE = 4,
    SG_ERR_RUNTIME = 5,
    SG_ERR_CUDA = 6,
    SG_ERR_WORKSPACE = 7
};

/* Element types accepted for successor arrays, edge arrays and outputs. */
enum sg_dtype { SG_U32 = 0, SG_I32 = 1, SG_I64 = 2 };

/* wyllie variants (listrank.py:75-155) */
enum sg_wyllie_variant { SG_WY_MULTI_KERNEL = 0, SG_WY_SINGLE_BLOCK = 1 };

/* connected-components variants (concomp.py:208-246 is the reference) */
enum sg_cc_variant {
    SG_CC_UF = 0,   /* one hook sweep: CAS root hooking + path halving   */
    SG_CC_SV = 1    /* synchronous min-hook rounds + root shortcut sweep */
};

/* List violation kinds, in the reference's report order (core.py:148-167). */
enum sg_list_violation {
    SG_LIST_OK = 0,
    SG_LIST_OUT_OF_RANGE = 1,
    SG_LIST_NO_TAIL = 2,
    SG_LIST_MULTIPLE_SELF_LOOPS = 3,
    SG_LIST_UNREACHABLE = 4
};

/* Graph violation kinds (core.py:196-206). */
enum sg_graph_violation {
    SG_GRAPH_OK = 0,
    SG_GRAPH_OUT_OF_RANGE = 1,
    SG_GRAPH_SELF_LOOP = 2
};

#define SG_MAX_LAUNCHES 192
#define SG_MAX_ROUNDS 96
#define SG_MAX_LEVELS 8

/* One kernel launch (mirrors core.LaunchRecord, core.py:305-310). */
typedef struct sg_launch {
    int32_t kernel;     /* id, sg_kernel_name() gives the name            */
    int32_t round;      /* algorithm round / ruling-set level             */
    uint32_t blocks;    /* grid size                                      */
    uint32_t threads;   /* block size                                     */
    uint64_t items;     /* work items the launch covers (nodes / edges)   */
    float ms;           /* CUDA-event duration on the launching stream,
                           filled by sg_stats_resolve()                   */
    uint32_t pad;       /* library-private: event indices                 */
} sg_launch;

/* Execution statistics (the fields ExecStats needs, core.py:317-405). */
typedef struct sg_stats {
    uint32_t n_launches;
    uint32_t rounds;          /* jump rounds / CC rounds                  */
    uint32_t levels;          /* ruling-set recursion depth               */
    uint32_t fallback;        /* 1: ruling set fell back to pointer jumping */
    uint64_t edge_sweeps;     /* CC: passes over the stored edge list      */
    uint64_t vertex_sweeps;   /* CC: passes over the vertex array          */
    uint64_t level_size[SG_MAX_LEVELS];   /* nodes per ruling-set level    */
    uint32_t n_roots;         /* entries in roots_per_round               */
    uint32_t list_path;       /* rs: 0 ruling-set walk, 1 tile contraction */
    uint64_t roots_per_round[SG_MAX_ROUNDS];
    float total_ms;           /* event time of the whole device pipeline
                                 (filled by sg_stats_resolve())           */
    uint32_t pad2;            /* library-private: event-set ticket        */
    sg_launch launch[SG_MAX_LAUNCHES];
} sg_stats;

/* Detail of an input violation found on the device (index = first
 * offending element / row in the reference's report order, -1 if none). */
typedef struct sg_violation {
    int32_t kind;
    int32_t pad;
    int64_t index;
} sg_violation;

/* ---- boundary copies (host int64 <-> device 32-bit ids) ------------------
 * The reference's arrays are int64 (core.py:77-110); the kernels take 32-bit
 * ids.  These copies narrow / widen on host threads, pipelined against the
 * DMA through a pinned staging ring (sg_xfer.cu).  Both are synchronous for
 * the host arrays (they may be reused on return) and ordered on `stream`.
 *   sg_h2d_narrow_i64: *in_range = 0 if a value lies outside [0, bound)
 *     (the device copy is then incomplete; copy int64 instead so the device
 *     reports the exact error).
 *   sg_d2h_widen_u32: waits for the stream's earlier work on `dev`. */
int sg_h2d_narrow_i64(const int64_t* host, uint64_t count, uint32_t* dev, uint64_t bound, void* stream,
                      int* in_range);
int sg_d2h_widen_u32(const uint32_t* dev, uint64_t count, int64_t* host, void* stream);
/* Host threads the two copies convert with (the process's usable CPUs: the
 * affinity mask capped by a cgroup CPU quota, at most 32; SG_XFER_THREADS
 * overrides).  Starts the pool on first use. */
int sg_xfer_threads(void);

/* ---- library ------------------------------------------------------------ */
const char* sg_strerror(int status);
const char* sg_kernel_name(int kernel_id);
int sg_version(void);
/* Re-read the SG_* experiment switches from the environment (they are
 * otherwise parsed once per process; defaults = the measured configuration).
 * Not a reference interface: tests use it to force rare paths. */
int sg_tuning_reload(void);
/* sha256 (hex, ';'-terminated) of the sources, headers and nvcc flags this
 * library was built from (paper_1002_4482_b200/build.py). */
const char* sg_source_hash(void);
/* Fill launch[k].ms and total_ms of a finished call.  Calls return without
 * reading their CUDA events (that costs ~3 us per launch of host time after
 * the pipeline's last kernel); the events of one call stay valid for the
 * next 63 calls on the device.  SG_ERR_RUNTIME: recycled (ms stay 0). */
int sg_stats_resolve(sg_stats* st);
/* last CUDA error string seen by this thread (for SG_ERR_CUDA) */
const char* sg_last_cuda_error(void);

/* ---- list ranking ------------------------------------------------------- */

/* Scratch bytes for sg_wyllie_rank / sg_rs_rank on an n-node list. */
size_t sg_wyllie_workspace_bytes(uint64_t n);
size_t sg_rs_workspace_bytes(uint64_t n);

/* Pointer jumping over packed {rank,succ} 64-bit words.
 * Replaces listrank.wyllie_rank (listrank.py:75-155): variant
 * SG_WY_MULTI_KERNEL = init + ceil(log2 n) jump launches (:95-118),
 * SG_WY_SINGLE_BLOCK = one CTA with block barriers (:120-150).
 * succ: n successors (head 0, tail self-loop; core.py:77-94), dtype
 * SG_U32/SG_I32/SG_I64.  rank: n outputs of rank_dtype.
 * Returns SG_ERR_INVALID_LIST (viol filled with the cheap device checks:
 * out-of-range / tail count; otherwise kind = UNREACHABLE, index -1 --
 * sg_list_violation_host() gives the reference's exact first violation). */
int sg_wyllie_rank(const void* succ, int succ_dtype, void* rank, int rank_dtype,
                   uint64_t n, int variant, void* ws, size_t ws_bytes,
                   void* stream, sg_stats* st, sg_violation* viol);

/* Sparse ruling-set list ranking (Helman-JaJa style, recursive).
 * Replaces listrank.rs_rank / rs_rank_even's device pipeline
 * (_rs_pipeline, listrank.py:385-408: RS1..RS5, :197-382).  The splitter
 * set the reference reports (meta["splitter_set"], :405-407) is derived
 * from the ranks by the caller; the device picks its own ruling set
 * (Fibonacci-hashed node ids, `seed` salts the hash) so the walk has
 * enough independent chains for 148 SMs.  rank may alias succ when both
 * dtypes match (reuse_succ, listrank.py:186-187). */
int sg_rs_rank(const void* succ, int succ_dtype, void* rank, int rank_dtype,
               uint64_t n, uint64_t seed, void* ws, size_t ws_bytes,
               void* stream, sg_stats* st, sg_violation* viol);

/* sg_rs_rank plus meta["splitter_set"] (see sg_splitter_meta) for the r
 * splitter nodes spl, computed on the same stream before the call's single
 * synchronisation: meta_dev (device, 3 x r int64) and, if meta_host is not
 * NULL, a copy in meta_host (host, pinned for best speed).  meta_ws holds
 * sg_splitter_meta_workspace_bytes(r) bytes. */
int sg_rs_rank_meta(const void* succ, int succ_dtype, void* rank, int rank_dtype,
                    uint64_t n, uint64_t seed, void* ws, size_t ws_bytes,
                    const int64_t* spl, uint32_t r, int64_t* meta_dev, int64_t* meta_host,
                    void* meta_ws, size_t meta_ws_bytes,
                    void* stream, sg_stats* st, sg_violation* viol);

/* rs_rank_even's perfect splitters (listrank.py:431-436): out[k] (int64,
 * device) = the node at chain position k * (n / p), i.e. whose rank is
 * n - 1 - k * (n / p), for k < p; p must divide n.  One streaming pass over
 * the ranks (replaces the reference's position array). */
int sg_even_splitters(const void* rank, int rank_dtype, uint64_t n, uint64_t p, int64_t* out, void* stream);

/* out[i] = src[idx[i]] for i < k (int64 ranks at the official splitters;
 * listrank.py:355-356 splitter_rank is the global rank of the splitter). */
int sg_gather_i64(const int64_t* src, const int64_t* idx, uint64_t k,
                  int64_t* out, void* stream);

/* meta["splitter_set"] from the device ranks (listrank.py:252-357): for the
 * r splitter nodes spl (int64, device), out (int64, device, 3 x r) receives
 * the splitter ranks, the sublist lengths (to the next splitter in list
 * order; the last to the tail) and the reduced successors (the last splitter
 * points at itself).  One radix sort of the r ranks; n < 2^32. */
size_t sg_splitter_meta_workspace_bytes(uint32_t r);
int sg_splitter_meta(const void* rank, int rank_dtype, uint64_t n, const int64_t* spl,
                     uint32_t r, int64_t* out, void* ws, size_t ws_bytes, void* stream);

/* ---- connected components ---------------------------------------------- */

size_t sg_cc_workspace_bytes(uint64_t n, uint64_t m);

/* Connected components of an undirected graph stored once per edge as
 * (m,2) pairs (core.EdgeGraph, core.py:97-110), labels canonicalised to the
 * smallest vertex of each component (core.py:240-257).
 * Replaces concomp.sv_components (concomp.py:208-246).  Validates the edge
 * list on the device (core.py:196-206).  round_bound: RuntimeError
 * (SG_ERR_RUNTIME) if the SV variant needs more rounds (concomp.py:227-229).
 * labels: n outputs of label_dtype. */
int sg_cc(const void* edges, int edge_dtype, uint64_t m, uint64_t n,
          void* labels, int label_dtype, int variant, int round_bound,
          void* ws, size_t ws_bytes, void* stream, sg_stats* st,
          sg_violation* viol);

/* Building blocks of the edge-sharded multi-GPU components (one process per
 * GPU; the Python layer merges parent arrays with an NCCL min all-reduce).
 * D is the parent array (u32, D[i] <= i).  flags (device, 4 x u32, zeroed by
 * the caller): [0] = a hook changed D, [1] = first out-of-range row (low),
 * [2] = first self-loop row (low), [3] = unused. */
int sg_cc_init(uint32_t* D, uint64_t n, void* stream);
int sg_cc_hook(const void* edges, int edge_dtype, uint64_t m, uint64_t row0,
               uint64_t n, uint32_t* D, int variant, int validate,
               uint64_t* flags, void* stream);
/* As sg_cc_hook, for large n: the block is first split by 2^23-vertex window
 * of the larger endpoint into `ws` (validating rows; reuse != 0 skips the
 * split and hooks the copy a previous call left in `ws`), then hooked window
 * by window so the parent gathers stay L2-resident. */
size_t sg_cc_hook_workspace_bytes(uint64_t n, uint64_t m);
int sg_cc_hook_part(const void* edges, int edge_dtype, uint64_t m, uint64_t row0,
                    uint64_t n, uint32_t* D, int variant, int validate, uint64_t* flags,
                    void* ws, size_t ws_bytes, int reuse, void* stream);
/* D[i] = root(i) for lo <= i < hi; adds the number of roots in [lo,hi)
 * to *roots (device u64). */
/* Sparse merge for the sharded rounds: append (i, D[i]) for every i < n with
 * D[i] != Dold[i] (count accumulates; at most cap written), and lower
 * D[idx[j]] to val[j] (atomic min) for j < k. */
int sg_cc_changes(const uint32_t* Dold, const uint32_t* D, uint64_t n, uint32_t* idx,
                  uint32_t* val, uint64_t cap, uint64_t* count, void* stream);
int sg_cc_apply_min(uint32_t* D, const uint32_t* idx, const uint32_t* val, uint64_t k,
                    void* stream);
int sg_cc_compress(uint32_t* D, uint64_t lo, uint64_t hi, uint64_t* roots,
                   void* stream);
/* out[i] = (dtype) D[i] for i < n */
int sg_cc_labels(const uint32_t* D, uint64_t n, void* out, int out_dtype,
                 void* stream);

/* ---- connected components over G GPUs, one host thread ------------------
 * Replaces the reference's sv_components over the edge-sharded layout
 * (SURVEY §8(b) sg_cc_multi; rounds as concomp.py:225-240): device g hooks
 * its shard edges[g] (m_shard[g] rows; global row = the shards before it +
 * the local row, for InvalidGraphError) into its replica of D, the replicas
 * merge with an NCCL min all-reduce per round until no device changed
 * anything, then a sharded shortcut + all-gather; labels[g] (n entries,
 * label_dtype) receive the component-minimum labels on every device.
 * comms[g]: one NCCL clique (e.g. sg_nccl_comms_init), streams[g] on
 * devs[g], ws[g]: sg_cc_multi_workspace_bytes(n, m_shard[g], G) bytes on
 * devs[g].  NCCL is the process's own libnccl.so.2, resolved at run time. */
size_t sg_cc_multi_workspace_bytes(uint64_t n, uint64_t m_shard, int G);
int sg_cc_multi(int G, const int* devs, const void* const* edges, int edge_dtype, const uint64_t* m_shard,
                uint64_t n, void* const* labels, int label_dtype, int variant, int round_bound,
                void* const* ws, const size_t* ws_bytes, void* const* comms, void* const* streams,
                sg_stats* st, sg_violation* viol);
/* ncclCommInitAll / ncclCommDestroy of the process's NCCL (comms: G opaque handles) */
int sg_nccl_comms_init(int G, const int* devs, void** comms);
int sg_nccl_comms_destroy(int G, void** comms);

/* ---- input generation (gen.py) ----------------------------------------- */

/* KISS64 draws on the host (gen.py:30-64); state[4] = {x,y,z,c} in/out. */
int sg_kiss_batch_host(uint64_t* state, uint64_t n, uint64_t* out);
/* KISS64 draws on the device: chunk k (k < chunks) starts from
 * states[4k..4k+3] (jump-ahead computed by the caller) and produces
 * out[k*chunk_len .. min((k+1)*chunk_len, n)). */
int sg_kiss_device(const uint64_t* states, uint64_t chunks, uint64_t chunk_len,
                   uint64_t n, uint64_t* out, void* stream);
/* succ[order[j]] = order[j+1], succ[order[n-1]] = order[n-1] with
 * order[0] = 0 and order[j] = 1 + perm[j-1] (gen.py:118-127). */
int sg_list_from_order(const int64_t* perm, uint64_t n, void* succ,
                       int succ_dtype, void* stream);
/* (u,v) = (draw[2i] % n, draw[2i+1] % n); key = min*n+max or -1 on a
 * self-loop draw (gen.py:203-209). */
int sg_edge_keys(const uint64_t* draws, uint64_t pairs, uint64_t n,
                 int64_t* keys, void* stream);
/* edges[i] = (key/n, key%n) as int64 pairs (gen.py:215-217). */
int sg_edges_from_keys(const int64_t* keys, uint64_t m, uint64_t n,
                       int64_t* edges, void* stream);

/* ---- host-side validation (error path) ---------------------------------- */

/* The reference's validate_list (core.py:148-167) on a host int64 array:
 * first violation in report order.  Used only to build the exception
 * message once the device pipeline has reported an invalid list. */
int sg_list_violation_host(const int64_t* succ, uint64_t n, sg_violation* v);

#ifdef __cplusplus
}
#endif

#endif /* SG_H */
