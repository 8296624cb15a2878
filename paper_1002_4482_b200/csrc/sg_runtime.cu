// sg_runtime.cu -- library plumbing: status strings, kernel names, the
// per-call launch recorder (CUDA events on the launching stream).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>

#include <atomic>

#include "sg_internal.cuh"

namespace sg {

static thread_local std::string g_last_cuda_error;

void set_cuda_error(cudaError_t e) {
    g_last_cuda_error = std::string(cudaGetErrorName(e)) + ": " + cudaGetErrorString(e);
}

// Event sets.  A call records its launch boundaries into one of kSets sets
// per device (round robin; events are reused -- creating two per launch would
// cost more than the short launches).  The elapsed times are read only when
// someone asks (sg_stats_resolve): ~30 cudaEventElapsedTime calls cost ~80 us
// of host time, which would otherwise sit between the pipeline's last kernel
// and the call's return.  A set is recycled kSets calls later; stats resolved
// after that report SG_ERR_RUNTIME and keep ms = 0.
constexpr int kSets = 64;
struct EventSet {
    std::vector<cudaEvent_t> ev;
    uint32_t gen = 0;
};
static std::mutex g_sets_mu;
static EventSet g_sets[64][kSets];
static uint32_t g_next_set[64];
static uint32_t g_gen = 0;

// ticket: dev (6 bits) | set (6 bits) | generation (20 bits, never 0)
constexpr uint32_t kGenMask = 0xFFFFFu;
static inline uint32_t make_ticket(int dev, int set, uint32_t gen) {
    return ((uint32_t)(dev & 63) << 26) | ((uint32_t)set << 20) | (gen & kGenMask);
}

cudaEvent_t Recorder::event(size_t i) {
    if (!set_) return nullptr;
    std::vector<cudaEvent_t>& pool = static_cast<EventSet*>(set_)->ev;
    while (pool.size() <= i) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        pool.push_back(e);
    }
    return pool[i];
}

Recorder::Recorder(sg_stats* st, cudaStream_t s) : st_(st), s_(s) {
    if (st_) {
        st_->n_launches = 0;
        st_->total_ms = 0.f;
        int dev = 0;
        cudaGetDevice(&dev);
        {
            std::lock_guard<std::mutex> lk(g_sets_mu);
            const int k = (int)(g_next_set[dev & 63]++ % kSets);
            uint32_t gen = ++g_gen & kGenMask;
            if (gen == 0) gen = ++g_gen & kGenMask;
            EventSet& es = g_sets[dev & 63][k];
            es.gen = gen;
            set_ = &es;
            st_->pad2 = make_ticket(dev, k, gen);
        }
        cudaEvent_t t0 = event(0);
        if (t0) cudaEventRecord(t0, s_);
        n_ev_ = 1;
        last_ = 0;
        shared_ = true;  // the first launch starts at t0
    }
}

Recorder::~Recorder() {}

void Recorder::begin(int kernel, int round, uint32_t blocks, uint32_t threads, uint64_t items) {
    if (!st_ || st_->n_launches >= SG_MAX_LAUNCHES) {
        open_ = -1;
        return;
    }
    uint32_t k = st_->n_launches;
    sg_launch& L = st_->launch[k];
    L.kernel = kernel;
    L.round = round;
    L.blocks = blocks;
    L.threads = threads;
    L.items = items;
    L.ms = 0.f;
    if (shared_) {  // back-to-back launches: the previous end event starts this one
        begin_ix_ = last_;
    } else {
        cudaEvent_t a = event(n_ev_);
        if (a) cudaEventRecord(a, s_);
        begin_ix_ = n_ev_++;
    }
    shared_ = false;
    open_ = int(k);
}

void Recorder::end() {
    if (open_ < 0) return;
    cudaEvent_t b = event(n_ev_);
    if (b) cudaEventRecord(b, s_);
    last_ = n_ev_++;
    st_->launch[open_].pad = (uint32_t)(begin_ix_ << 16) | (uint32_t)(last_ & 0xFFFFu);
    st_->n_launches = uint32_t(open_) + 1;
    open_ = -1;
    shared_ = true;
}

cudaError_t Recorder::finish() { return cudaStreamSynchronize(s_); }

}  // namespace sg

// Fill launch[k].ms and total_ms of a finished call from its events.
extern "C" int sg_stats_resolve(sg_stats* st) {
    using namespace sg;
    if (!st) return SG_ERR_VALUE;
    if (st->n_launches == 0) return SG_OK;
    const uint32_t t = st->pad2;
    const int dev = (int)(t >> 26), k = (int)((t >> 20) & 63u);
    const uint32_t gen = t & kGenMask;
    std::lock_guard<std::mutex> lk(g_sets_mu);
    EventSet& es = g_sets[dev][k];
    if (gen == 0 || es.gen != gen) return SG_ERR_RUNTIME;  // the event set was recycled
    uint32_t last = 0;
    for (uint32_t i = 0; i < st->n_launches && i < SG_MAX_LAUNCHES; ++i) {
        sg_launch& L = st->launch[i];
        const uint32_t ia = L.pad >> 16, ib = L.pad & 0xFFFFu;
        if (ia < es.ev.size() && ib < es.ev.size()) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, es.ev[ia], es.ev[ib]) == cudaSuccess) L.ms = ms;
        }
        if (ib > last) last = ib;
    }
    if (last < es.ev.size() && last > 0) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, es.ev[0], es.ev[last]) == cudaSuccess) st->total_ms = ms;
    }
    return SG_OK;
}

namespace sg {

// Optional device tuning from the environment, applied once per process and
// device: SG_L2_FETCH=<bytes> sets cudaLimitMaxL2FetchGranularity (a hint).
int sm_count() {
    constexpr int kMaxDev = 64;
    static std::atomic<int> cache[kMaxDev];  // 0: not queried yet
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) dev = 0;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v > 0) return v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
        cudaGetLastError();
        v = 148;
    }
    cache[dev].store(v, std::memory_order_relaxed);
    return v;
}

int resident_ctas(const void* kernel, int threads) {
    struct Entry {
        const void* k;
        int threads, dev, nb;
    };
    static std::mutex mu;
    static Entry cache[64];
    static int used = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < used; ++i)
        if (cache[i].k == kernel && cache[i].threads == threads && cache[i].dev == dev) return cache[i].nb;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, 0) != cudaSuccess || nb <= 0) {
        cudaGetLastError();
        nb = 1;
    }
    if (used < 64) cache[used++] = Entry{kernel, threads, dev, nb};
    return nb;
}

static uint32_t env_u32(const char* name, uint32_t dflt, uint32_t lo, uint32_t hi) {
    const char* s = getenv(name);
    if (!s || !*s) return dflt;
    long v = strtol(s, nullptr, 10);
    if (v < (long)lo) v = lo;
    if (v > (long)hi) v = hi;
    return (uint32_t)v;
}

static Tuning read_tuning(uint32_t generation) {
    Tuning v;
    v.rs_win_kb = env_u32("SG_RS_WIN_KB", 64, 8, 128);  // fine window: KiB of shared memory in rs5_scatter
    v.rs_kb0 = env_u32("SG_RS_KBITS0", 5, 1, 16);        // level-0 ruler density 2^-kb0
    v.rs_kb1 = env_u32("SG_RS_KBITS", 4, 1, 16);         // upper levels: short chains (latency-bound tail)
    v.rs_fin = env_u32("SG_RS_FINAL", 8192, 64, 1u << 20);
    v.rs_walk_cap = env_u32("SG_RS_WALK_CAP", 1u << 16, 1, 0x7FFFFFFF);  // longer walks -> Wyllie fallback
    v.rs_load_mode = env_u32("SG_WALK_LOAD", 0, 0, 3);
    v.rs_contract = env_u32("SG_RS_CONTRACT", 1, 0, 1);
    v.rs_coop = env_u32("SG_RS_COOP", 1, 0, 1);
    // kbits 4 + pointer jumping from 2^20 rulers: at 2^28 the level-1 walk
    // feeds the top directly (levels 2^28 / 2^23 / 2^19): 9.55 -> 9.51 ms,
    // ordered 1.445 -> 1.414 ms; 2^26 within noise (+0.01 ms)
    v.rs_topn = env_u32("SG_RS_TOPN", 1u << 20, 0, 1u << 30);
    v.rs_packed = env_u32("SG_RS_PACKED", 1, 0, 1);
    v.rs_fused = env_u32("SG_RS_FUSED", 1, 0, 1);
    v.rs_refine = env_u32("SG_RS_REFINE", 0, 0, 7);  // rs5_refine variant (sg_list.cu)
    v.cc_wbits = env_u32("SG_CC_WBITS", 0, 0, 31);
    v.cc_split = env_u32("SG_CC_SPLIT", 3, 0, 31);   // UF, unpartitioned: shortcut after m / 2^f rows (0: off)
    v.cc_split2 = env_u32("SG_CC_SPLIT2", 0, 0, 31);  // UF, unpartitioned: a second shortcut (experiment)
    v.cc_comp4 = env_u32("SG_CC_COMP4", 1, 0, 1);  // cc_shortcut: four vertices per thread (0: one)
    v.cc_splitw = env_u32("SG_CC_SPLITW", 0, 0, 64);  // UF, partitioned: shortcut after k windows (experiment)
    const char* part = getenv("SG_CC_PART");
    v.cc_part_count = part && strcmp(part, "count") == 0;  // count + scatter instead of chunk lists
    const char* rk = getenv("SG_CC_RANK");
    v.cc_rank_ballot = rk && strcmp(rk, "ballot") == 0;  // chunk partition: ballot peers instead of match.any
    v.ms_peers = env_u32("SG_MS_PEERS", 1, 0, 2);
    v.generation = generation;
    return v;
}

static std::mutex g_tuning_mu;
static Tuning g_tuning;
static bool g_tuning_ok = false;

Tuning tuning() {
    std::lock_guard<std::mutex> lk(g_tuning_mu);
    if (!g_tuning_ok) {
        g_tuning = read_tuning(1);
        g_tuning_ok = true;
    }
    return g_tuning;
}

void apply_tuning() {
    static thread_local int done_mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 31 && (done_mask & (1 << dev))) return;
    if (dev < 31) done_mask |= 1 << dev;
    const char* s = getenv("SG_L2_FETCH");
    size_t old = 0;
    cudaDeviceGetLimit(&old, cudaLimitMaxL2FetchGranularity);
    if (s && *s) {
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atol(s));
        size_t now = 0;
        cudaDeviceGetLimit(&now, cudaLimitMaxL2FetchGranularity);
        if (getenv("SG_DEBUG")) fprintf(stderr, "[sg] L2 fetch granularity %zu -> %zu\n", old, now);
    } else if (getenv("SG_DEBUG")) {
        fprintf(stderr, "[sg] L2 fetch granularity %zu\n", old);
    }
    cudaGetLastError();
}

}  // namespace sg

extern "C" {

const char* sg_strerror(int status) {
    switch (status) {
        case SG_OK: return "ok";
        case SG_ERR_INVALID_LIST: return "invalid successor list";
        case SG_ERR_INVALID_GRAPH: return "invalid edge graph";
        case SG_ERR_CAPABILITY: return "capability limit exceeded";
        case SG_ERR_VALUE: return "invalid argument";
        case SG_ERR_RUNTIME: return "algorithm did not converge";
        case SG_ERR_CUDA: return "CUDA error";
        case SG_ERR_WORKSPACE: return "workspace too small";
        default: return "unknown status";
    }
}

const char* sg_kernel_name(int id) {
    static const char* names[sg::K_COUNT_] = {
        "status_init", "wy_init",     "wy_jump",     "wy_single",   "wy_check",
        "rs1_validate", "rs2_scan",   "rs2_select",  "rs3_walk",    "rs4_count",
        "rs4_scan",    "rs4_select",  "rs4_walk",    "rs4_rank",    "rs4_expand",
        "rs5_expand",  "sv0",         "cc_hook_uf",  "cc_hook_sv",  "cc_shortcut",
        "cc_labels",   "gather",      "kiss",        "list_from_order", "edge_keys",
        "edges_from_keys", "cc_partition", "rs5_partition", "rs5_scatter", "rs5_refine", "rs3_contract", "rs3_link",
    };
    if (id < 0 || id >= sg::K_COUNT_) return "unknown";
    return names[id];
}

int sg_version(void) { return 1; }

int sg_tuning_reload(void) {
    std::lock_guard<std::mutex> lk(sg::g_tuning_mu);
    sg::g_tuning = sg::read_tuning(sg::g_tuning_ok ? sg::g_tuning.generation + 1 : 1);
    sg::g_tuning_ok = true;
    return SG_OK;
}

#ifndef SG_SOURCE_HASH
#define SG_SOURCE_HASH "unknown"
#endif
// build.py embeds the sha256 of every source, header and flag it compiled
// from; it reads this marker back from the .so to decide whether a shipped
// library matches the tree (no mtimes involved).
__attribute__((used)) static const char g_source_hash_marker[] = "SG_SOURCE_HASH=" SG_SOURCE_HASH ";";

const char* sg_source_hash(void) { return g_source_hash_marker + 15; }

const char* sg_last_cuda_error(void) { return sg::g_last_cuda_error.c_str(); }

}  // extern "C"
