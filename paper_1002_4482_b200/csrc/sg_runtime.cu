// sg_runtime.cu -- library plumbing: status strings, kernel names, the
// per-call launch recorder (CUDA events on the launching stream).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>

#include "sg_internal.cuh"

namespace sg {

static thread_local std::string g_last_cuda_error;

void set_cuda_error(cudaError_t e) {
    g_last_cuda_error = std::string(cudaGetErrorName(e)) + ": " + cudaGetErrorString(e);
}

// Events are reused across calls (one pool per device per host thread):
// creating two events per launch would cost more than the short launches.
static thread_local std::vector<cudaEvent_t> g_pool[64];

static cudaEvent_t pool_event(size_t i) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::vector<cudaEvent_t>& pool = g_pool[dev & 63];
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
        t0_ = pool_event(0);
        if (t0_) cudaEventRecord(t0_, s_);
        ev_.push_back(t0_);
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
    L.pad = 0;
    if (shared_) {  // back-to-back launches: the previous end event starts this one
        begin_ix_.push_back(ev_.size() - 1);
    } else {
        cudaEvent_t a = pool_event(ev_.size());
        if (a) cudaEventRecord(a, s_);
        ev_.push_back(a);
        begin_ix_.push_back(ev_.size() - 1);
    }
    shared_ = false;
    open_ = int(k);
}

void Recorder::end() {
    if (open_ < 0) return;
    cudaEvent_t b = pool_event(ev_.size());
    if (b) cudaEventRecord(b, s_);
    ev_.push_back(b);
    end_ix_.push_back(ev_.size() - 1);
    st_->n_launches = uint32_t(open_) + 1;
    open_ = -1;
    shared_ = true;
}

cudaError_t Recorder::finish() {
    cudaError_t e = cudaStreamSynchronize(s_);
    if (e != cudaSuccess || !st_) return e;
    for (uint32_t k = 0; k < st_->n_launches && k < begin_ix_.size() && k < end_ix_.size(); ++k) {
        const size_t ia = begin_ix_[k], ib = end_ix_[k];
        if (ib < ev_.size() && ev_[ia] && ev_[ib]) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, ev_[ia], ev_[ib]) == cudaSuccess) st_->launch[k].ms = ms;
        }
    }
    if (ev_.size() > 1 && ev_[0] && ev_.back()) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ev_[0], ev_.back()) == cudaSuccess) st_->total_ms = ms;
    }
    return cudaSuccess;
}

// Optional device tuning from the environment, applied once per process and
// device: SG_L2_FETCH=<bytes> sets cudaLimitMaxL2FetchGranularity (a hint).
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

const char* sg_last_cuda_error(void) { return sg::g_last_cuda_error.c_str(); }

}  // extern "C"
