// sg_internal.cuh -- shared device/host helpers for libsg (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <chrono>
#include <cstdio>
#include <map>
#include <utility>
#include <vector>

#include "sg.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libsg is built for sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

namespace sg {

constexpr uint32_t NIL = 0xFFFFFFFFu;
constexpr unsigned long long NONE64 = ~0ull;
// SMs of the current device (148 on a B200), queried once per device; every
// persistent grid is sized from it
int sm_count();
// CTAs of `kernel` resident per SM at `threads` threads (no dynamic shared
// memory), queried once per (kernel, threads, device): grids of persistent
// loops are sized sm_count() x this, so no CTA waits for a slot
int resident_ctas(const void* kernel, int threads);
template <class K>
int resident_ctas(K* kernel, int threads) {
    return resident_ctas(reinterpret_cast<const void*>(kernel), threads);
}

// Experiment switches (SG_* environment variables).  The defaults are the
// measured configuration; the switches exist to re-run the comparisons
// DESIGN.md records and to force rare paths in tests.  They are parsed once
// and again only when sg_tuning_reload() is called (tests do, after
// changing the environment), never per call.
struct Tuning {
    // list ranking (sg_list.cu)
    uint32_t rs_win_kb, rs_kb0, rs_kb1, rs_fin, rs_walk_cap, rs_load_mode, rs_contract, rs_coop, rs_topn,
        rs_packed, rs_fused, rs_refine;
    // components (sg_cc.cu): window bits (0 = default), one-pass tile partition
    uint32_t cc_wbits, cc_part_count, cc_rank_ballot, cc_split, cc_split2, cc_splitw, cc_comp4;
    // block multisplit peer ranking (sg_msplit.cuh): 0 match.any, 1 ballots, 2 alternate
    uint32_t ms_peers;
    uint32_t generation;  // bumped by every reload
};
Tuning tuning();

// Kernel ids; names are returned by sg_kernel_name().  Names follow the
// reference's phase names where a kernel does that phase's job
// (listrank.py:197-382, concomp.py:69-205).
enum KernelId : int {
    K_STATUS_INIT = 0,
    K_WY_INIT,        // wy_init     listrank.py:98-102 (+ device validation)
    K_WY_JUMP,        // wy_jump     listrank.py:104-117
    K_WY_SINGLE,      // wy_single   listrank.py:127-148
    K_WY_CHECK,       // wy_check    head reaches tail with rank n-1
    K_RS_COUNT,       // rs1_validate: validation + ruling-set census (RS1/RS2)
    K_RS_SCAN,        // rs2_scan:   tile offsets of the ruling set
    K_RS_SELECT,      // rs2_select: install splitter ids (listrank.py:234-249)
    K_RS3_WALK,       // rs3_walk:   sublist walk, level 0 (listrank.py:252-299)
    K_RS4_COUNT,      // rs4_count:  ruling-set census at level >= 1
    K_RS4_SCAN,       // rs4_scan
    K_RS4_SELECT,     // rs4_select
    K_RS4_WALK,       // rs4_walk:   weighted sublist walk, level >= 1
    K_RS4_RANK,       // rs4_rank:   single-CTA weighted pointer jumping (listrank.py:333-342)
    K_RS4_EXPAND,     // rs4_expand: level >= 1 fix-up
    K_RS5_EXPAND,     // rs5_expand: rank = splitter rank - local (listrank.py:360-382)
    K_CC_INIT,        // sv0         D[i] = i (concomp.py:69-79)
    K_CC_HOOK_UF,     // cc_hook_uf  CAS root hooking over the stored edges
    K_CC_HOOK_SV,     // cc_hook_sv  atomicMin conditional hook (concomp.py:136-154)
    K_CC_COMPRESS,    // cc_shortcut root chase to stars (concomp.py:88-103,178-180)
    K_CC_LABELS,      // cc_labels   dtype conversion of the parent array
    K_GATHER,         // gather
    K_KISS,           // kiss        device KISS64 draws (gen.py:51-64)
    K_LIST_FROM_ORDER,
    K_EDGE_KEYS,
    K_EDGES_FROM_KEYS,
    K_CC_PARTITION,   // cc_partition stable split of the edges by endpoint window
    K_RS5_PARTITION,  // rs5_partition: rank the walk records, split by output window
    K_RS5_SCATTER,    // rs5_scatter:   fine window -> shared memory -> coalesced ranks
    K_RS5_REFINE,     // rs5_refine:    coarse window -> fine windows
    K_RS_CONTRACT,    // rs3_contract:  tile contraction of a local layout (segments in shared memory)
    K_RS_CONTRACT_LINK,  // rs3_link:   contracted-list successors
    K_COUNT_
};

// Device status block for one list-ranking call (zeroed / ~0 by status_init).
struct ListStatus {
    unsigned long long oor_first;   // min index with succ out of range
    unsigned long long loop_first;  // min index with succ[i] == i
    unsigned long long loop_count;  // number of self-loops
    unsigned long long overflow;    // walk cap or level capacity exceeded
    unsigned long long head_sum;    // final inclusive suffix sum at the head
    unsigned long long head_ok;     // 1: the head's pointer reached the tail
    unsigned long long bad;         // walk saw an out-of-range successor
    unsigned long long local;       // 1: local layout, ranked by tile contraction
    unsigned long long R[SG_MAX_LEVELS + 1];      // nodes per level (R[0] = n)
    unsigned long long qhead[SG_MAX_LEVELS + 1];  // walk work-queue heads
    unsigned long long chunks;      // record chunks handed out by the level-0 record walk
    unsigned long long top_live[3]; // cooperative top-level jumping: live pointers seen per round (mod 3)
};

// Error plumbing -------------------------------------------------------------
void set_cuda_error(cudaError_t e);
void apply_tuning();

#define SG_CUDA(call)                                   \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) {                        \
            ::sg::set_cuda_error(e_);                   \
            return SG_ERR_CUDA;                         \
        }                                               \
    } while (0)

#define SG_LAUNCH_CHECK()                               \
    do {                                                \
        cudaError_t e_ = cudaGetLastError();            \
        if (e_ != cudaSuccess) {                        \
            ::sg::set_cuda_error(e_);                   \
            return SG_ERR_CUDA;                         \
        }                                               \
    } while (0)

// Per-call launch recorder: brackets every launch with events on the
// launching stream so ExecStats gets device time per kernel.
class Recorder {
  public:
    Recorder(sg_stats* st, cudaStream_t s);
    ~Recorder();
    // returns false if the launch table is full (recording stops, launches do not)
    void begin(int kernel, int round, uint32_t blocks, uint32_t threads, uint64_t items);
    void end();
    // synchronises the stream; the ms fields are filled later by
    // sg_stats_resolve from the call's event set (ticket in sg_stats.pad2,
    // event indices in sg_launch.pad)
    cudaError_t finish();

  private:
    cudaEvent_t event(size_t i);
    sg_stats* st_;
    cudaStream_t s_;
    void* set_ = nullptr;  // this call's event set
    size_t n_ev_ = 0;      // events recorded so far
    size_t last_ = 0;      // index of the last end event
    size_t begin_ix_ = 0;  // begin event of the open launch
    int open_ = -1;
    bool shared_ = false;  // the last end event doubles as the next begin event
};

// SG_HOST_TIMING=1: host-side timestamps of a call's phases on stderr
struct HostClock {
    const char* name;
    bool on;
    std::chrono::steady_clock::time_point t0, last;
    explicit HostClock(const char* nm) : name(nm), on(getenv("SG_HOST_TIMING") != nullptr) {
        if (on) t0 = last = std::chrono::steady_clock::now();
    }
    void mark(const char* what) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[sg %s] %-20s +%8.1f us  (total %8.1f us)\n", name, what,
                std::chrono::duration<double, std::micro>(t - last).count(),
                std::chrono::duration<double, std::micro>(t - t0).count());
        last = t;
    }
};

// Raise a kernel's dynamic shared memory limit once per device (the attribute
// persists; setting it on every call costs host time on short pipelines).
template <class F>
inline cudaError_t set_smem_max(F* f, size_t bytes) {
    static thread_local std::map<std::pair<int, const void*>, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    size_t& have = done[std::make_pair(dev, (const void*)f)];
    if (have >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

// Workspace carving ------------------------------------------------------------
struct Carver {
    char* base;
    size_t cap;
    size_t off = 0;
    bool ok = true;
    Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
    template <class T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        size_t bytes = count * sizeof(T);
        if (base == nullptr) {  // sizing pass
            off += bytes;
            return nullptr;
        }
        if (off + bytes > cap) {
            ok = false;
            return nullptr;
        }
        T* p = reinterpret_cast<T*>(base + off);
        off += bytes;
        return p;
    }
};

inline uint32_t grid_for(uint64_t items, uint32_t threads, uint32_t per_thread, uint32_t max_blocks) {
    uint64_t b = (items + uint64_t(threads) * per_thread - 1) / (uint64_t(threads) * per_thread);
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return uint32_t(b);
}

// Device helpers ---------------------------------------------------------------
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Load through L2 only (parent arrays that other CTAs update).
__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }

}  // namespace sg
